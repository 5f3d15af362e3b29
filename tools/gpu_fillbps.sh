# Sweep the overlapped fill's grid cap (MANDEL_FILL_BPS blocks per SM) on full C3/C5 and the
# emulated 8-way C3 rank shares.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for PT in "" "FILL_BPS=1" "FILL_BPS=2" "FILL_BPS=4"; do
  SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PT'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
  echo "[$PT]"
  MANDEL_B200_LIB=$SO timeout 300 python tools/ab.py C3 C5 --reps 5 --variants b200 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['w'], round(d['b200']['ms_mean'],3), round(d['b200']['ms_notiming_mean'],3), d['b200']['kernels'])"
  MANDEL_B200_LIB=$SO timeout 300 python tools/emulate_scaling.py C3 --ranks 8 --deals lpt --reps 3 2>&1 | grep '"deal"' | cut -c1-120
done

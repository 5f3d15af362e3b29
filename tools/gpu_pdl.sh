# PDL A/B: parity subset with the in-tree build (PDL on), then C3/C5 timing and the emulated
# 8-way C3 rank for MANDEL_PDL=1 (in-tree) vs MANDEL_PDL=0.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or tiles_subset or full_size_ask or groups or ab_variants" > gpurun_out/pytest_pdl.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_pdl.log
for PT in "" "PDL=0"; do
  SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PT'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
  echo "[$PT]"
  for rep in 1 2; do
  MANDEL_B200_LIB=$SO timeout 300 python tools/ab.py C3 C5 --reps 5 --variants b200 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['w'], round(d['b200']['ms_mean'],3), 'notiming', round(d['b200']['ms_notiming_mean'],3))"
  MANDEL_B200_LIB=$SO timeout 300 python tools/emulate_scaling.py C3 --ranks 1,8 --deals lpt --reps 5 2>&1 | grep '"deal"' | cut -c1-120
  done
done

# Two library variants, alternating, C3 + C5 timing (5 reps x 3 rounds) and the 8-way rank.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mk() { python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$1'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))"; }
A=$(mk "$PA"); B=$(mk "$PB")
for round in 1 2 3; do
  for V in A B; do
    SO=$A; [ $V = B ] && SO=$B
    echo "[$V round $round]"
    MANDEL_B200_LIB=$SO timeout 300 python tools/ab.py C3 C5 --reps 5 --variants b200 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['w'], round(d['b200']['ms_notiming_mean'],3), {k: round(v, 3) for k, v in d['b200']['kernels'].items()})"
  done
done

# Per-level border time, default vs a -D variant ($PB), full image and one 8-way rank.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PB'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
for LIB in in-tree $SO; do
  for TO in 0 8; do
    if [ $LIB = in-tree ]; then E=""; else E="MANDEL_B200_LIB=$LIB"; fi
    env $E timeout 300 python tools/level_profile.py C3 --reps 5 --tiles-of $TO 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$LIB'[-12:], 'tiles_of=$TO', [round(x['border_ms']*1000) for x in d['levels']], round(d['leaf_ms'],3))"
  done
done

# A/B of two variants: C3/C5 untimed step + per-kernel breakdown, and the 8-way C3 rank.
bash tools/gpu_ab2.sh
for PT in "$PA" "$PB"; do
  SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PT'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
  echo "[$PT]"
  MANDEL_B200_LIB=$SO timeout 300 python tools/emulate_scaling.py C3 --ranks 8 --deals lpt --reps 5 2>&1 | grep '"deal"' | grep -o '"max_rank_ms": [0-9.]*'
done

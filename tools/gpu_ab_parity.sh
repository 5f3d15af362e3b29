# A/B of two variants (tools/gpu_ab3.sh) plus the parity subset run against variant B's library.
bash tools/gpu_ab3.sh
SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PB'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
MANDEL_B200_LIB=$SO timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or tiles_subset or full_size_ask or tile_costs or maxdwell_not_multiple or outside_radius" 2>&1 | tail -2

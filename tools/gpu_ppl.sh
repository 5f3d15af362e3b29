# Sweep the scalar refill engine's launch shape (MANDEL_RF_PPL / MANDEL_RF_MINW) on full C3
# and on the emulated 8-way C3 rank shares.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for PT in ${POINTS:-"" "RF_PPL=4u" "RF_PPL=2u" "RF_PPL=1u" "RF_MINW=16u" "RF_MINW=16u,RF_PPL=2u" "RF_MINW=4u"}; do
  SO=$(python -c "
import hashlib, sys; sys.path.insert(0, '.')
from paper_2206_02255_b200 import build
pt='$PT'; defs=['MANDEL_'+d for d in pt.split(',') if d]
so='/tmp/libm_'+hashlib.md5(pt.encode()).hexdigest()[:8]+'.so'
print(build.build(out=so, defines=defs))")
  echo "[$PT]"
  MANDEL_B200_LIB=$SO timeout 300 python tools/emulate_scaling.py C3 --ranks 1,8 --deals lpt --reps 3 2>&1 | grep '"deal"' | cut -c1-160
done

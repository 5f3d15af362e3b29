set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/debug_mismatch.py C1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/libL.so', defines=['MANDEL_RFB_PACK=0'])
build.build(out='/tmp/libB.so', defines=['MANDEL_RFL_PACK=0'])"
MANDEL_B200_LIB=/tmp/libL.so python tools/debug_mismatch.py C1
MANDEL_B200_LIB=/tmp/libB.so python tools/debug_mismatch.py C1

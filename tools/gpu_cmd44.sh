set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/libBS.so', defines=['MANDEL_RFB_PACK=0'])
build.build(out='/tmp/libBS4.so', defines=['MANDEL_RFB_PACK=0', 'MANDEL_RF_MINB=4'])"
for L in in-tree /tmp/libBS.so /tmp/libBS4.so; do
  if [ "$L" != "in-tree" ]; then export MANDEL_B200_LIB=$L; fi
  echo "== $L"
  timeout 300 python tools/emulate_scaling.py C3 --ranks 1,8 --deals costrank > gpurun_out/emu44.jsonl 2>&1; grep '"deal"' gpurun_out/emu44.jsonl | cut -c1-200
  timeout 300 python tools/level_profile.py C3 --tiles-of 8 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print([ (l['level'], l['border_ms']) for l in r['levels']], r['leaf_ms'])"
done

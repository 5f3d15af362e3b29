set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pt in "RF_MINW=2" "RF_MINW=4" "RF_MINW=6" "RF_MINW=12" "RF_PPL=2,RF_MINW=4" "RF_PPL=1,RF_MINW=6" "RF_PPL=4,RF_MINW=6" "RF_PPL=2,RF_MINW=12"; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/lib_rp.so', defines=['MANDEL_'+d for d in '$pt'.split(',')])"
  MANDEL_B200_LIB=/tmp/lib_rp.so timeout 600 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof15.jsonl 2>&1; echo "== $pt"; head -1 gpurun_out/rankprof15.jsonl; grep "border\|leaf" gpurun_out/rankprof15.jsonl | python -c "
import json,sys
r=[json.loads(l) for l in sys.stdin]
print('border rank ms', round(sum(x['rank_ms'] for x in r if 'border' in x['kernel']),3), 'full', round(sum(x['full_ms'] for x in r if 'border' in x['kernel']),3), 'leaf rank', [x['rank_ms'] for x in r if 'leaf' in x['kernel']], 'full', [x['full_ms'] for x in r if 'leaf' in x['kernel']])"
done

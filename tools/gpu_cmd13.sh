set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build13.log 2>&1
timeout 1200 python tools/tune_refill.py C3 C5 --points "RF_WPS=12;RF_WPS=2;RF_WPS=3;RF_WPS=4;RF_WPS=6;RFL_WPS=4;RFL_WPS=6;RFL_WPS=8" > gpurun_out/tune13.txt 2>&1; cat gpurun_out/tune13.txt | cut -c1-300
for pt in "RF_WPS=12" "RF_WPS=3" "RF_WPS=4,RFL_WPS=6"; do
  python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/lib_rp.so', defines=['MANDEL_'+d for d in '$pt'.split(',')])"
  MANDEL_B200_LIB=/tmp/lib_rp.so timeout 600 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof13.jsonl 2>&1; echo "$pt"; head -1 gpurun_out/rankprof13.jsonl; grep border gpurun_out/rankprof13.jsonl | cut -c1-200 | head -3
done

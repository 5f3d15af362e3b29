set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest23.log 2>&1; tail -2 gpurun_out/pytest23.log
timeout 600 python tools/tune_ex.py C3 C5 > gpurun_out/tune_ex23.txt 2>&1; cat gpurun_out/tune_ex23.txt
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/lib64.so', defines=['MANDEL_RF_TPB=64'])"
MANDEL_B200_LIB=/tmp/lib64.so timeout 300 python tools/ab.py C3 --variants b200,g2,g4 > gpurun_out/ab23_tpb64.jsonl 2>&1; cut -c1-200 gpurun_out/ab23_tpb64.jsonl
for G in 1 2 4; do MANDEL_B200_LIB=/tmp/lib64.so timeout 300 python tools/rank_profile.py C3 --P 8 --groups $G > gpurun_out/rp23_g$G.jsonl 2>&1; head -1 gpurun_out/rp23_g$G.jsonl; done
timeout 600 python bench.py --workload C4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench23_c4.json 2> gpurun_out/bench23_c4.err; cut -c1-1500 gpurun_out/bench23_c4.json; tail -3 gpurun_out/bench23_c4.err

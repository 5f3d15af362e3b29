set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/libS.so', defines=['MANDEL_RFB_PACK=0','MANDEL_RFL_PACK=0'])
build.build(out='/tmp/libP3.so', defines=['MANDEL_RF2_MINB=3'])"
for V in S P3; do
MANDEL_B200_LIB=/tmp/lib$V.so timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_b200_leaf" -s 1 -c 1 -o gpurun_out/leaf_$V -f python tools/prof_step.py --workload C3 --warm 1 --no-ex > gpurun_out/ncu27_$V.log 2>&1; tail -2 gpurun_out/ncu27_$V.log
done

set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/tune_refill.py C3 C5 --points ";RFB_PACK=1;RFB_PACK=1,RFB_PRE=0;RFB_PACK=1,RF2_MINB=4" > gpurun_out/tune53.txt 2>&1
python - <<'PY'
import json,re
txt=open('gpurun_out/tune53.txt').read()
for m in re.finditer(r'(\[[^\]]*\])?\s*(\{"w".*?\}\}\})', txt):
    d=json.loads(m.group(2)); print((m.group(1) or '').ljust(34), d['w'], round(d['b200']['ms_mean'],3), d['b200']['kernels'].get('b200_border'), d['b200']['kernels'].get('b200_leaf'), d['b200']['same_image'])
PY
for P in "" "MANDEL_RFB_PACK=1"; do
python -c "
import sys; sys.path.insert(0,'.')
from paper_2206_02255_b200 import build
build.build(out='/tmp/libE.so', defines=[d for d in ['$P'] if d])"
MANDEL_B200_LIB=/tmp/libE.so timeout 300 python tools/emulate_scaling.py C3 --ranks 1,8 --deals costrank > gpurun_out/emu53.jsonl 2>&1; echo "$P"; grep '"deal"' gpurun_out/emu53.jsonl | cut -c1-150
done

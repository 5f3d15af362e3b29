set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest51.log 2>&1; tail -2 gpurun_out/pytest51.log
timeout 1200 python tools/tune_refill.py C3 C5 --points ";RFL_PRE=0;RFL_PRE=8;RFL_PRE=32;RFL_PRE=16,RF2_MINB=2" > gpurun_out/tune51.txt 2>&1
python - <<'PY'
import json,re
txt=open('gpurun_out/tune51.txt').read()
for m in re.finditer(r'(\[[^\]]*\])?\s*(\{"w".*?\}\}\})', txt):
    d=json.loads(m.group(2)); print((m.group(1) or '').ljust(30), d['w'], round(d['b200']['ms_mean'],3), d['b200']['kernels'].get('b200_border'), d['b200']['kernels'].get('b200_leaf'), d['b200']['same_image'])
PY

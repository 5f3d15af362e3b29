set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/tune_refill.py C3 C5 --points "RFB_PACK=0,RF_MINB=3;RFB_PACK=0,RF_MINB=4;RFB_PACK=0,RF_MINB=5;RFB_PACK=0,RF_MINB=4,RFB_T=2;RFB_PACK=0,RF_MINB=4,RFB_T=8;RFB_PACK=0,RF_MINB=4,RFB_CH=32;RFB_PACK=0,RF_MINB=4,RFB_K=8" > gpurun_out/tune46.txt 2>&1
python - <<'PY'
import json,re
for line in open('gpurun_out/tune46.txt'):
    m = re.match(r'\[(.*?)\] (\{.*?\})\s*(\{.*\})?', line.strip())
    if not m: 
        try:
            d=json.loads(line); print('   ', d['w'], round(d['b200']['ms_mean'],3), d['b200']['kernels'].get('b200_border'), d['b200']['kernels'].get('b200_leaf'))
        except Exception: pass
        continue
    d=json.loads(m.group(2)); print(m.group(1), d['w'], round(d['b200']['ms_mean'],3), d['b200']['kernels'].get('b200_border'), d['b200']['kernels'].get('b200_leaf'))
PY

# Packed (FMUL2/FADD2) refill engine: parity + A/B against the scalar engine and knob points.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest24.log 2>&1; tail -3 gpurun_out/pytest24.log
timeout 1500 python tools/tune_refill.py C3 C5 --points ";RFB_PACK=0,RFL_PACK=0;RF2_MINB=3;RF2_MINB=5;RFL2_T=8,RFB2_T=4;RFL2_T=24,RFB2_T=12;RFL_K=32,RFB_K=32" > gpurun_out/tune24.txt 2>&1; cat gpurun_out/tune24.txt | cut -c1-700

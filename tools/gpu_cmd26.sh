set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/debug_mismatch.py C1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest26.log 2>&1; tail -3 gpurun_out/pytest26.log
timeout 1500 python tools/tune_refill.py C3 C5 --points ";RF2_MINB=3;RF2_MINB=3,RFL2_T=24,RFB2_T=12;RF2_MINB=3,RFL_K=32,RFB_K=32;RF2_MINB=2" > gpurun_out/tune26.txt 2>&1; cat gpurun_out/tune26.txt | cut -c1-600

set -x
./tools/micro/fp32x2 > gpurun_out/micro_fp32x2.txt 2>&1; cat gpurun_out/micro_fp32x2.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu3.log
timeout 600 python tools/ab.py C3 C5 > gpurun_out/ab3.jsonl 2>&1; cat gpurun_out/ab3.jsonl
timeout 900 python tools/tune_refill.py C3 C5 --points 16:16:128,16:8:128,16:16:64,32:16:128,16:24:128 > gpurun_out/tune3.txt 2>&1; cat gpurun_out/tune3.txt

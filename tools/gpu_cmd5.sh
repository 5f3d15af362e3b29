set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build5.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu5.log
timeout 600 python tools/ab.py C3 C5 > gpurun_out/ab5.jsonl 2>&1; cat gpurun_out/ab5.jsonl
timeout 900 python tools/tune_refill.py C3 C5 > gpurun_out/tune5.txt 2>&1; cat gpurun_out/tune5.txt
timeout 900 python tools/sweep_c2.py > gpurun_out/sweep_c2.log 2>&1; tail -3 gpurun_out/sweep_c2.log

set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu2.log
timeout 600 python tools/ab.py C3 C5 C1 --ex > gpurun_out/ab2.jsonl 2>&1; cat gpurun_out/ab2.jsonl
timeout 900 python tools/tune_refill.py C3 > gpurun_out/tune2.txt 2>&1; cat gpurun_out/tune2.txt

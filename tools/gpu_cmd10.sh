set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build10.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu10.log
timeout 600 python tools/ab.py C3 C5 --variants b200,serial > gpurun_out/ab10.jsonl 2>&1; cat gpurun_out/ab10.jsonl
timeout 900 python tools/emulate_scaling.py C3 --deals costrank > gpurun_out/emul10.jsonl 2>&1; head -4 gpurun_out/emul10.jsonl

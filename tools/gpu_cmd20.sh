set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or random_small or groups or maxdwell or edge" > gpurun_out/pytest20.log 2>&1; tail -3 gpurun_out/pytest20.log

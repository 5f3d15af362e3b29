python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_3d.py -x -q > gpurun_out/pytest_3d.log 2>&1; echo rc=$?; tail -4 gpurun_out/pytest_3d.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 600 python tools/bench3d.py V1 V2 > gpurun_out/bench3d.jsonl 2>&1; cut -c1-900 gpurun_out/bench3d.jsonl

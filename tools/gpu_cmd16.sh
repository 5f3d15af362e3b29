set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or random_small or groups or maxdwell" > gpurun_out/pytest16.log 2>&1; tail -2 gpurun_out/pytest16.log
timeout 600 python tools/trace_refill.py C3 --P 8 > gpurun_out/trace16.jsonl 2>&1; cat gpurun_out/trace16.jsonl

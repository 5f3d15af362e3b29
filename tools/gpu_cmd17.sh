set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or random_small or groups or maxdwell or full_size" > gpurun_out/pytest18.log 2>&1; tail -2 gpurun_out/pytest18.log
timeout 600 python tools/trace_refill.py C3 --P 8 > gpurun_out/trace18.jsonl 2>&1; cat gpurun_out/trace18.jsonl
timeout 600 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof18.jsonl 2>&1; head -1 gpurun_out/rankprof18.jsonl
timeout 600 python tools/ab.py C3 C5 --variants b200 > gpurun_out/ab18.jsonl 2>&1; cut -c1-300 gpurun_out/ab18.jsonl

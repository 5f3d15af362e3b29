python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "defer" > gpurun_out/pytest_defer.log 2>&1; tail -5 gpurun_out/pytest_defer.log
timeout 600 python tools/ab.py C3 C5 --reps 5 --variants b200,d128,d256,d512,d1024 > gpurun_out/ab_defer.jsonl 2>&1; cat gpurun_out/ab_defer.jsonl | cut -c1-3000
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,8 --deals costrank --defer 256 > gpurun_out/emu_defer.jsonl 2>&1; head -3 gpurun_out/emu_defer.jsonl

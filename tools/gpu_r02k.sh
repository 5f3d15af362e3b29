#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sampled or frame_loop or device or tile_costs or subset or groups" 2>&1 | tail -3
timeout 600 python tools/cost_overhead.py C3 C5 > gpurun_out/cost_overhead.jsonl 2>&1; cat gpurun_out/cost_overhead.jsonl
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl | head -2
done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; head -c 400 gpurun_out/bench.json; echo
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log

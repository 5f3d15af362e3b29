#!/bin/bash
# Round-2 re-entry check of HEAD: full GPU suite, bench line, A/B vs HEAD~1, emulated scaling.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json | head -c 600; echo
timeout 1500 python tools/ab_variants.py run base prev --workloads C3,C5,C4,C3r8 --rounds 3 --reps 5 > gpurun_out/ab_d.jsonl 2>&1; tail -6 gpurun_out/ab_d.jsonl
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl | head -2
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2

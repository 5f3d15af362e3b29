#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python tools/cost_overhead.py C3 C5 > gpurun_out/cost_overhead.jsonl 2>&1; cat gpurun_out/cost_overhead.jsonl
timeout 1800 python tools/ab_variants.py run base ckpt1 ppl16 ppl32 ppl4 --workloads C3,C5,C4,C3r8 --rounds 3 --reps 5 > gpurun_out/ab_g.jsonl 2>&1; grep -A5 summary gpurun_out/ab_g.jsonl | tail -5

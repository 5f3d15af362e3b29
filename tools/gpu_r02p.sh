#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 2400 python tools/ab_variants.py run base prev bk16 lk16 lk64 --workloads C3,C5,C4,C3r8 --rounds 3 --reps 5 --check > gpurun_out/ab_p.jsonl 2>&1; grep -A5 summary gpurun_out/ab_p.jsonl | tail -5; grep -o '"tiles_differing_from_oracle": [0-9]*' gpurun_out/ab_p.jsonl | sort | uniq -c
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; head -c 600 gpurun_out/bench.json; echo

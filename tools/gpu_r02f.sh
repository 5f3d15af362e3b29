#!/bin/bash
# sampled tile costs + lagged plan + scalar-engine checkpoints: tests, A/B, emulated scaling
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sampled or frame_loop or device or tile_costs" 2>&1 | tail -3
timeout 1800 python tools/ab_variants.py run base head ckpt2 ckpt4 k16c2 --workloads C3,C5,C4,C3r8 --rounds 3 --reps 5 --check > gpurun_out/ab_f.jsonl 2>&1; tail -6 gpurun_out/ab_f.jsonl; grep -o '"variant": "[a-z0-9]*", "w": "C[0-9]"\|tiles_differing_from_oracle": [0-9]*' gpurun_out/ab_f.jsonl | paste - - | sort | uniq | head -20
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl | head -2
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log

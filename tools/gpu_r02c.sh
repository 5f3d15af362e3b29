mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_parity.py -x -q -k "device or one_graph or ask_c1 or random_small or edge or tiles_subset or groups or full_image or tile_costs or to_host" 2>&1 | tail -3
timeout 1500 python tools/ab_variants.py run base prev --workloads C3,C5,C3r8 --rounds 3 --reps 5 > gpurun_out/ab_c.jsonl 2>&1; tail -4 gpurun_out/ab_c.jsonl
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl | head -2
done

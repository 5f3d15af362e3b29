mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "device or one_graph or ask_c1 or random_small or edge or tiles_subset or groups" 2>&1 | tail -3
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl | head -4
done
bash tools/gpu_sanitize.sh

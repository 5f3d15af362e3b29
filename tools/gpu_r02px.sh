# Per-pixel cost in the sampled counters: the sampled-cost and frame-loop tests, bench N=2 gloo
# test, and the emulated scaling of C3/C5/C4 (ranks 1,2,4,8).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -x -q -k "sampled or frame_loop or plan or two_ranks" 2>&1 | tail -2
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,2,4,8 --steps 3 --reps 3 > gpurun_out/emul_px_$W.jsonl 2>&1; grep '^{"P"' gpurun_out/emul_px_$W.jsonl
done

# Late PDL trigger for device-list calls: tests touching dtiles/plan/bench, A/B timing, emulated scaling.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py tests/test_gpu_multigpu.py -x -q -k "dtiles or sampled or frame_loop or plan or two_ranks or deal or tiles" 2>&1 | tail -2
timeout 1500 python tools/ab_variants.py run --workloads C3,C5,C3r8d,C4r8d --rounds 3 --reps 5 base > gpurun_out/ab_late_rt.jsonl 2>&1; tail -5 gpurun_out/ab_late_rt.jsonl
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,2,4,8 --steps 3 --reps 3 > gpurun_out/emul_late_$W.jsonl 2>&1; grep '^{"P"' gpurun_out/emul_late_$W.jsonl
done

# Round evidence: bench line, ncu launch list of the bench command, ncu --set full of one step.
set -x
TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; cat gpurun_out/bench_${TAG}.json; tail -2 gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu_${TAG}.log 2>&1; tail -1 gpurun_out/bench_under_ncu_${TAG}.log | cut -c1-200
KPS=$(python -c "import paper_2206_02255_b200 as m, workloads as W; w=W.CONFIGS['C3']; print(m.kernel_count(w.n,w.g,w.r,w.B,'b200'))")
NM=$((KPS-1))
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_b200|k_fill|k_exhaustive" \
  -s $NM -c $((NM+1)) -o gpurun_out/prof_${TAG}_final_C3 -f python tools/prof_step.py --workload C3 --warm 1 > gpurun_out/ncu_final_${TAG}.log 2>&1; tail -2 gpurun_out/ncu_final_${TAG}.log

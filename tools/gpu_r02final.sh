# Closing evidence of round 2 (final kernels): bench lines C3 (default), C5, C4; ncu launch list
# of the bench command; ncu --set full of one C3 step + Ex (tools/gpu_prof.sh); GPU tests; smoke.
mkdir -p gpurun_out
TAG=${TAG:-r02l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench_C3_${TAG}.json 2> gpurun_out/bench_C3_${TAG}.err; echo "bench C3 rc=$?"
for W in C5 C4; do
  timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_${W}_${TAG}.json 2> gpurun_out/bench_${W}_${TAG}.err; echo "bench $W rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_C3_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu bench rc=$?"
TAG=$TAG W=C3 S=b200 bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1; echo "prof rc=$?"

#!/bin/bash
# evidence refresh with the current kernels: C4/C5 bench lines, schemes vs Ex, ncu launch list of
# the bench command + --set full of one C3 step + Ex, emulated scaling
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for W in C5 C4; do
  timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench $W rc=$?"
done
timeout 1500 python tools/ab.py C1 C3 C5 --ex --variants b200,sbr,mbr,dp > gpurun_out/ab_schemes.jsonl 2>&1; echo "ab rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_C3_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu bench rc=$?"
bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1; echo "prof rc=$?"
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,2,4,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '^{"P": 8' gpurun_out/emul_$W.jsonl
done
timeout 1200 python tools/sweep_c2.py --out gpurun_out/sweep_c2.json > gpurun_out/sweep_c2.log 2>&1; echo "sweep rc=$?"; tail -2 gpurun_out/sweep_c2.log

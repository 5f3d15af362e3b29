#!/bin/bash
# round-2 results table: bench lines at C4 and C5, schemes (b200/sbr/mbr/dp) with Ex at C1/C3/C5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for W in C5 C4; do
  timeout 1200 python bench.py --workload $W --steps 10 --warmup 3 > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "bench $W rc=$?"; head -c 300 gpurun_out/bench_$W.json; echo
done
timeout 1500 python tools/ab.py C1 C3 C5 --ex --variants b200,sbr,mbr,dp > gpurun_out/ab_schemes.jsonl 2>&1; echo "ab rc=$?"; cut -c1-400 gpurun_out/ab_schemes.jsonl
timeout 1200 python tools/sweep_c2.py --out gpurun_out/sweep_c2.json > gpurun_out/sweep_c2.log 2>&1; echo "sweep rc=$?"; tail -5 gpurun_out/sweep_c2.log

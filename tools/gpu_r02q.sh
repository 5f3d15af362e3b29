#!/bin/bash
# closing evidence of the 6-instruction step: ncu launch list of the bench command, full capture
# of one C3 step + Ex, emulated 8-way scaling, 3-D suite + bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_bench_C3_r02q.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu bench rc=$?"
TAG=r02q bash tools/gpu_prof.sh > gpurun_out/prof.log 2>&1; echo "prof rc=$?"
for W in C3 C5 C4; do
  timeout 900 python tools/emulate_scaling.py $W --ranks 1,2,4,8 --steps 3 --reps 3 > gpurun_out/emul_$W.jsonl 2>&1; grep '"P"' gpurun_out/emul_$W.jsonl
done
bash tools/gpu_3d.sh

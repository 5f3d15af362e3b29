# Dependent-latency micro-benchmark + per-level profile of the full image and of the
# heaviest 8-way rank at C3 and C4 (where the rank's time over 1/8 of the step goes).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/chain_lat tools/micro/chain_lat.cu && /tmp/chain_lat | tee gpurun_out/chain_lat.jsonl
timeout 600 python tools/rank_profile.py C3 --P 8 > gpurun_out/rank_profile_C3.txt 2>&1; echo "rp C3 rc=$?"
timeout 600 python tools/rank_profile.py C4 --P 8 > gpurun_out/rank_profile_C4.txt 2>&1; echo "rp C4 rc=$?"
timeout 600 python tools/level_profile.py C3 C4 --tiles-of 8 > gpurun_out/level_profile_rank8.jsonl 2>&1; echo "lp rc=$?"

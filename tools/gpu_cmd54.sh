set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench54_c4.json 2> gpurun_out/bench54_c4.err; cut -c1-400 gpurun_out/bench54_c4.json; tail -2 gpurun_out/bench54_c4.err
timeout 900 python bench.py --workload C5 --steps 10 --warmup 3 > gpurun_out/bench54_c5.json 2> gpurun_out/bench54_c5.err; cut -c1-400 gpurun_out/bench54_c5.json; tail -2 gpurun_out/bench54_c5.err

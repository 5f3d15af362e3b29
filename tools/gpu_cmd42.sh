set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 180 python -m pytest tests -m gpu -x -q -k "flow" > gpurun_out/pytest42.log 2>&1; tail -3 gpurun_out/pytest42.log
timeout 180 python -m pytest tests -m gpu -x -q -k "flow_full_size" > gpurun_out/pytest42b.log 2>&1; tail -1 gpurun_out/pytest42b.log
timeout 180 python tools/ab.py C3 C5 --variants b200,flow --reps 3 > gpurun_out/ab42.jsonl 2>&1; cut -c1-900 gpurun_out/ab42.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k "regex:k_flow$|k_flow<" -s 1 -c 1 -o gpurun_out/flow42 -f python tools/prof_step.py --workload C3 --scheme flow --warm 1 --no-ex > gpurun_out/ncu42.log 2>&1; tail -1 gpurun_out/ncu42.log

set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "flow and not full_size" > gpurun_out/pytest37.log 2>&1; tail -3 gpurun_out/pytest37.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_flow$|k_flow<" -s 1 -c 1 -o gpurun_out/flow37 -f python tools/prof_step.py --workload C3 --scheme flow --warm 1 --no-ex > gpurun_out/ncu37.log 2>&1; tail -3 gpurun_out/ncu37.log

set -x
TAG=r01rf2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200|k_fill" \
  -s 22 -c 22 -o gpurun_out/prof_${TAG}_C3 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex > gpurun_out/ncu7.log 2>&1
timeout 900 python tools/emulate_scaling.py C3 > gpurun_out/emul7.jsonl 2>&1; cat gpurun_out/emul7.jsonl

# ncu full capture of the lane-refill leaf kernel and the last border level (C3, one step)
set -x
TAG=${TAG:-r01rf}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200_leaf_rf|k_b200_border_rf" \
  -s 8 -c 8 -o gpurun_out/prof_${TAG}_C3 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex
ls -la gpurun_out | tail -3

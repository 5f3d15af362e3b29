# ncu --set full with source correlation of the lane-refill kernels of one C3 step (border levels
# + leaf), and of the heaviest rank of an 8-way deal; reports land in gpurun_out/.
set -x
TAG=${TAG:-r02src}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200_leaf_rf|k_b200_border_rf" \
  -s 8 -c 8 -o gpurun_out/prof_${TAG}_C3 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200_leaf_rf|k_b200_border_rf|k_b200_classify" \
  -s 22 -c 22 -o gpurun_out/prof_${TAG}_C3_rank8 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex --heavy-rank-of 8
ls -la gpurun_out | tail -4

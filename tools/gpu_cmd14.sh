set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
# kernels of the profiled (last) step only: the preview/cost passes and the warm step come first
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200_border_rf|k_b200_leaf_rf|k_b200_classify" \
  -s 30 -c 200 -o gpurun_out/prof_r01_rank8 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex --heavy-rank-of 8 > gpurun_out/ncu14.log 2>&1
tail -3 gpurun_out/ncu14.log

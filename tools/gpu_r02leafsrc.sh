# ncu --set full with source correlation of the C3 leaf kernel (one launch, after one warm step).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_b200_leaf_rf" \
  -s 1 -c 1 -o gpurun_out/prof_leafsrc_C3 -f python tools/prof_step.py --workload C3 --warm 1 --no-ex > gpurun_out/ncu_leafsrc.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_leafsrc.log

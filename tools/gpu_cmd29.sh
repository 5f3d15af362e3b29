set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for S in sbr mbr b200; do timeout 1200 python tools/sweep_c2.py --scheme $S --out gpurun_out/sweep_c2_$S.json > gpurun_out/sweep_c2_$S.log 2>&1; tail -4 gpurun_out/sweep_c2_$S.log | cut -c1-400; done

#!/bin/bash
# dwell census (C3, C5, C4) + ncu source-level capture of the refill kernels of one C3 step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python tools/dwell_census.py C3 C5 C4 > gpurun_out/dwell_census.jsonl 2> gpurun_out/census.err; echo "census rc=$?"; tail -2 gpurun_out/census.err
TAG=r02e bash tools/gpu_prof_src.sh > gpurun_out/prof.log 2>&1; echo "prof rc=$?"; tail -3 gpurun_out/prof.log

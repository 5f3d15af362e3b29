#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python tools/groups_rank.py C3 C4 > gpurun_out/groups_rank.jsonl 2>&1; cat gpurun_out/groups_rank.jsonl
bash tools/gpu_multirank.sh 2>&1 | grep -o 'rc=[0-9]*\|"value": [0-9.]*\|"bit_exact_vs_1gpu_ask": [a-z]*' | paste - - - 
TAG=r02l bash tools/gpu_prof_src.sh > gpurun_out/prof.log 2>&1; echo "prof rc=$?"

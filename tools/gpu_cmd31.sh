set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/level_profile.py C3 C5 C4 > gpurun_out/level31.jsonl 2>&1; cat gpurun_out/level31.jsonl
timeout 600 python tools/level_profile.py C3 --tiles-of 8 > gpurun_out/level31_p8.jsonl 2>&1; cat gpurun_out/level31_p8.jsonl

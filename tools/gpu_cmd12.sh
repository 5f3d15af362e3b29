set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build12.log 2>&1
timeout 600 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof12.jsonl 2>&1; cat gpurun_out/rankprof12.jsonl
timeout 600 python tools/rank_profile.py C3 --P 2 > gpurun_out/rankprof12_p2.jsonl 2>&1; head -1 gpurun_out/rankprof12_p2.jsonl

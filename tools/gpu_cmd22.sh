set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest22.log 2>&1; tail -2 gpurun_out/pytest22.log
timeout 300 python tools/ab.py C3 C5 --variants b200,g2 > gpurun_out/ab22.jsonl 2>&1; cut -c1-330 gpurun_out/ab22.jsonl
timeout 300 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof22.jsonl 2>&1; head -1 gpurun_out/rankprof22.jsonl

set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest21.log 2>&1; tail -2 gpurun_out/pytest21.log
timeout 300 python tools/trace_refill.py C3 --P 8 > gpurun_out/trace21.jsonl 2>&1; cat gpurun_out/trace21.jsonl
timeout 300 python tools/rank_profile.py C3 --P 8 > gpurun_out/rankprof21.jsonl 2>&1; head -1 gpurun_out/rankprof21.jsonl
timeout 300 python tools/ab.py C3 C5 --variants b200 > gpurun_out/ab21.jsonl 2>&1; cut -c1-330 gpurun_out/ab21.jsonl
timeout 600 python tools/tune_refill.py C3 C5 --points "RF_MIGRATE=4;RF_MIGRATE=16;RF_MIGRATE=0" > gpurun_out/tune21.txt 2>&1
cat gpurun_out/tune21.txt | cut -c1-400

set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "dp" > gpurun_out/pytest30.log 2>&1; tail -15 gpurun_out/pytest30.log
timeout 900 python tools/ab.py C1 C3 C5 --variants b200,sbr,mbr,dp --reps 5 --ex > gpurun_out/ab30.jsonl 2>&1; cut -c1-1500 gpurun_out/ab30.jsonl

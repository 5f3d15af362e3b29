set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest28.log 2>&1; tail -3 gpurun_out/pytest28.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python tools/ab.py C3 C5 --variants b200,sbr,mbr --reps 5 --ex > gpurun_out/ab28.jsonl 2>&1; cut -c1-900 gpurun_out/ab28.jsonl

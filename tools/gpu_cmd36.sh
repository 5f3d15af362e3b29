set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "flow and not full_size" > gpurun_out/pytest36.log 2>&1; tail -3 gpurun_out/pytest36.log
timeout 300 python tools/ab.py C3 --variants b200,flow --reps 3 > gpurun_out/ab36.jsonl 2>&1; cut -c1-900 gpurun_out/ab36.jsonl

set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest48.log 2>&1; tail -2 gpurun_out/pytest48.log
timeout 300 python tools/ab.py C3 C5 --variants b200 --reps 5 > gpurun_out/ab48.jsonl 2>&1; cut -c1-500 gpurun_out/ab48.jsonl
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,2,4,8 --deals costrank > gpurun_out/emu48.jsonl 2>&1; grep '"deal"' gpurun_out/emu48.jsonl | cut -c1-200
timeout 300 python tools/level_profile.py C3 --tiles-of 8 | python -c "import json,sys; r=json.loads(sys.stdin.read()); print([ (l['level'], l['border_ms']) for l in r['levels']], r['leaf_ms'])"

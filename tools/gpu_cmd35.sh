set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "flow" > gpurun_out/pytest35.log 2>&1; tail -3 gpurun_out/pytest35.log
timeout 600 python tools/ab.py C3 C5 --variants b200,flow --reps 5 > gpurun_out/ab35.jsonl 2>&1; cut -c1-900 gpurun_out/ab35.jsonl
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,2,4,8 --deals costrank > gpurun_out/emu35_b200.jsonl 2>&1; grep '"deal"' gpurun_out/emu35_b200.jsonl | cut -c1-300
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,2,4,8 --deals costrank --scheme flow > gpurun_out/emu35_flow.jsonl 2>&1; grep "\"deal\"" gpurun_out/emu35_flow.jsonl | cut -c1-300

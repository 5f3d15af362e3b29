set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,2,4,8 --deals costrank --scheme flow > gpurun_out/emu43_flow.jsonl 2>&1; grep '"deal"' gpurun_out/emu43_flow.jsonl | cut -c1-300

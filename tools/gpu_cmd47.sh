set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest47.log 2>&1; tail -2 gpurun_out/pytest47.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/bench47.json 2> gpurun_out/bench47.err; cat gpurun_out/bench47.json; tail -2 gpurun_out/bench47.err
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,2,4,8 --deals costrank > gpurun_out/emu47.jsonl 2>&1; grep '"deal"' gpurun_out/emu47.jsonl | cut -c1-200

# Parity subset + A/B timing + emulated 8-way after a kernel change.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "ask_c1 or random_small or edge or tiles_subset or full_size_ask or defer_random_small" > gpurun_out/pytest_quick.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_quick.log
timeout 600 python tools/ab.py C3 C5 --reps 5 --variants b200 > gpurun_out/ab_quick.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/ab_quick.jsonl'):
    d=json.loads(l); print(d['w'], d['b200']['ms_mean'], d['b200']['kernels'])"
timeout 600 python tools/emulate_scaling.py C3 --ranks 1,8 --deals lpt --reps 3 2>&1 | grep '"deal"' | cut -c1-140

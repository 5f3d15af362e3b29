set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "to_host" > gpurun_out/pytest50.log 2>&1; tail -2 gpurun_out/pytest50.log
timeout 900 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench50.json 2> gpurun_out/bench50.err; python -c "
import json; d=json.load(open('gpurun_out/bench50.json')); print(d['ms_per_step'], d['e2e'])"; tail -2 gpurun_out/bench50.err

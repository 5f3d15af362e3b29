#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 2400 python tools/ab_variants.py run base prev precount l16c2 l32c2 l32c2pc l32c4 --workloads C3,C5,C4,C3r8 --rounds 3 --reps 5 --check > gpurun_out/ab_m.jsonl 2>&1; grep -A5 summary gpurun_out/ab_m.jsonl | tail -5; grep -o '"variant": "[a-z0-9]*", "w": "C[0-9]", [^}]*tiles_differing_from_oracle": [0-9]*' gpurun_out/ab_m.jsonl | grep -o '"variant": "[a-z0-9]*", "w": "C[0-9]"\|differing_from_oracle": [0-9]*' | paste - - | sort -u

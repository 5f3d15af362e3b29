# Deal / preview-estimator study for the emulated 8-way split (C5 seahorse, C3).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for P in "16,8" "8,4" "16,2" "8,2" "8,1" "4,2"; do
  timeout 300 python tools/emulate_scaling.py C5 --ranks 8 --deals costrank,lpt --preview $P > gpurun_out/deals_C5_$P.jsonl 2>&1
done
timeout 300 python tools/emulate_scaling.py C5 --ranks 8 --deals costrank_exact,lpt_exact > gpurun_out/deals_C5_exact.jsonl 2>&1
for P in "16,8" "8,2"; do
  timeout 300 python tools/emulate_scaling.py C3 --ranks 8 --deals costrank,lpt,lpt_exact --preview $P > gpurun_out/deals_C3_$P.jsonl 2>&1
done
for f in gpurun_out/deals_*.jsonl; do echo $f; grep '"deal"' $f | cut -c1-200; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('preview_ms', d.get('preview_ms'), 't1', d.get('t1_ms'))"; done

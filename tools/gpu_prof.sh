# ncu evidence for one bench step (launch list + full capture), run under gpurun.
set -x
W=${W:-C3}; S=${S:-b200}; TAG=${TAG:-r01}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
KPS=$(python -c "import paper_2206_02255_b200 as m, workloads as W; w=W.CONFIGS['$W']; print(m.kernel_count(w.n,w.g,w.r,w.B,'$S'))")
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s $KPS -c $((KPS+1)) --csv \
  --log-file gpurun_out/launches_${TAG}_${W}_${S}.csv python tools/prof_step.py --workload $W --scheme $S --warm 1
NM=$((KPS-1))
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_b200|k_sbr|k_fill|k_exhaustive" \
  -s $NM -c $((NM+1)) -o gpurun_out/prof_${TAG}_${W}_${S} -f python tools/prof_step.py --workload $W --scheme $S --warm 1
ls -la gpurun_out

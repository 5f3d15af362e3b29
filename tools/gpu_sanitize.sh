# compute-sanitizer over tools/sanitize_driver.py: one log per tool under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitizer_$T.txt 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitizer_$T.txt
done

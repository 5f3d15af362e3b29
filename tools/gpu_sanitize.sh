# compute-sanitizer over tools/sanitize_driver.py: one log per tool under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
# Dynamic Parallelism (libmandel_dp.so) is supported by memcheck only: the other tools run
# the driver without it (SANITIZE_NO_DP=1).
for T in memcheck racecheck synccheck initcheck; do
  NODP=1; [ $T = memcheck ] && NODP=
  SANITIZE_NO_DP=$NODP timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_driver.py > gpurun_out/sanitizer_$T.txt 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitizer_$T.txt
done

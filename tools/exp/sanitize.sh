# compute-sanitizer over tools/sanitize_workload.py (memcheck, racecheck, synccheck, initcheck)
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"
  timeout 900 compute-sanitizer --tool $t --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py > gpurun_out/san_$t.log 2>&1
  echo "rc=$?"; tail -4 gpurun_out/san_$t.log
done

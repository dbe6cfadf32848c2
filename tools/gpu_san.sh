# compute-sanitizer over every entry point: full logs in gpurun_out/san_<tool>_<set>.log
for t in memcheck racecheck synccheck initcheck; do
  for w in tc ffma ext; do
    timeout 900 compute-sanitizer --tool $t --print-limit 200 python tools/sanitize_run.py $w > gpurun_out/san_${t}_${w}.log 2>&1
    echo "$t $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${t}_${w}.log | tail -1)"
  done
done

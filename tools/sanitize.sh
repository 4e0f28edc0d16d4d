# compute-sanitizer over the C1 (and C4) sanitize workload; logs summarised into gpurun_out/
O=gpurun_out; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for cl in 0 1; do
    for ln in 12 13; do
      CKKS_KS_CLUSTER=$cl LOGN=$ln timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_c1.py > $O/san_${tool}_n${ln}_c${cl}.log 2>&1
      echo "$tool logN=$ln cluster=$cl rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload ok' $O/san_${tool}_n${ln}_c${cl}.log | tr '\n' ' ')"
    done
  done
done

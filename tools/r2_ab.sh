# A/B timing of C3 / 2^15 / C4-batched ops: bash tools/r2_ab.sh "ENV1" "ENV2" ...
O=gpurun_out; mkdir -p $O
for e in "$@"; do
  echo "== $e"
  for cfg in "16 30 10 1" "15 16 10 1" "14 8 10 1" "13 5 10 51" "12 3 10 170" "16 30 10 1 10 7"; do
    env $e timeout 120 python tools/time_ops.py $cfg 2>&1 | grep -v "two calls"
  done
done

#!/bin/bash
# One profiling pass on the GPU box: launch list of the bench command (ncu, serialised,
# cold-cache) and --set full captures of the top PrivFT kernels.  Usage: TAG=r1_v7 bash tools/prof_round.sh
TAG=${TAG:-r1}
O=gpurun_out
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $O/launches_bench_$TAG.log 2>&1
for k in k_ks_mac k_fwd_cols k_fwd_rows_submul k_inv_rows k_inv_cols; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 3 -f -o $O/prof_${TAG}_$k \
      python tools/prof_privft.py 32 1 > $O/prof_${TAG}_$k.log 2>&1
done
ls -la $O

#!/bin/bash
# One profiling pass on the GPU box: launch list of the bench command (ncu, serialised,
# cold-cache) and --set full captures of the top PrivFT kernels, summarised ON THE BOX
# (gpurun copies back <= 64 MiB).  Usage: TAG=r1_v7 KERNELS="k_ks_mac k_fwd_cols" [PROG="python tools/time_ops.py 16 30 2 1"]
#   [NO_LAUNCHES=1] [SKIP=40] [COUNT=3] bash tools/prof_round.sh
TAG=${TAG:-r1}
O=gpurun_out
mkdir -p $O/summ_$TAG
if [ -z "$NO_LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu > $O/launches_bench_$TAG.log 2>&1
python tools/make_profiles.py $O/summ_$TAG $O/launches_$TAG.csv launches_$TAG.txt
fi
for k in ${KERNELS:-k_ks_mac k_fwd_cols k_fwd_rows_submul k_inv_rows k_inv_cols}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-40} -c ${COUNT:-3} -f -o /tmp/prof_${TAG}_$k \
      ${PROG:-python tools/prof_privft.py 32 1} > $O/prof_${TAG}_$k.log 2>&1
  python tools/make_profiles.py $O/summ_$TAG /tmp/prof_${TAG}_$k.ncu-rep ncu_${TAG}_$k.txt
  ncu -i /tmp/prof_${TAG}_$k.ncu-rep --page source --csv --print-source sass > /tmp/src_$k.csv 2>/dev/null && gzip -c /tmp/src_$k.csv > $O/summ_$TAG/src_$k.csv.gz
done
ls -la $O $O/summ_$TAG

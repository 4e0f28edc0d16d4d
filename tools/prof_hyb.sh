#!/bin/bash
# ncu --set full of every kernel of one C3 HMult+relin+rescale (hybrid alpha=10, K=10 x 40-bit, and
# alpha=1), summarised on the box.  TAG=r2_c bash tools/prof_hyb.sh
TAG=${TAG:-r2}
O=gpurun_out; mkdir -p $O/summ_$TAG
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "mul_relin_rescale/" -c 40 -f \
    -o /tmp/hyb_$TAG python tools/one_op.py 16 30 hmult 1 1 10 10 40 > $O/prof_hyb_$TAG.log 2>&1
python tools/make_profiles.py $O/summ_$TAG /tmp/hyb_$TAG.ncu-rep ncu_${TAG}_c3_hybrid.txt
ncu -i /tmp/hyb_$TAG.ncu-rep --page raw --csv > $O/summ_$TAG/raw_c3_hybrid.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "mul_relin_rescale/" -c 40 -f \
    -o /tmp/a1_$TAG python tools/one_op.py 16 30 hmult 1 1 > $O/prof_a1_$TAG.log 2>&1
python tools/make_profiles.py $O/summ_$TAG /tmp/a1_$TAG.ncu-rep ncu_${TAG}_c3_alpha1.txt
ncu -i /tmp/a1_$TAG.ncu-rep --page raw --csv > $O/summ_$TAG/raw_c3_alpha1.csv 2>/dev/null
ls -la $O/summ_$TAG

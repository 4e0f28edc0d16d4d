#!/bin/bash
# Full round check on one GPU box: parity suite, smoke, the bench line, the launch list of the
# bench command and --set full captures of the top kernels.  Usage: TAG=r2_b bash tools/round_check.sh
TAG=${TAG:-r2}
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; tail -3 $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke_$TAG.log 2>&1; tail -1 $O/smoke_$TAG.log
timeout 900 python bench.py > $O/bench_$TAG.json 2> $O/bench_$TAG.err; tail -c 600 $O/bench_$TAG.json; tail -3 $O/bench_$TAG.err
KERNELS=${KERNELS:-"k_ks_mac k_inv_cols_modup"} TAG=$TAG bash tools/prof_round.sh > $O/prof_$TAG.log 2>&1
PROG="python tools/time_ops.py 16 30 3 1" NO_LAUNCHES=1 SKIP=${C3SKIP:-60} COUNT=2 KERNELS=${C3KERNELS:-"k_ks_mac k_fwd_cols_r16"} TAG=${TAG}_c3 bash tools/prof_round.sh >> $O/prof_$TAG.log 2>&1
echo done

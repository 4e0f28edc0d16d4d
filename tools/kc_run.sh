O=gpurun_out; mkdir -p $O
timeout 120 python -m pytest tests/test_gpu_fullsize.py -x -q -k "n15 or c3_hmult" > $O/kc_t1.log 2>&1; echo "t1 rc=$?" >> $O/kc_t1.log; tail -15 $O/kc_t1.log
timeout 600 python -m pytest tests -m gpu -q -x > $O/kc_t2.log 2>&1; echo "t2 rc=$?" >> $O/kc_t2.log; tail -25 $O/kc_t2.log
for e in CKKS_KS_CLUSTER=0 CKKS_KS_CLUSTER=1; do
  echo "== $e"
  for cfg in "16 30 10 1" "15 16 10 1" "14 8 10 1" "13 5 10 1" "13 5 10 51" "12 3 10 1"; do
    env $e timeout 120 python tools/time_ops.py $cfg 2>&1 | head -3
  done
  env $e timeout 300 python bench.py --no-e2e --no-hmult --no-cpu --no-sweep --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('privft', round(d['ms_per_step'],1), 'ms/step', round(d['value'],2), 'inf/s', {k: round(v['share'],3) for k,v in d['kernels'].items() if v['share']>0.02})"
done

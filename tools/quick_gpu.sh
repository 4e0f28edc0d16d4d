#!/bin/bash
# Quick GPU check: parity suite + PrivFT step time + C3 HMult (extra env via ENVS="A=1 B=2").
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for e in ${ENVS:-X=0}; do
  echo "== $e"
  env $e timeout 300 python bench.py --no-e2e --no-hmult --no-cpu --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('privft', round(d['ms_per_step'],1), 'ms/step', round(d['value'],2), 'inf/s', 'frac', round(d['roofline']['frac'],3), {k: round(v['share'],3) for k,v in d['kernels'].items() if v['share']>0.02})"
  env $e timeout 300 python tools/time_ops.py 16 30 10 1 2>&1 | head -3
done

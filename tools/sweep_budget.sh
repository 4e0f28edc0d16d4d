#!/bin/bash
# Key-switch chunk budget sweep: PrivFT C4 step time and C3 HMult latency per CKKS_KS_BUDGET_MB.
for b in ${BUDGETS:-1024 512 256 128 64 32}; do
  echo "== budget $b MB"
  CKKS_KS_BUDGET_MB=$b timeout 300 python bench.py --no-e2e --no-hmult --no-cpu --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('privft', round(d['ms_per_step'],1), 'ms/step', {k: round(v['share'],3) for k,v in d['kernels'].items() if v['share']>0.02})"
  CKKS_KS_BUDGET_MB=$b timeout 300 python tools/time_ops.py 16 30 10 1 | head -2
done

#!/bin/bash
# A/B timing of library variants in one GPU session: VARIANTS="base nolazy" bash tools/ab.sh
export CKKS_NO_BUILD=1  # time the shipped builds as they are (no rebuild on the box)
for r in 1 2; do
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then unset CKKS_LIB_VARIANT; else export CKKS_LIB_VARIANT=$v; fi
  echo "== $v (round $r)"
  timeout 300 python bench.py --no-e2e --no-hmult --no-cpu --steps 3 --warmup 2 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('privft', round(d['ms_per_step'],1), 'ms/step', {k: round(v['share'],3) for k,v in d['kernels'].items() if v['share']>0.04})"
  timeout 300 python tools/time_ops.py 16 30 10 1 2>&1 | head -1
done; done
unset CKKS_LIB_VARIANT

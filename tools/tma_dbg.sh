#!/bin/bash
run() {
  env "$@" python bench.py --workload c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>&1 \
   | python -c "import json,sys
l=sys.stdin.read().strip().splitlines()
try:
  d=json.loads(l[-1]); print('$*', 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])
except Exception: print('$*', 'FAILED', l[-3:])"
}
for d in ${DBGS:-0 2 3}; do
  for v in ${VARIANTS:-0 5}; do
    run MMLTTB_TMA_VARIANT=$v MMLTTB_TMA_STAGES=${STAGES:-2} MMLTTB_TMA_DEBUG=$d
  done
done

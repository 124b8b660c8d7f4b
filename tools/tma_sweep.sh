#!/bin/bash
# TMA-fed fused kernel on C4 (4096 x 1e6 f32): variants x tile bytes x stages
run() {
  env "$@" python bench.py --workload c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>&1 \
   | python -c "import json,sys
l=sys.stdin.read().strip().splitlines()
try:
  d=json.loads(l[-1]); print('$*', 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])
except Exception: print('$*', 'FAILED', l[-3:])"
}
[ -n "$BASE" ] && run MMLTTB_TMA_VARIANT=-1
for v in ${VARIANTS:-0 1 2 3}; do
  for t in ${TILES:-16384 32768 65536}; do
    for s in ${STAGES:-2 3 4}; do
      run MMLTTB_TMA_VARIANT=$v MMLTTB_TMA_TILE=$t MMLTTB_TMA_STAGES=$s
    done
  done
done

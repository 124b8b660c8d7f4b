#!/bin/bash
# K1 load-variant sweep on the headline workload (stage timer, device events)
for v in ${VARIANTS:-0 1 2 3 4 5 6 7 8 9 10 11}; do
  MMLTTB_K1_VARIANT=$v python bench.py --steps 100 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('variant $v', 'k1_ms=%.4f'%d['stage_ms']['k1_extrema'], 'k2=%.4f'%d['stage_ms']['k2_compact'], 'k3=%.4f'%d['stage_ms']['k3_lttb'], 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"
done

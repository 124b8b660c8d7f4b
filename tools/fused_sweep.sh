#!/bin/bash
# fused per-series kernel variants on C4 (4096 x 1e6 f32)
for v in ${VARIANTS:-0 1 2 3 4 5 6 7 8}; do
  MMLTTB_FUSED_VARIANT=$v python bench.py --workload c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('variant $v', 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"
done
MMLTTB_NO_FUSED=1 python bench.py --workload c4 --steps 10 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('unfused', 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"

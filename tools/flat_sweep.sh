#!/bin/bash
# flat K1 split vs per-bucket chunks (MMLTTB_K1_FLAT_WARPS=0)
run() {
  python bench.py --workload $1 --steps 50 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', '$2', 'k1_ms=%.4f'%d['stage_ms']['k1_extrema'], 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"
}
for w in c3 c3_1e9 c5; do
  MMLTTB_K1_FLAT_WARPS=0 run $w chunked
  for fw in 3552 7104 10656 14208; do MMLTTB_K1_FLAT_WARPS=$fw run $w "flat=$fw"; done
done

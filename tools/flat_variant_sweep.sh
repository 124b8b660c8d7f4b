#!/bin/bash
# flat K1 template variants (U, load policy, CTAs/SM) x warp counts on C3 (1e8) and the 1e9 headline
run() {
  env "$@" python bench.py --workload $W --steps 50 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$W', '$*', 'k1_ms=%.4f'%d['stage_ms']['k1_extrema'])"
}
for W in ${WORKLOADS:-c3 c3_1e9}; do
  run MMLTTB_K1_FLAT_VARIANT=0
  run MMLTTB_K1_FLAT_VARIANT=1 MMLTTB_K1_FLAT_WARPS=4736
  run MMLTTB_K1_FLAT_VARIANT=2 MMLTTB_K1_FLAT_WARPS=4736
  run MMLTTB_K1_FLAT_VARIANT=3
  run MMLTTB_K1_FLAT_VARIANT=4 MMLTTB_K1_FLAT_WARPS=2368
  run MMLTTB_K1_FLAT_VARIANT=5 MMLTTB_K1_FLAT_WARPS=2368
done

for fw in 1184 1776 2368 2960 3552 4144; do
  MMLTTB_K1_FLAT_WARPS=$fw python bench.py --workload c3 --steps 100 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('flat=$fw', 'k1_ms=%.4f'%d['stage_ms']['k1_extrema'], 'step=%.4f'%d['ms_per_step'])"
done

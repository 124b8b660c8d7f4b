#!/bin/bash
# K1 chunk-planning sweep (env knobs read by capi.cu plan_extrema)
run() {
  python bench.py --workload $1 --steps 50 --warmup 3 --e2e-steps 0 --no-cpu --no-check 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', '$2', 'k1_ms=%.4f'%d['stage_ms']['k1_extrema'], 'k2=%.4f'%d['stage_ms']['k2_compact'], 'k3=%.4f'%d['stage_ms']['k3_lttb'], 'step=%.4f'%d['ms_per_step'], 'frac=%.3f'%d['roofline']['frac'])"
}
for w in c1 c4; do run $w default; done
for ww in 9472 18944 37888 75776 151552; do
  for mc in 1024 4096 8192; do
    MMLTTB_K1_WANT_WARPS=$ww MMLTTB_K1_MIN_CHUNK=$mc run c3 "want=$ww minchunk=$mc"
  done
done
for ww in 18944 75776; do MMLTTB_K1_WANT_WARPS=$ww run c3_1e9 "want=$ww"; done

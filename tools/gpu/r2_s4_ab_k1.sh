O=gpurun_out/s4
mkdir -p $O
: > $O/ab_k1.log
for i in 1 2 3; do
  for v in k1defer k1eager; do
    for w in c3 c3_1e9 c5; do
      MMLTTB_LIB=$PWD/_ab/lib_$v.so timeout 600 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v $w', round(d['ms_per_step']*1000,2), 'k1', round(d['roofline']['kernel_ms']*1000,2), d['details']['parity'][:5])
" >> $O/ab_k1.log
    done
  done
done

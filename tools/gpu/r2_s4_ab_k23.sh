O=gpurun_out/s4
mkdir -p $O
: > $O/ab_k23.log
for i in 1 2 3; do
  for v in lb32 lb64; do
    for w in c1 c3; do
      MMLTTB_LIB=$PWD/_ab/lib_$v.so timeout 600 python bench.py --workload $w --steps 300 --warmup 5 --no-cpu --graph 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v $w graph', round(d['ms_per_step']*1000,2), d['details']['parity'][:5])
" >> $O/ab_k23.log
    done
  done
done

for ch in 0 4096 8192 16384; do
  MMLTTB_K1_DYN_CHUNK=$ch timeout 600 python bench.py --workload c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/k1dyn_c3_$ch.log 2>&1
done
for ch in 8192 16384; do
  MMLTTB_K1_DYN_CHUNK=$ch timeout 600 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu > gpurun_out/k1dyn_c5_$ch.log 2>&1
  MMLTTB_K1_DYN_CHUNK=$ch timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/k1dyn_1e9_$ch.log 2>&1
done

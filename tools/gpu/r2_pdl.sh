for pdl in 1 0; do for w in c3 c1 c5; do
  MMLTTB_K23_PDL=$pdl timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/pdl${pdl}_$w.log 2>&1
done; done
timeout 600 python bench.py --workload c1 --steps 50 --warmup 5 --no-cpu --graph > gpurun_out/pdl1_c1g.log 2>&1
timeout 300 python tools/sanitize_cases.py post_smem c3_multi k1_flat > gpurun_out/pdl_cases.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_cases.log

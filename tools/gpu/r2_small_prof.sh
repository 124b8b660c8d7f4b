NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:"k_post_smem" -s 3 -c 1 -o gpurun_out/c1_post python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/c1_ncu.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:"k_compact_pairs|k_lttb_tables|k_lttb_scan|k_extrema_flat" -s 8 -c 4 -o gpurun_out/c3_k23 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/c3_ncu.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-check > gpurun_out/c3_launches.log 2>&1
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 6 -c 8 python bench.py --workload c1 --steps 3 --warmup 3 --no-cpu --no-check > gpurun_out/c1_launches.log 2>&1

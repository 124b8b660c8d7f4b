mkdir -p gpurun_out/s3e
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_extrema_tiles -s 6 -c 1 -o gpurun_out/s3e/tiles_c3 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/s3e/ncu.log 2>&1

mkdir -p gpurun_out/s3c
timeout 600 python -m pytest tests/test_gpu_k1_tiles.py -q -x -p no:randomly > gpurun_out/s3c/pytest_tiles.log 2>&1; echo "rc=$?" >> gpurun_out/s3c/pytest_tiles.log
for T in 1 0; do
for w in c3 c3_1e9 c5 c3r2 c3r8 c3r16; do
  MMLTTB_K1_TILES=$T timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/s3c/bench_${w}_T$T.log 2>&1
done; done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/s3c/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3c/pytest_gpu.log

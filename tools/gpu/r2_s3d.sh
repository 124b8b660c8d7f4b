mkdir -p gpurun_out/s3d
timeout 600 python -m pytest tests/test_gpu_k1_tiles.py -q -x -p no:randomly > gpurun_out/s3d/pytest_tiles.log 2>&1; echo "rc=$?" >> gpurun_out/s3d/pytest_tiles.log
for T in 1 0; do
for w in c3 c3_1e9; do
  MMLTTB_K1_TILES=$T timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/s3d/bench_${w}_T$T.log 2>&1
done; done

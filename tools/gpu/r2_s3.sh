python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s3_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/r2s3_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s3_pytest_gpu.log
timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu > gpurun_out/r2s3_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r2s3_bench_c2.log

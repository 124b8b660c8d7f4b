set -x
free -g > gpurun_out/r2_host.txt; nproc >> gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/r2_pytest_gpu_1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest_gpu_1.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_1.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2_bench_1.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_1.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2_ref_1.log

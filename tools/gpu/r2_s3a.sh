set -x
mkdir -p gpurun_out/s3a
nvidia-smi -L > gpurun_out/s3a/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s3a/smoke.log
CS=/usr/local/cuda/bin/compute-sanitizer
ls -la $CS > gpurun_out/s3a/sanitize_probe.log 2>&1
timeout 300 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py k23 >> gpurun_out/s3a/sanitize_probe.log 2>&1; echo "rc=$?" >> gpurun_out/s3a/sanitize_probe.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/s3a/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s3a/pytest_gpu.log
for w in c3_1e9 c1 c2 c3; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/s3a/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/s3a/bench_$w.log
done

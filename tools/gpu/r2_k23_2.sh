timeout 300 python tools/sanitize_cases.py post_smem c3_multi k1_flat shards > gpurun_out/k23b_cases.log 2>&1; echo "rc=$?" >> gpurun_out/k23b_cases.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -m gpu -x -q -p no:randomly > gpurun_out/k23b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k23b_pytest.log
for w in c1 c3 c3r32 c5; do timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/k23b_bench_$w.log 2>&1; done
MMLTTB_K3S_PROF=1 python tools/k23_prof.py > gpurun_out/k23_prof.log 2>&1

for c in post_smem c3_multi k1_flat k1_chunked shards p2p; do timeout 300 python tools/sanitize_cases.py $c >> gpurun_out/k23_cases.log 2>&1; echo "$c rc=$?" >> gpurun_out/k23_cases.log; done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/k23_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k23_pytest.log
for w in c1 c3 c3r32 c5; do timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/k23_bench_$w.log 2>&1; done

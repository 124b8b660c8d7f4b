MMLTTB_K3S_PROF=1 python tools/k23_prof.py > gpurun_out/bar_k23_prof.log 2>&1
MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 --prof > gpurun_out/bar_k3s_prof.log 2>&1
timeout 300 python tools/k3s_check.py c2 c2_f32y --time > gpurun_out/bar_k3s.log 2>&1
for w in c1 c3; do timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/bar_bench_$w.log 2>&1; done
timeout 600 python bench.py --workload c1 --steps 200 --warmup 5 --no-cpu --graph > gpurun_out/bar_bench_c1g.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:randomly -k "k3s or c1 or c3 or golden or fuzz" > gpurun_out/bar_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/bar_pytest.log

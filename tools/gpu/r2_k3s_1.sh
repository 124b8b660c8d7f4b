set -x
timeout 600 python tools/k3s_check.py --time > gpurun_out/k3s_check.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check.log
MMLTTB_K3S=0 timeout 600 python tools/k3s_check.py --time > gpurun_out/k3s_check_off.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check_off.log
for c in k3c_flat k3c_repair k3c_cert k3c_batch; do
  timeout 300 python tools/sanitize_cases.py $c >> gpurun_out/k3s_cases.log 2>&1; echo "$c rc=$?" >> gpurun_out/k3s_cases.log
done
timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu > gpurun_out/k3s_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_bench_c2.log

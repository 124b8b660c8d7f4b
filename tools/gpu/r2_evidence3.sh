set -x
mkdir -p gpurun_out/ev3
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev3/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/ev3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev3/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ev3/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/ev3/bench_default.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ev3/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/ev3/bench_reference.log
for w in c1 c2 c3 c3r2 c3r8 c3r16 c3r32 c4 c5 c5s; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/ev3/bench_$w.log 2>&1
done
timeout 600 python bench.py --workload c1 --steps 200 --warmup 5 --no-cpu --graph > gpurun_out/ev3/bench_c1g.log 2>&1
timeout 600 python bench.py --workload c3 --steps 200 --warmup 5 --no-cpu --graph > gpurun_out/ev3/bench_c3g.log 2>&1
timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 > gpurun_out/ev3/bench_c2_cpu.log 2>&1
NCU=/usr/local/cuda/bin/ncu
for w in c1 c2 c3 c5 c3_1e9; do
  timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" -s 4 -c 8 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu --no-check > gpurun_out/ev3/launches_$w.log 2>&1
done
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_lttb_k3s -s 3 -c 1 -o gpurun_out/ev3/c2_k3s_full python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/ev3/ncu_c2.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_k23 -s 3 -c 1 -o gpurun_out/ev3/c3_k23_full python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/ev3/ncu_c3.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_extrema_flat -s 3 -c 1 -o gpurun_out/ev3/c3_1e9_k1_full python bench.py --steps 2 --warmup 3 --no-cpu --no-check > gpurun_out/ev3/ncu_1e9.log 2>&1
# K3s shapes beyond C2 (tools/k3s_check.py): timing per call, all index-exact
timeout 900 python tools/k3s_check.py --time > gpurun_out/ev3/k3s_check.log 2>&1
MMLTTB_K3S_PRUNE=0 MMLTTB_K3S_JMAX=0 timeout 900 python tools/k3s_check.py --time > gpurun_out/ev3/k3s_check_noprune_nofix.log 2>&1

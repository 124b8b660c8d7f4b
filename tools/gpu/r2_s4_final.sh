O=gpurun_out/s4f
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_reference.log 2>&1
for w in c1 c2 c3; do timeout 900 python bench.py --workload $w --steps 100 --warmup 5 --no-cpu > $O/bench_$w.log 2>&1; done
timeout 900 python tools/k3s_check.py --time > $O/k3s_check.log 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^k_" -s 4 -c 8 python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu --no-check > $O/launches_c2.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_lttb_k3s -s 3 -c 1 -o $O/c2_k3s_full python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-check > $O/ncu_c2.log 2>&1

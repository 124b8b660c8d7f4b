set -x
O=gpurun_out/s4
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > $O/bench_$w.log 2>&1
done
timeout 600 python bench.py --workload c1 --steps 200 --warmup 5 --no-cpu --graph > $O/bench_c1g.log 2>&1
timeout 600 python bench.py --workload c3 --steps 200 --warmup 5 --no-cpu --graph > $O/bench_c3g.log 2>&1

set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2s2_smoke.log
for w in c1 c2 c3; do
  timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu > gpurun_out/r2s2_bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/r2s2_bench_$w.log
done
timeout 3000 tools/sanitize.sh > gpurun_out/r2s2_sanitize.log 2>&1

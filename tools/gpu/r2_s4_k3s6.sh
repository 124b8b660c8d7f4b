set -x
O=gpurun_out/s4
mkdir -p $O
MMLTTB_K3S_PROF=1 timeout 900 python tools/k3s_check.py --time --prof c2 smooth const > $O/k3s_j3.log 2>&1; echo "rc=$?" >> $O/k3s_j3.log
timeout 900 python tools/k3s_check.py --time > $O/k3s_j3_noprof.log 2>&1
MMLTTB_K3S_JMIN=0 MMLTTB_K3S_JMAX=2 timeout 900 python tools/k3s_check.py --time smooth const big_buckets huge_buckets steps > $O/k3s_j3_jmax2.log 2>&1
MMLTTB_K3S_JMIN=0 timeout 900 python tools/k3s_check.py --time smooth const big_buckets huge_buckets steps > $O/k3s_j3_jmin0.log 2>&1
timeout 600 python bench.py --workload c2 --steps 50 --warmup 5 --no-cpu > $O/bench_c2_v7.log 2>&1

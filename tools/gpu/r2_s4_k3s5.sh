set -x
O=gpurun_out/s4
mkdir -p $O
MMLTTB_K3S_PROF=1 timeout 900 python tools/k3s_check.py --time --prof c2 > $O/k3s_j2.log 2>&1; echo "rc=$?" >> $O/k3s_j2.log
timeout 900 python tools/k3s_check.py --time > $O/k3s_j2_noprof.log 2>&1
timeout 900 python tools/k3s_check.py --time c2 c2_f32y few_buckets neg_dx >> $O/k3s_j2_noprof.log 2>&1

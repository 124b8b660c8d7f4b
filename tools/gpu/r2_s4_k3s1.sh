set -x
O=gpurun_out/s4
mkdir -p $O
MMLTTB_K3S_PROF=1 timeout 900 python tools/k3s_check.py --time --prof > $O/k3s_prune.log 2>&1; echo "rc=$?" >> $O/k3s_prune.log
MMLTTB_K3S_PRUNE=0 timeout 900 python tools/k3s_check.py --time c2 big_buckets smooth > $O/k3s_noprune.log 2>&1
timeout 900 python tools/k3s_check.py --time c2 c2_f32y big_buckets smooth > $O/k3s_prune_noprof.log 2>&1

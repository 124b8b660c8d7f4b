set -x
O=gpurun_out/s4
mkdir -p $O
MMLTTB_K3S_PROF=1 timeout 900 python tools/k3s_check.py --time --prof c2 smooth const steps big_buckets > $O/k3s_j.log 2>&1; echo "rc=$?" >> $O/k3s_j.log
timeout 900 python tools/k3s_check.py --time > $O/k3s_j_noprof.log 2>&1
MMLTTB_K3S_JMIN=0 timeout 900 python tools/k3s_check.py --time > $O/k3s_j_jmin0.log 2>&1
MMLTTB_K3S_JMIN=0 MMLTTB_K3S_JMAX=2 timeout 900 python tools/k3s_check.py --time > $O/k3s_j_jmax2.log 2>&1

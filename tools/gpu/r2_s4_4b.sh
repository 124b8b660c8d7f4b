O=gpurun_out/s4
mkdir -p $O
: > $O/k3s_4b.log
run() { echo "== knobs: $*" >> $O/k3s_4b.log; env "$@" timeout 900 python tools/k3s_check.py --time c2 c2_f32y mid big_buckets big_buckets_f32 huge_buckets smooth ties const f64x_irregular steps neg_dx many_1500pt >> $O/k3s_4b.log 2>&1; echo "rc=$?" >> $O/k3s_4b.log; }
run X=1
run MMLTTB_K3S_JMAX=0
run MMLTTB_K3C_CAND_CAP=2 MMLTTB_K3S_JMAX=0
run MMLTTB_K3C_CAND_CAP=1 MMLTTB_K3S_JMIN=100000
run MMLTTB_K3C_CERT_FORCE=1 MMLTTB_K3S_JMAX=0

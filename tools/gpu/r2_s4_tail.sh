O=gpurun_out/s4
mkdir -p $O
MMLTTB_LIB=$PWD/_ab/lib_$1.so timeout 900 python tools/k3s_check.py > $O/k3s_tail_parity.log 2>&1; echo "rc=$?" >> $O/k3s_tail_parity.log
MMLTTB_K3C_CAND_CAP=2 MMLTTB_LIB=$PWD/_ab/lib_$1.so timeout 900 python tools/k3s_check.py c2 mid smooth ties const >> $O/k3s_tail_parity.log 2>&1; echo "rc=$?" >> $O/k3s_tail_parity.log
VARIANTS="$1 $2" CASES="c2 c2_f32y mid neg_dx few_buckets" bash tools/gpu/r2_s4_ab.sh

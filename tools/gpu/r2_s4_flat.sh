O=gpurun_out/s4
mkdir -p $O
# parity of every shape with the flat-split statistics, then A/B timing
MMLTTB_LIB=$PWD/_ab/lib_flat.so timeout 900 python tools/k3s_check.py > $O/k3s_flat_parity.log 2>&1; echo "rc=$?" >> $O/k3s_flat_parity.log
VARIANTS="flat preflat" CASES="c2 c2_f32y mid i32x few_buckets wide_1000 many_1500pt big_buckets neg_dx f64x_irregular" bash tools/gpu/r2_s4_ab.sh

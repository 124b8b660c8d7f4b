O=gpurun_out/s4
mkdir -p $O
: > $O/k3s_many.log
for k in 1 0; do
  echo "== MMLTTB_K3S=$k" >> $O/k3s_many.log
  MMLTTB_K3S=$k timeout 900 python tools/k3s_check.py --time many_100pt many_500pt many_1500pt wide_1000 mid few_buckets tiny_k3 wide_300 >> $O/k3s_many.log 2>&1
done

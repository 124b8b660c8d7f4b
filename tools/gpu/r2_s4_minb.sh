O=gpurun_out/s4
mkdir -p $O
: > $O/k3s_minb.log
for mb in 32 0; do
  echo "== MINB4=$mb" >> $O/k3s_minb.log
  MMLTTB_K3S_MINB4=$mb timeout 900 python tools/k3s_check.py --time wide_300 wide_1000 wide_100 wide_30 tiny_k3 few_buckets >> $O/k3s_minb.log 2>&1
done

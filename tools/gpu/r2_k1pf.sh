for v in "0 -1" "1 2368" "1 -1" "2 -1"; do set -- $v
  MMLTTB_K1_PF=$1 MMLTTB_K1_FLAT_WARPS=$2 timeout 600 python bench.py --workload c3 --steps 50 --warmup 5 --no-cpu > gpurun_out/k1pf_c3_$1_$2.log 2>&1
  MMLTTB_K1_PF=$1 MMLTTB_K1_FLAT_WARPS=$2 timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/k1pf_1e9_$1_$2.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/k1pf_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k1pf_pytest.log

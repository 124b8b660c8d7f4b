set -x
O=gpurun_out/s4
mkdir -p $O
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_lttb_k3s -s 3 -c 1 -o $O/c2_k3s_v6 python bench.py --workload c2 --steps 2 --warmup 3 --no-cpu --no-check > $O/ncu_c2_v6.log 2>&1

set -x
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:k_lttb_k3s -s 2 -c 1 -o gpurun_out/k3s_c2_full python tools/k3s_check.py c2 --time > gpurun_out/k3s_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_ncu.log
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 10 -c 6 python tools/k3s_check.py c2 few_buckets --time > gpurun_out/k3s_launches.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_launches.log

set -x
timeout 600 python tools/k3s_check.py --time > gpurun_out/k3s_check.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check.log
for c in k3c_flat k3c_repair k3c_cert k3c_batch; do
  timeout 300 python tools/sanitize_cases.py $c >> gpurun_out/k3s_cases.log 2>&1; echo "$c rc=$?" >> gpurun_out/k3s_cases.log
done
MMLTTB_K3C_CAND_CAP=1 timeout 300 python tools/k3s_check.py c2 mid ties --time > gpurun_out/k3s_check_cap1.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check_cap1.log
MMLTTB_K3C_CERT_FORCE=1 timeout 300 python tools/k3s_check.py mid ties --time > gpurun_out/k3s_check_cert.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check_cert.log
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_lttb_k3s -s 2 -c 1 -o gpurun_out/k3s_c2_full2 python tools/k3s_check.py c2 --time > gpurun_out/k3s_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_ncu.log

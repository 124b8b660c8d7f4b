MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof.log 2>&1
timeout 300 python tools/k3s_check.py --time > gpurun_out/k3s_t.log 2>&1
MMLTTB_K3C_CAND_CAP=1 timeout 300 python tools/k3s_check.py c2 ties --time > gpurun_out/k3s_check_cap1.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check_cap1.log
MMLTTB_K3C_CERT_FORCE=1 timeout 300 python tools/k3s_check.py c2 --time > gpurun_out/k3s_check_cert.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_check_cert.log

timeout 300 python tools/k3s_check.py --time > gpurun_out/ring_check.log 2>&1; echo "rc=$?" >> gpurun_out/ring_check.log
MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/ring_prof.log 2>&1
MMLTTB_K3C_CAND_CAP=1 timeout 300 python tools/k3s_check.py c2 --time > gpurun_out/ring_cap1.log 2>&1; echo "rc=$?" >> gpurun_out/ring_cap1.log

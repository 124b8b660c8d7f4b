MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_prof.log

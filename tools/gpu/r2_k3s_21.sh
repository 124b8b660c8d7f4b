MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_prof.log
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_d16.so MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof16.log 2>&1; echo "rc=$?" >> gpurun_out/k3s_prof16.log
timeout 300 python tools/k3s_check.py c2 c2_f32y --time > gpurun_out/k3s_t8.log 2>&1
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_d16.so timeout 300 python tools/k3s_check.py --time > gpurun_out/k3s_t16.log 2>&1

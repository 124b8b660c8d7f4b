for D in 12 16; do
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_d$D.so MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof$D.log 2>&1
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_d$D.so timeout 300 python tools/k3s_check.py c2 c2_f32y --time > gpurun_out/k3s_t$D.log 2>&1
done
timeout 300 python tools/k3s_check.py c2 c2_f32y --time > gpurun_out/k3s_t8.log 2>&1

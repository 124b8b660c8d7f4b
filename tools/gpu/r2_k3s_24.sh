for v in d8s1 d12s1 d6s1; do
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_$v.so MMLTTB_K3S_PROF=1 timeout 300 python tools/k3s_check.py c2 c2_f32y --prof > gpurun_out/k3s_prof_$v.log 2>&1
MMLTTB_LIB=paper_2305_00332_b200/libmmlttb_$v.so timeout 300 python tools/k3s_check.py c2 c2_f32y --time > gpurun_out/k3s_t_$v.log 2>&1
done

O=gpurun_out/s4
mkdir -p $O
MMLTTB_K3S_PROF=1 timeout 600 python tools/k3s_check.py --time --prof --ctas c2 > $O/k3s_ctas.log 2>&1
MMLTTB_K3S_PROF=1 timeout 600 python tools/k3s_check.py --time --prof --ctas c2 >> $O/k3s_ctas.log 2>&1

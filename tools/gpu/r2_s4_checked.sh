# range-checked K3s build (-DK3S_CHECKED: a violated index / vector range traps) over every k3s_check shape and knob
O=gpurun_out/s4
mkdir -p $O
export MMLTTB_LIB=$PWD/_ab/lib_checked.so
: > $O/k3s_checked.log
run() { echo "== knobs: $*" >> $O/k3s_checked.log; env "$@" timeout 900 python tools/k3s_check.py >> $O/k3s_checked.log 2>&1; echo "rc=$?" >> $O/k3s_checked.log; }
run X=1
run MMLTTB_K3C_CAND_CAP=1
run MMLTTB_K3C_CAND_CAP=2 MMLTTB_K3S_JMIN=0
run MMLTTB_K3C_CERT_FORCE=1
run MMLTTB_K3S_JMIN=0 MMLTTB_K3S_JMAX=2
run MMLTTB_K3S_JMAX=0

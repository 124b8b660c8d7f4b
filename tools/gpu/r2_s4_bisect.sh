O=gpurun_out/s4i
mkdir -p $O
: > $O/bisect.log
run() { echo "== $*" >> $O/bisect.log; env LTTB_FUZZ_ONLY=42 "$@" timeout 600 python tools/lttb_fuzz.py 43 2 2>&1 | tail -2 >> $O/bisect.log; }
run MMLTTB_K3C_CAND_CAP=3
run MMLTTB_K3C_CAND_CAP=3 MMLTTB_K3S_PRUNE=0
run MMLTTB_K3C_CAND_CAP=3 MMLTTB_K3S_JMAX=0
run MMLTTB_K3C_CAND_CAP=3 MMLTTB_K3S_JMAX=0 MMLTTB_K3S_PRUNE=0
run MMLTTB_K3C_CAND_CAP=3 MMLTTB_K3S=0
run MMLTTB_K3C_CAND_CAP=3 MMLTTB_K3S_JMIN=100000
run MMLTTB_K3C_CAND_CAP=2
run MMLTTB_K3C_CAND_CAP=4
run X=1

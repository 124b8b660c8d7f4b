O=gpurun_out/s4
mkdir -p $O
: > $O/ab.log
for i in 1 2 3; do
  for v in $VARIANTS; do
    echo "== $v" >> $O/ab.log
    MMLTTB_LIB=$PWD/_ab/lib_$v.so timeout 600 python tools/k3s_check.py --time $CASES 2>&1 | grep -v "ALL OK" >> $O/ab.log
  done
done

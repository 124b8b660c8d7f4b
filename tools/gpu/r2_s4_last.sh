O=gpurun_out/s4
mkdir -p $O
timeout 900 python tools/k3s_check.py --time > $O/k3s_last.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > $O/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu4.log

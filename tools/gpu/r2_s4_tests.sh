O=gpurun_out/s4
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -p no:randomly > $O/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu3.log

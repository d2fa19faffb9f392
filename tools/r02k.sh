set -u
O=gpurun_out/${TAG}; mkdir -p $O
timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools/epoch_timing')
import build_and_run as b
b.run('build/epoch_timing/libds2ctc_timing_base.so', brief=True)" > $O/epoch.txt 2>&1
TAG=$TAG VARIANTS="head headlayout cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -s > $O/pytest_parity.log 2>&1; echo PYTEST $? >> $O/pytest_parity.log

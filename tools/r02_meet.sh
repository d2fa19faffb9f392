# Meet logZ in one load pass + rank-swap timing experiment.
set -u
O=gpurun_out/${TAG:-r02meet}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
timeout 900 python tools/epoch_timing/build_and_run.py variants base SWAPRANK > $O/timing.txt 2>&1
TAG=$(basename $O)/ab WORKLOAD=english VARIANTS="prev cur" ROUNDS=3 bash tools/ab_bench.sh > /dev/null 2>&1
TAG=$(basename $O)/ab WORKLOAD=config1 VARIANTS="prev cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
TAG=$(basename $O)/ab WORKLOAD=sortagrad VARIANTS="prev cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1

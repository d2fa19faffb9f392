# 3-way A/B: prev (HEAD), meet (one-pass logZ), cur (+ drain rows over all warps); parity of cur.
set -u
O=gpurun_out/${TAG:-r02meet2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
TAG=$(basename $O)/ab WORKLOAD=english VARIANTS="prev meet cur" ROUNDS=3 bash tools/ab_bench.sh > /dev/null 2>&1
TAG=$(basename $O)/ab WORKLOAD=config1 VARIANTS="prev meet cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
TAG=$(basename $O)/ab WORKLOAD=mandarin VARIANTS="prev meet cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1

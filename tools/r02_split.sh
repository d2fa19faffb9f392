# Split path: occupancy rows written by the gradient warp (cur) vs the service warp (prev).
set -u
O=gpurun_out/${TAG:-r02split}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for w in mandarin english config1; do
  TAG=$(basename $O)/ab WORKLOAD=$w VARIANTS="prev cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
done

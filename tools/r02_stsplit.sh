# Split path: key-column staging shared by the service and gradient warps (cur) vs prev; then the 4-GPU Mandarin probe.
set -u
O=gpurun_out/${TAG:-r02stsplit}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for w in mandarin english; do
  TAG=$(basename $O)/ab WORKLOAD=$w VARIANTS="prev cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
done

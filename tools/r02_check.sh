#!/bin/bash
# Quick GPU check: gpu tests, parity probe, English + SortaGrad + Mandarin bench lines.
# usage: TAG=r02c bash tools/r02_check.sh
set -u
O=gpurun_out/${TAG:-r02c}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "PYTEST $?" >> $O/pytest_gpu.log
timeout 900 python tools/parity_probe.py --json $O/parity.json > $O/parity.log 2>&1; echo "PROBE $?" >> $O/parity.log
for w in english sortagrad mandarin; do
  timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/b_$w.json 2> $O/b_$w.err
done
echo done

set -u
O=gpurun_out/r02p; mkdir -p $O
for v in base; do
  timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools/epoch_timing')
import build_and_run as b
b.run('build/epoch_timing/libds2ctc_timing_$v.so', brief=False)" > $O/epoch_$v.txt 2>&1
done
TAG=r02p VARIANTS="head cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1

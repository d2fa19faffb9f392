set -u
O=gpurun_out/r02ep4; mkdir -p $O
for v in base noframemass_nonorm; do
  timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools/epoch_timing')
import build_and_run as b
b.run('build/epoch_timing/libds2ctc_timing_$v.so', 29, 1500, 300, 16, brief=False)" > $O/epoch_$v.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_cpp.py -m gpu -q -s > $O/cpp.log 2>&1; echo PYTEST $? >> $O/cpp.log

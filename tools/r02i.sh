set -u
O=gpurun_out/r02i; mkdir -p $O
for v in head base noframemass_nonorm_nopoison noframemass; do
  echo "== $v" >> $O/epoch.txt
  timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools/epoch_timing')
import build_and_run as b
b.run('build/epoch_timing/libds2ctc_timing_$v.so', brief=True)" 2>&1 | grep -E "cta" >> $O/epoch.txt
done

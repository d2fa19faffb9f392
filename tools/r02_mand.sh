# Mandarin overlap A/B: serial pass, overlap with co-resident dense blocks,
# overlap with the SM-exclusion request (default); parity of the split path.
set -u
O=gpurun_out/${TAG:-r02mand}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mandarin or split or nan or poison" > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for rep in 1 2; do
  DS2CTC_DENSE_OVERLAP=0 timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/serial_$rep.json 2> $O/serial_$rep.err
  DS2CTC_DENSE_EXCLUDE=0 timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/coresident_$rep.json 2> $O/coresident_$rep.err
  timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/exclude_$rep.json 2> $O/exclude_$rep.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mandarin.csv python bench.py --workload mandarin --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

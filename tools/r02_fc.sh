# FC backward check: fc tests, english-step bench, per-kernel launch list.
set -u
O=gpurun_out/${TAG:-r02fc}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for r in 1 2; do
  timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_$r.json 2> $O/step_$r.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fc|k_pad|k_transpose|k_bias" --csv --log-file $O/fc_launches.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

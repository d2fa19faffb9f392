# FC dx: epilogue staging aliased over the operand tiles (5 CTAs per SM) vs prev (4).
set -u
O=gpurun_out/${TAG:-r02fc4}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for r in 1 2; do
  for v in prev cur; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_LIB=$L timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_${v}_$r.json 2> $O/step_${v}_$r.err
    python -c "import json; d=json.load(open('$O/step_${v}_$r.json')); f=d['fc_backward']; print('$v', $r, round(d['value']), round(d['ms_per_step']*1e3,1), 'fc', round(f['ms']*1e3,1), round(f['achieved_gbs']))" >> $O/summary.txt
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fc" --csv --log-file $O/fc_launches.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

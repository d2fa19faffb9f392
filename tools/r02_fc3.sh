# FC dW: two 2-stage CTAs per SM vs one 4-stage CTA per SM.
set -u
O=gpurun_out/${TAG:-r02fc3}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
DS2CTC_FC_DW_STAGES=2 timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest_s2.log 2>&1; echo PYTEST $? >> $O/pytest_s2.log
for r in 1 2; do
  for st in 4 2; do
    DS2CTC_FC_DW_STAGES=$st timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_s${st}_$r.json 2> $O/step_s${st}_$r.err
    python -c "import json; d=json.load(open('$O/step_s${st}_$r.json')); f=d['fc_backward']; print('stages $st', $r, round(d['value']), round(d['ms_per_step']*1e3,1), 'fc', round(f['ms']*1e3,1), round(f['achieved_gbs']))" >> $O/summary.txt
  done
done
DS2CTC_FC_DW_STAGES=2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fc" --csv --log-file $O/fc_launches_s2.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

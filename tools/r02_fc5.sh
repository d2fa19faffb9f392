# FC dx: six CTAs per SM (<= 56 registers) vs five; traffic stamp of this build.
set -u
O=gpurun_out/${TAG:-r02fc5}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for r in 1 2; do
  for v in prev cur; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_LIB=$L timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_${v}_$r.json 2> $O/step_${v}_$r.err
    python -c "import json; d=json.load(open('$O/step_${v}_$r.json')); f=d['fc_backward']; print('$v', $r, round(d['value']), round(d['ms_per_step']*1e3,1), 'fc', round(f['ms']*1e3,1), round(f['achieved_gbs']))" >> $O/summary.txt
  done
done
timeout 900 python tools/ncu/traffic.py english:k_pair mandarin:k_dense_t english-step:k_pair > $O/traffic.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1

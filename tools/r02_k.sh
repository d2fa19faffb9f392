set -u
O=gpurun_out/${TAG}; mkdir -p $O
for r in 1 2; do
for w in english sortagrad; do
  for cfg in "cur 3" "cur 2" "halo6 3" "halo6 2"; do
    set -- $cfg; v=$1; mc=$2
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_MAX_CHAIN_WARPS=$mc DS2CTC_LIB=$L timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > $O/${w}_${v}_$mc.json 2> $O/${w}_${v}_$mc.err
    python -c "import json; d=json.load(open('$O/${w}_${v}_$mc.json')); print('$w $v maxwarps=$mc', round(d['value']), round(d['ms_per_step']*1000,1), 'us', 'k_pair', round(d['stage_ms']['k_pair']*1000,1), 'K', d['roofline']['chain']['pairs_per_lane'])" >> $O/summary.txt 2>&1
  done
done
done
DS2CTC_MAX_CHAIN_WARPS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_mc2.log 2>&1; echo PYTEST $? >> $O/pytest_mc2.log
DS2CTC_LIB=build/variants/libds2ctc_halo6.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_halo6.log 2>&1; echo PYTEST $? >> $O/pytest_halo6.log
cat $O/summary.txt

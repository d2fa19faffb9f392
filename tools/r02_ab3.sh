set -u
O=gpurun_out/${TAG}; mkdir -p $O
for w in english sortagrad edge1500; do
  for v in head nonorm cur; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_LIB=$L timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}_${v}.json 2> $O/${w}_${v}.err
    python -c "import json; d=json.load(open('$O/${w}_${v}.json')); print('$w $v', round(d['value']), round(d['ms_per_step']*1000,1), 'us', 'k_pair', round(d['stage_ms']['k_pair']*1000,1))" >> $O/summary.txt 2>&1
  done
done
for v in cur; do
  if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
  DS2CTC_LIB=$L timeout 600 python tools/parity_probe.py --only t1500-peaked8 sortagrad-320 sortagrad-512 english-peaked8 --analyse none > $O/probe_$v.log 2>&1
done
cat $O/summary.txt
timeout 300 python -c "
import sys; sys.argv=['x']; sys.path.insert(0,'tools/epoch_timing')
import build_and_run as b
b.run('build/epoch_timing/libds2ctc_timing_base.so', 29, 1500, 300, 16, brief=False)" > $O/epoch_k4.txt 2>&1

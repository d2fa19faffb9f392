set -u
O=gpurun_out/${TAG}; mkdir -p $O
for r in 1; do
for w in english config1; do
  for v in head norefresh halo6 cur; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_LIB=$L timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-cpu-baseline > $O/${w}_${v}.json 2> $O/${w}_${v}.err
    python -c "import json; d=json.load(open('$O/${w}_${v}.json')); print('$w $v', round(d['value']), round(d['ms_per_step']*1000,1), 'us', 'k_pair', round(d['stage_ms']['k_pair']*1000,1))" >> $O/summary.txt 2>&1
  done
done
done
cat $O/summary.txt

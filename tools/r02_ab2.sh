set -u
O=gpurun_out/${TAG}; mkdir -p $O
for w in english sortagrad edge1500; do
  for v in head preearly cur; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    for d in 0 1; do
      if [ "$w" = english ] && [ "$d" = 1 ]; then continue; fi
      DS2CTC_DUAL=$d DS2CTC_LIB=$L timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > $O/${w}_${v}_d$d.json 2> $O/${w}_${v}_d$d.err
      python -c "import json; d=json.load(open('$O/${w}_${v}_d$d.json')); print('$w $v dual$d', round(d['value']), round(d['ms_per_step']*1000,1), 'us', 'k_pair', round(d['stage_ms']['k_pair']*1000,1))" >> $O/summary.txt 2>&1
    done
  done
done
cat $O/summary.txt

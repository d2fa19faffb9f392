#!/bin/bash
# A/B of library variants on one box: bench.py with DS2CTC_LIB per variant, interleaved.
# usage: TAG=x WORKLOAD=english VARIANTS="head nofm cur" ROUNDS=2 bash tools/ab_bench.sh
set -u
O=gpurun_out/${TAG:-ab}; mkdir -p $O
W=${WORKLOAD:-english}
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in ${VARIANTS}; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    DS2CTC_LIB=$L timeout 300 python bench.py --workload $W --steps 50 --warmup 5 --no-cpu-baseline > $O/${W}_${v}_$r.json 2> $O/${W}_${v}_$r.err
    python -c "import json; d=json.load(open('$O/${W}_${v}_$r.json')); print('$v', $r, round(d['value']), round(d['stage_ms']['k_pair']*1e3,1), 'us')" >> $O/summary.txt
  done
done
cat $O/summary.txt

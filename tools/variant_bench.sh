#!/bin/bash
# Debug experiments: k_pair time of variant builds (build/variants/*.so) on the english workload.
mkdir -p gpurun_out
for so in build/variants/libds2ctc_*.so; do
  n=$(basename $so .so)
  DS2CTC_LIB=$so timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --soak-seconds 0.2 ${WORKLOAD:+--workload $WORKLOAD} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['value']), d['stage_ms'])"
done

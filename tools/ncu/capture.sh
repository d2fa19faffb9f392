#!/bin/bash
# Evidence capture for profiles/ (run on the GPU box, one GPU):
#   1. the bench command without ncu (must exit 0 first),
#   2. the launch list (gpu__time_duration, serialised, cold caches),
#   3. one `ncu --set full` capture of the dominant kernel.
# usage: WORKLOAD=english KERNEL=k_pair TAG=r01 bash tools/ncu/capture.sh
set -u
W=${WORKLOAD:-english}; KER=${KERNEL:-k_pair}; TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${W}_bench.json 2>gpurun_out/${TAG}_${W}_bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${TAG}_${W}_launches.csv python bench.py --workload $W --steps 2 --warmup 3 \
  --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KER --launch-skip 3 -c 1 \
  -o gpurun_out/${TAG}_${W}_${KER} python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline \
  --soak-seconds 0 > /dev/null 2>&1
echo done

set -u
O=gpurun_out/r02l; mkdir -p $O
TAG=r02l VARIANTS="head headnok8 headlayout cur" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
for d in 0 1; do
  DS2CTC_DUAL=$d timeout 300 python bench.py --workload sortagrad --steps 20 --warmup 5 --no-cpu-baseline > $O/sorta_dual$d.json 2> $O/sorta_dual$d.err
  DS2CTC_DUAL=$d timeout 300 python bench.py --workload edge1500 --steps 10 --warmup 3 --no-cpu-baseline > $O/edge_dual$d.json 2> $O/edge_dual$d.err
done
for f in $O/sorta_dual*.json $O/edge_dual*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value']), round(d['ms_per_step'],3), 'ms')" >> $O/summary.txt; done
DS2CTC_DUAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sortagrad or edge or geometry" > $O/pytest_dual.log 2>&1; echo PYTEST $? >> $O/pytest_dual.log

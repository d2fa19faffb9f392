# Host call: two-pass enqueue (uploads + launches, then downloads) vs one pass.
set -u
O=gpurun_out/${TAG:-r02twopass}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
run() {  # name workload env...
  n=$1; w=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  python -c "import json; d=json.load(open('$O/$n.json')); print('$n', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'us e2e; value', round(d['value']))" >> $O/summary.txt 2>&1
}
for r in 1 2 3; do
  run eng_2p_$r english
  run eng_1p_$r english DS2CTC_HOST_TWO_PASS=0
done
for w in config1 sortagrad mandarin edge1500; do
  run ${w}_2p $w
  run ${w}_1p $w DS2CTC_HOST_TWO_PASS=0
done

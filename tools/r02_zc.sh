# Zero-copy host call: parity (host tests), then e2e A/B zero-copy vs chunked.
set -u
O=gpurun_out/${TAG:-r02zc}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" -s > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
python -c "from paper_1512_02595_b200 import _lib; print('watchdog', _lib.watchdog())" >> $O/pytest.log 2>&1
run() {  # name workload env...
  n=$1; w=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  python -c "import json; d=json.load(open('$O/$n.json')); print('$n', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'us e2e; value', round(d['value']))" >> $O/summary.txt 2>&1
}
for r in 1 2; do
  run eng_zc_$r english
  run eng_chunk_$r english DS2CTC_HOST_ZEROCOPY=0 DS2CTC_HOST_STREAM=0
done
for w in config1 sortagrad edge1500; do
  run ${w}_zc $w
  run ${w}_chunk $w DS2CTC_HOST_ZEROCOPY=0 DS2CTC_HOST_STREAM=0
done
# FC backward (decoupled raw ring for dW)
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest_fc.log 2>&1; echo PYTEST $? >> $O/pytest_fc.log
for r in 1 2; do
  timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_$r.json 2> $O/step_$r.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fc|k_pad|k_transpose|k_bias" --csv --log-file $O/fc_launches.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

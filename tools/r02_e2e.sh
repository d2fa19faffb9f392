# Host-path (e2e) A/B: serial vs concurrent chunk uploads, chunk counts.
set -u
O=gpurun_out/${TAG:-r02e2e}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
run() {  # name workload env...
  n=$1; w=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  python -c "import json; d=json.load(open('$O/$n.json')); print('$n', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'us e2e; value', round(d['value']))" >> $O/summary.txt 2>&1
}
for r in 1 2; do
  run eng_c4_serial_$r english DS2CTC_HOST_CHUNKS=4
  run eng_c4_conc_$r english DS2CTC_HOST_CHUNKS=4 DS2CTC_HOST_SERIAL_UPLOAD=0
  run eng_c8_serial_$r english DS2CTC_HOST_CHUNKS=8
  run eng_c2_serial_$r english DS2CTC_HOST_CHUNKS=2
  run eng_c6_serial_$r english DS2CTC_HOST_CHUNKS=6
done
for w in config1 sortagrad mandarin; do
  run ${w}_serial $w DS2CTC_HOST_SERIAL_UPLOAD=1
  run ${w}_conc $w DS2CTC_HOST_SERIAL_UPLOAD=0
done
run mandarin_c4_serial mandarin DS2CTC_HOST_CHUNKS=4

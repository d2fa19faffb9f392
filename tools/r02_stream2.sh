# Streamed host call: which side costs (input flag writes vs output waits).
set -u
O=gpurun_out/${TAG:-r02stream2}; mkdir -p $O
run() {  # name workload env...
  n=$1; w=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  python -c "import json; d=json.load(open('$O/$n.json')); print('$n', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'us e2e; value', round(d['value']))" >> $O/summary.txt 2>&1
}
for r in 1 2; do
  run i1o1_$r english DS2CTC_STREAM_IN=1 DS2CTC_STREAM_OUT=1
  run i8o1_$r english DS2CTC_STREAM_IN=8 DS2CTC_STREAM_OUT=1
  run i1o8_$r english DS2CTC_STREAM_IN=1 DS2CTC_STREAM_OUT=8
  run i2o2_$r english DS2CTC_STREAM_IN=2 DS2CTC_STREAM_OUT=2
  run chunk_$r english DS2CTC_HOST_STREAM=0
done

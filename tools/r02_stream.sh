# Streamed host call: parity (host tests), then e2e A/B streamed vs chunked.
set -u
O=gpurun_out/${TAG:-r02stream}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "host" -s > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
python -c "from paper_1512_02595_b200 import _lib; print('watchdog', _lib.watchdog())" >> $O/pytest.log 2>&1
run() {  # name workload env...
  n=$1; w=$2; shift 2
  env "$@" timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-cpu-baseline > $O/$n.json 2> $O/$n.err
  python -c "import json; d=json.load(open('$O/$n.json')); print('$n', round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1), 'us e2e; value', round(d['value']))" >> $O/summary.txt 2>&1
}
for r in 1 2; do
  run eng_stream_$r english
  run eng_chunk_$r english DS2CTC_HOST_STREAM=0
  run eng_stream_i4o4_$r english DS2CTC_STREAM_IN=4 DS2CTC_STREAM_OUT=4
  run eng_stream_i16o16_$r english DS2CTC_STREAM_IN=16 DS2CTC_STREAM_OUT=16
done
run mandarin_default mandarin
run edge1500_stream edge1500
run edge1500_chunk edge1500 DS2CTC_HOST_STREAM=0

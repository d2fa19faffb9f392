# Mandarin: k_pair dual-resident (64 SMs) with the dense pass overlapped on the freed SMs.
set -u
O=gpurun_out/${TAG:-r02mdual}; mkdir -p $O
for r in 1 2; do
  for cfg in "0 0" "1 0" "1 1" "0 1"; do
    set -- $cfg
    DS2CTC_DENSE_OVERLAP=$1 DS2CTC_DUAL=$2 timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/ov$1_dual$2_$r.json 2> $O/ov$1_dual$2_$r.err
    python -c "import json; d=json.load(open('$O/ov$1_dual$2_$r.json')); print('overlap $1 dual $2', $r, round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k,x in d['stage_ms'].items()})" >> $O/summary.txt 2>&1
  done
done
DS2CTC_DENSE_OVERLAP=1 DS2CTC_DUAL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "shape1 or nan or cost_only or blank" > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log

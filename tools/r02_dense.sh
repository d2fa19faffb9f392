# Dense-pass A/B (Mandarin): CTA width variants, serial vs overlapped; gpu parity suite on the default build.
set -u
O=gpurun_out/${TAG:-r02dense}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for r in 1 2; do
  for v in cur d512 d512m4 d384 d1024m2; do
    if [ "$v" = cur ]; then L=""; else L=build/variants/libds2ctc_$v.so; fi
    for ov in 0 1; do
      DS2CTC_DENSE_OVERLAP=$ov DS2CTC_LIB=$L timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/${v}_ov${ov}_$r.json 2> $O/${v}_ov${ov}_$r.err
      python -c "import json; d=json.load(open('$O/${v}_ov${ov}_$r.json')); print('$v ov$ov', $r, round(d['value']), round(d['ms_per_step']*1e3,1), {k: round(x*1e3,1) for k,x in d['stage_ms'].items()})" >> $O/summary.txt 2>&1
    done
  done
done

# Evidence capture for profiles/ (one GPU): gpu tests, smoke, bench lines, ncu
# full captures of the dominant kernels (bank conflicts, stalls, DRAM bytes),
# launch lists, the hash-stamped traffic json, the parity probe. The full
# captures run the host call unchunked (DS2CTC_HOST_CHUNKS=1) so that the
# captured launch is a whole B = 64 batch, like the device-resident one.
set -u
O=gpurun_out/${TAG:-r02ev}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST $? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
for w in english mandarin sortagrad english-step config1 edge1500; do
  timeout 400 python bench.py --workload $w --steps 30 --warmup 5 --cpu-seconds 6 > $O/b_$w.json 2> $O/b_$w.err
done
timeout 200 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_english.json 2> $O/ref_english.err
timeout 900 python tools/parity_probe.py --json $O/parity.json > $O/parity.log 2>&1; echo "PROBE $?" >> $O/parity.log
DS2CTC_HOST_CHUNKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -s 3 -c 1 -o $O/k_pair_english python bench.py --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu1.log 2>&1
DS2CTC_HOST_CHUNKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dense_t -s 2 -c 1 -o $O/k_dense_mandarin python bench.py --workload mandarin --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fc_gemm -c 2 -o $O/k_fc_gemm_step python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_english.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mandarin.csv python bench.py --workload mandarin --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step.csv python bench.py --workload english-step --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 900 python tools/ncu/traffic.py english:k_pair mandarin:k_dense_t english-step:k_pair > $O/traffic.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json

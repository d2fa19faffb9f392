set -u
O=gpurun_out/r02y; mkdir -p $O
for ov in 0 1; do
  DS2CTC_DENSE_OVERLAP=$ov timeout 300 python bench.py --workload mandarin --steps 20 --warmup 5 --no-cpu-baseline > $O/mand_ov$ov.json 2> $O/mand_ov$ov.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mandarin or poisoned or blank or cost_only or geometry or golden" > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fc_gemm -c 4 --csv --log-file $O/fc_launches.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

set -u
O=gpurun_out/r02z; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -q -s > $O/fc.log 2>&1; echo PYTEST $? >> $O/fc.log
timeout 300 python bench.py --workload english-step --steps 20 --warmup 5 --no-cpu-baseline > $O/b_step.json 2> $O/b_step.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fc_gemm -c 4 --csv --log-file $O/fc_launches.csv python bench.py --workload english-step --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

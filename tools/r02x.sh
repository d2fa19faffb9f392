set -u
O=gpurun_out/r02x; mkdir -p $O
timeout 300 python bench.py --workload english-step --steps 20 --warmup 5 --no-cpu-baseline > $O/b_step.json 2> $O/b_step.err
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 4 > $O/b_english.json 2> $O/b_english.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_fc_gemm|k_pair|k_bias|k_pad|k_transpose" -s 10 -c 14 --csv --log-file $O/launches_step.csv python bench.py --workload english-step --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1

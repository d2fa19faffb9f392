#!/bin/bash
# Round-2 first GPU call: baseline state of the round-1 kernels on this box.
#   gpu tests, the parity-margin probe, English/Mandarin bench lines, and
#   ncu captures with shared-memory bank-conflict counters.
set -u
O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "PYTEST $?" >> $O/pytest_gpu.log
timeout 900 python tools/parity_probe.py --json $O/parity.json > $O/parity.log 2>&1; echo "PROBE $?" >> $O/parity.log
timeout 300 python bench.py --steps 30 --warmup 5 --cpu-seconds 5 > $O/b_english.json 2> $O/b_english.err
timeout 300 python bench.py --workload mandarin --steps 20 --warmup 5 --no-cpu-baseline > $O/b_mandarin.json 2> $O/b_mandarin.err
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_pair|k_dense" -s 3 -c 2 --csv \
  --log-file $O/bank_english.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_pair|k_dense" -s 6 -c 4 --csv \
  --log-file $O/bank_mandarin.csv python bench.py --workload mandarin --steps 2 --warmup 3 --no-cpu-baseline --soak-seconds 0 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -s 3 -c 1 \
  -o $O/k_pair_english python bench.py --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu_full.log 2>&1
echo done

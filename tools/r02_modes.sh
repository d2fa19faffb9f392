set -u
O=gpurun_out/${TAG:-r02modes}; mkdir -p $O
for i in 1 2 3 4 5 6; do timeout 120 python tools/e2e_modes.py >> $O/modes.txt 2>&1; done
for cpu in 0 3 7 11 15; do timeout 120 taskset -c $cpu python tools/e2e_modes.py >> $O/modes.txt 2>&1; done

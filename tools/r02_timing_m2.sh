set -u
O=gpurun_out/${TAG:-r02timing_m2}; mkdir -p $O
SHAPE=6000,350,60,64 timeout 900 python tools/epoch_timing/build_and_run.py variants base > $O/mandarin_brief.txt 2>&1

set -u
O=gpurun_out/${TAG:-r02timing_m}; mkdir -p $O
timeout 900 python tools/epoch_timing/build_and_run.py 6000 350 60 64 > $O/mandarin_full.txt 2>&1

# Per-epoch / per-warp clock stamps of the first English cluster (debug build).
set -u
O=gpurun_out/${TAG:-r02timing}; mkdir -p $O
timeout 900 python tools/epoch_timing/build_and_run.py > $O/english_full.txt 2>&1
timeout 900 python tools/epoch_timing/build_and_run.py variants base > $O/english_brief.txt 2>&1

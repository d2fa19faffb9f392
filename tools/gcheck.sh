mkdir -p gpurun_out
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo PYTEST $? >> gpurun_out/t.log
timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b.log 2>&1
timeout 400 python tools/epoch_timing/build_and_run.py variants $VARIANTS > gpurun_out/efull.log 2>&1
grep -E "variant|cta0: (phase|chain warp 2|service epoch 19|total)" gpurun_out/efull.log > gpurun_out/e.log

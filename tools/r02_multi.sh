set -u
O=gpurun_out/${TAG:-r02m2}; mkdir -p $O
N=${NGPU:-2}
nvidia-smi -L > $O/gpus.txt
timeout 600 python -m pytest tests/test_gpu_multi.py -m gpu -x -q -s > $O/pytest_multi.log 2>&1; echo PYTEST $? >> $O/pytest_multi.log
for w in english sortagrad english-step; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --workload $w --steps 30 --warmup 5 > $O/b${N}_$w.json 2> $O/b${N}_$w.err
done

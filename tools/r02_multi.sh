# Multi-GPU evidence on one box: gpu multi tests, then bench lines at N=1,2,..,NGPU.
set -u
O=gpurun_out/${TAG:-r02m2}; mkdir -p $O
N=${NGPU:-2}
nvidia-smi -L > $O/gpus.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST $? >> $O/pytest_gpu.log
for w in ${WORKLOADS:-english sortagrad english-step}; do
  timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --cpu-seconds 3 > $O/b1_$w.json 2> $O/b1_$w.err
  n=2
  while [ $n -le $N ]; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $n --workload $w --steps 30 --warmup 5 > $O/b${n}_$w.json 2> $O/b${n}_$w.err
    n=$((n * 2))
  done
done

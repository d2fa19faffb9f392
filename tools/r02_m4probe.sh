# 4-GPU Mandarin step: mailbox vs NCCL reduce, and 4 independent single-GPU processes at once.
set -u
O=gpurun_out/${TAG:-r02m4probe}; mkdir -p $O
for r in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --workload mandarin --steps 30 --warmup 5 > $O/b4_mailbox_$r.json 2> $O/b4_mailbox_$r.err
  DS2CTC_NCCL_REDUCE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --workload mandarin --steps 30 --warmup 5 > $O/b4_nccl_$r.json 2> $O/b4_nccl_$r.err
done
for i in 0 1 2 3; do
  CUDA_VISIBLE_DEVICES=$i timeout 300 python bench.py --workload mandarin --steps 30 --warmup 5 --no-cpu-baseline > $O/solo_$i.json 2> $O/solo_$i.err &
done
wait
nproc > $O/nproc.txt; uptime >> $O/nproc.txt
for f in $O/*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d['n_gpus'], round(d['value']), round(d['ms_per_step']*1e3,1))" >> $O/summary.txt 2>&1; done

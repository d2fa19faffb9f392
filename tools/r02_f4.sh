# f4 over peer memory: 2-GPU tests, english-step at N=2 (peer vs NCCL), traffic re-stamp on GPU 0.
set -u
O=gpurun_out/${TAG:-r02f4}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multi.py -m gpu -x -q > $O/pytest_multi.log 2>&1; echo PYTEST $? >> $O/pytest_multi.log
for r in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload english-step --steps 30 --warmup 5 > $O/b2_step_peer_$r.json 2> $O/b2_step_peer_$r.err
  DS2CTC_NCCL_REDUCE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --workload english-step --steps 30 --warmup 5 > $O/b2_step_nccl_$r.json 2> $O/b2_step_nccl_$r.err
done
timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/b1_step.json 2> $O/b1_step.err
for f in $O/*.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f'.split('/')[-1], d['n_gpus'], round(d['value']), round(d['ms_per_step']*1e3,1), d.get('fc_backward',{}).get('param_grad_allreduce'), round(d.get('fc_backward',{}).get('ms',0)*1e3,1))" >> $O/summary.txt 2>&1; done
CUDA_VISIBLE_DEVICES=0 timeout 900 python tools/ncu/traffic.py english:k_pair mandarin:k_dense_t english-step:k_pair > $O/traffic.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json

# FC backward: dx concurrent with dW (forked stream) vs serial.
set -u
O=gpurun_out/${TAG:-r02fc2}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fc.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
for r in 1 2; do
  for c in 1 0; do
    DS2CTC_FC_CONCURRENT=$c timeout 300 python bench.py --workload english-step --steps 30 --warmup 5 --no-cpu-baseline > $O/step_c${c}_$r.json 2> $O/step_c${c}_$r.err
    python -c "import json; d=json.load(open('$O/step_c${c}_$r.json')); f=d['fc_backward']; print('c$c', $r, round(d['value']), round(d['ms_per_step']*1e3,1), 'fc', round(f['ms']*1e3,1), round(f['achieved_gbs']))" >> $O/summary.txt
  done
done
# host topology and e2e vs CPU placement
nvidia-smi topo -m > $O/topo.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
python - > $O/affinity.txt 2>&1 <<'PY'
import pynvml, os
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = os.cpu_count()
words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
cpus = [i for i in range(n) if (words[i // 64] >> (i % 64)) & 1]
print("cpu_count", n, "gpu0 local cpus", cpus)
print("sched_getaffinity", sorted(os.sched_getaffinity(0)))
PY
for r in 1 2; do
  timeout 300 python bench.py --workload english --steps 30 --warmup 5 --no-cpu-baseline > $O/eng_$r.json 2> $O/eng_$r.err
  python -c "import json; d=json.load(open('$O/eng_$r.json')); print('default', $r, round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1))" >> $O/summary.txt
  L=$(python -c "
import pynvml, os
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0); n = os.cpu_count()
w = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
print(','.join(str(i) for i in range(n) if (w[i // 64] >> (i % 64)) & 1))")
  taskset -c $L timeout 300 python bench.py --workload english --steps 30 --warmup 5 --no-cpu-baseline > $O/eng_local_$r.json 2> $O/eng_local_$r.err
  python -c "import json; d=json.load(open('$O/eng_local_$r.json')); print('gpu-local cpus', $r, round(d['e2e']['value']), round(d['e2e']['ms_per_step']*1e3,1))" >> $O/summary.txt
done

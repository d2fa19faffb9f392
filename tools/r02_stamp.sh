# Final build: gpu tests, smoke, traffic stamp, one English and one Mandarin bench line (traffic reported).
set -u
O=gpurun_out/${TAG:-r02stamp}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST $? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
timeout 900 python tools/ncu/traffic.py english:k_pair mandarin:k_dense_t english-step:k_pair > $O/traffic.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
for w in english mandarin; do
  timeout 400 python bench.py --workload $w --steps 30 --warmup 5 --cpu-seconds 6 > $O/b_$w.json 2> $O/b_$w.err
done

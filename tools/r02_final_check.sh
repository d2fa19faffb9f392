# Final build check: all gpu tests, smoke, English / Mandarin / English-step bench lines (traffic reported).
set -u
O=gpurun_out/${TAG:-r02final}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST $? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1
for w in english mandarin english-step; do
  timeout 400 python bench.py --workload $w --steps 30 --warmup 5 --cpu-seconds 6 > $O/b_$w.json 2> $O/b_$w.err
done
timeout 200 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_english.json 2> $O/ref_english.err

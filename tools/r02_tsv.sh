set -u
O=gpurun_out/${TAG:-r02tsv}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_cpp.py -m gpu -x -q -s > $O/pytest_cpp.log 2>&1; echo PYTEST $? >> $O/pytest_cpp.log
timeout 300 python bench.py --workload mandarin --steps 10 --warmup 3 --no-cpu-baseline > $O/b_mandarin.json 2> $O/b_mandarin.err
timeout 300 python bench.py --workload english --steps 10 --warmup 3 --no-cpu-baseline > $O/b_english.json 2> $O/b_english.err

set -u
O=gpurun_out/${TAG:-r02random}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "random or margin" -s > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log

set -u
O=gpurun_out/${TAG:-r02suite}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -s > $O/pytest_gpu_verbose.log 2>&1; echo PYTEST $? >> $O/pytest_gpu_verbose.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.log 2>&1

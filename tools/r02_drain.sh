# A/B: prev (HEAD), cur (last epoch's rows over all warps), drain2 (+ parts and prev2 rows over all warps).
set -u
O=gpurun_out/${TAG:-r02drain}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo PYTEST $? >> $O/pytest.log
DS2CTC_LIB=build/variants/libds2ctc_drain2.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "golden or fixed or peaked or sortagrad or nan or blank" > $O/pytest_drain2.log 2>&1; echo PYTEST $? >> $O/pytest_drain2.log
for w in english config1 mandarin sortagrad; do
  TAG=$(basename $O)/ab WORKLOAD=$w VARIANTS="prev cur drain2" ROUNDS=2 bash tools/ab_bench.sh > /dev/null 2>&1
done

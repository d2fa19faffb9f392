# ncu --set full captures of whole-batch launches (host call unchunked).
set -u
O=gpurun_out/${TAG:-r02cap}; mkdir -p $O
DS2CTC_HOST_CHUNKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -s 3 -c 1 -o $O/k_pair_english python bench.py --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu1.log 2>&1
DS2CTC_HOST_CHUNKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dense_t -s 2 -c 1 -o $O/k_dense_mandarin python bench.py --workload mandarin --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu2.log 2>&1
DS2CTC_HOST_CHUNKS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -s 3 -c 1 -o $O/k_pair_mandarin python bench.py --workload mandarin --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu3.log 2>&1

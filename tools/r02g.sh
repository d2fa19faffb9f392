set -u
O=gpurun_out/r02g; mkdir -p $O
for v in head noall; do
  DS2CTC_LIB=build/variants/libds2ctc_$v.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pair -s 3 -c 1 \
    -o $O/k_pair_$v python bench.py --steps 1 --warmup 3 --no-cpu-baseline --soak-seconds 0 > $O/ncu_$v.log 2>&1
done

# Radix pass timing probes (variants 1-4 of HBP_RADIX_VARIANT) and ncu of the in-place pass + histogram
for v in 1 2 3 4; do for args in "--n 9800000 --bits 15" "--n 10000000 --bits 1"; do echo "variant $v $args"; HBP_RADIX_VARIANT=$v timeout 120 python tools/radix_bench.py $args --reps 3; done; done > gpurun_out/radix_probe.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_os_pass_ip|k_os_hist" -s 6 -c 3 -o gpurun_out/r02_radix_ip python tools/radix_bench.py --n 9800000 --bits 15 --reps 1 > gpurun_out/ncu_radix.log 2>&1
echo done

# Look-back window A/B (variant 2: one word per round trip, 5: four) and parity of variant 5
for v in 2 5 2 5; do for args in "--n 9800000 --bits 15" "--n 10000000 --bits 1" "--n 9800000 --bits 17 --desc"; do echo "variant $v $args"; HBP_RADIX_VARIANT=$v timeout 120 python tools/radix_bench.py $args --reps 3; done; done > gpurun_out/radix_lb.log 2>&1
HBP_RADIX_VARIANT=5 timeout 600 python -m pytest tests/test_gpu_primitives.py tests/test_gpu_plan.py -x -q -m gpu > gpurun_out/radix_lb_tests.log 2>&1; echo "rc $?" >> gpurun_out/radix_lb_tests.log

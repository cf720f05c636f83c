set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
for v in 1 2; do for args in "--n 9800000 --bits 15" "--n 10000000 --bits 1" "--n 9800000 --bits 17 --desc" "--n 2000000 --bits 15"; do echo "variant $v $args"; HBP_RADIX_VARIANT=$v timeout 120 python tools/radix_bench.py $args --reps 3; done; done > gpurun_out/radix_ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log

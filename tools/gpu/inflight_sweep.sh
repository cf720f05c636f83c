# Plans in flight (HBP_BENCH_IN_FLIGHT) x steps, main legs only; histogram grid check
for f in 5 6 8 10; do for k in 10 20; do echo "in_flight $f steps $k"; HBP_BENCH_IN_FLIGHT=$f timeout 300 python bench.py --steps $k --no-cpu --no-sweep --no-c4 --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['one_at_a_time']['ms_per_step'],3), d['clocks']['sm_mhz'])"; done; done > gpurun_out/inflight_sweep.log 2>&1
for a in "--n 9800000 --bits 15" "--n 10000000 --bits 1" "--n 2000000 --bits 15"; do echo "$a"; timeout 120 python tools/radix_bench.py $a --reps 3; done > gpurun_out/hist_grid.log 2>&1
timeout 600 python -m pytest tests/test_gpu_primitives.py -x -q -m gpu > gpurun_out/prim.log 2>&1; echo "rc $?" >> gpurun_out/prim.log

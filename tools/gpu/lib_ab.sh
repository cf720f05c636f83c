# A/B of the committed library (abvar/base_libhbp_b200.so) against the working tree's on one box,
# alternated: device ms per plan in flight, one at a time, next-fit round family, C3 sweep
timeout 900 python -m pytest tests/test_gpu_plan.py tests/test_gpu_primitives.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1; echo "rc $?" >> gpurun_out/ab_tests.log
for r in 1 2 3; do
  for v in base new; do
    if [ $v = base ]; then export HBP_LIB_OVERRIDE=$PWD/abvar/base_libhbp_b200.so; else unset HBP_LIB_OVERRIDE; fi
    echo -n "$v "; timeout 300 python bench.py --no-cpu --no-c4 --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); f=d['roofline']['families']
print(round(d['ms_per_step'],3), round(d['one_at_a_time']['ms_per_step'],3), 'nf', f['nf.round']['ms'], 'chain', f['fit.chain']['ms'], 'fyl', f['fy.lists']['ms'], 'fys', f['fy.sources_gather']['ms'], 'fysc', f['fy.scatter']['ms'], round(d['sweep']['candidates_per_s']))"
  done
done > gpurun_out/lib_ab.log 2>&1

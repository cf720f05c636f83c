# C3 sweep A/B: the committed library (abvar/base_libhbp_b200.so) against the working tree's, alternated
for r in 1 2 3; do
  for v in base new; do
    if [ $v = base ]; then export HBP_LIB_OVERRIDE=$PWD/abvar/base_libhbp_b200.so; else unset HBP_LIB_OVERRIDE; fi
    echo -n "$v "; timeout 300 python bench.py --no-cpu --no-c4 --no-ingest 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['one_at_a_time']['ms_per_step'],3), d['sweep']['seconds_reps'], round(d['sweep']['candidates_per_s']))"
  done
done > gpurun_out/sweep_ab.log 2>&1

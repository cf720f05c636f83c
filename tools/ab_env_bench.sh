#!/bin/bash
# A/B of env settings on one box: C2 device step, e2e step, launches, and the
# nf / fy stage times (bench.py without the side legs). ("" = default)
#   bash tools/ab_env_bench.sh "" "HBP_NO_SIDE=1"
for e in "$@"; do
  env $e python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep --no-c4 --no-ingest 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); st=d['stages_ms']; print('[$e]', 'one-at-a-time', round(d['one_at_a_time']['ms_per_step'],3), round(d['e2e']['one_at_a_time']['ms_per_step'],3), 'in flight', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['gpu_launches'], {k:v for k,v in st.items() if k.startswith('nf') or k.startswith('fy') or k.startswith('fit')})"
done

#!/bin/bash
# A/B of the first-fit chain on the GPU box: parity tests, then fit.chain
# device time and the C2 step with and without an env switch ($1, e.g.
# HBP_CHAIN_NOSINGLE=1), plus the C1 [131072] chain of the C3 sweep.
sw=${1:-HBP_CHAIN_NOSINGLE=1}
python -m pytest tests/test_gpu_plan.py tests/test_gpu_reference_scale.py -x -q -p no:cacheprovider 2>&1 | tail -2
for e in "" "$sw"; do
  env $e python tools/stage_list.py 2>&1 | grep -E "total|fit.chain|fit.replay" | head -3 | sed "s/^/[${e:-new}] /"
  env $e HBP_TRACE=1 python tools/chain_dump_c1.py 131072 2>&1 | grep -E "fit chain" | sed "s/^/[${e:-new}] C1 /"
  env $e python tools/sweep_streams.py 16 | sed "s/^/[${e:-new}] C3 /"
done

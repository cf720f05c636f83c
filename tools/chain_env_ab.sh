#!/bin/bash
# fit.chain device time of the C2 step and of C1's [131072] plan, and C3
# throughput, under each env setting given ("" = default)
for e in "$@"; do
  env $e python tools/stage_list.py 2>&1 | grep -E "fit.chain" | head -1 | sed "s/^/[${e:-default}] C2 /"
  env $e HBP_TRACE=1 python tools/chain_dump_c1.py 131072 2>&1 | grep -E "fit chain" | sed "s/.*M \([0-9]*\) warps \([0-9]*\).*: \(.*\)/[${e:-default}] C1 M \1 warps \2 \3/"
  env $e HBP_TRACE=1 python tools/chain_dump_c1.py 8192 32768 131072 2>&1 | grep -E "fit chain" | sed "s/.*M \([0-9]*\) warps \([0-9]*\).*: \(.*\)/[${e:-default}] C1x3 M \1 warps \2 \3/"
  env $e python tools/sweep_streams.py 16 | sed "s/^/[${e:-default}] C3 /"
done

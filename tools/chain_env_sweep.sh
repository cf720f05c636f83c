#!/bin/bash
# Chain launch times (HBP_TRACE) of one C2 step under several settings of the
# chain's tuning environment variables. Usage: bash tools/chain_env_sweep.sh "VAR=a VAR=b ..."
for kv in $1; do
  echo "== $kv"
  env HBP_TRACE=1 $kv python tools/profile_step.py --steps 2 2>&1 | grep "fit chain" | tail -3 | sed 's/.*bins/bins/'
done

#!/bin/bash
# Per-launch device time of the first-fit chain (and its replay) in one C2
# step, under each env setting given ("" = default). ncu serialises the
# launches; the chain is one cooperative kernel, so its time is unaffected.
#   bash tools/chain_launch_ab.sh "" "HBP_CHAIN_RB=16"
for e in "$@"; do
  f=gpurun_out/chain_ab_$$.csv
  env $e ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_ff_(chain|replay)" --csv \
      --log-file $f python tools/profile_step.py --steps 1 > /dev/null 2>&1
  python - "$f" "${e:-default}" <<'PY'
import csv, sys
rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum"]
ch = [float(r["Metric Value"]) / 1e3 for r in rows if "k_ff_chain" in r["Kernel Name"]]
rp = [float(r["Metric Value"]) / 1e3 for r in rows if "k_ff_replay" in r["Kernel Name"]]
print(f"[{sys.argv[2]}] chain us {[round(x) for x in ch]} sum {sum(ch):.0f} | replay {[round(x) for x in rp]} sum {sum(rp):.0f}")
PY
  rm -f $f
done

#!/usr/bin/env bash
# Profiles one C2 step on the GPU box (run under gpurun, one GPU):
#   1. launch list (per-launch device time, clocks not pinned)
#   2. DRAM traffic of every launch of the step (roofline "traffic")
#   3. full-set captures of the first-fit chain (3 launches), the largest
#      next-fit round, the shuffle kernels and a radix pass
# Outputs go to gpurun_out/; summaries are copied into profiles/.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r02}
mkdir -p "$OUT"
STEP="python tools/profile_step.py --steps 1"

ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_launches_c2.csv" $STEP > /dev/null 2>&1
echo "launch list: $(grep -c '"gpu__time_duration.sum"' "$OUT/${TAG}_launches_c2.csv") launches"

ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_traffic_c2.csv" $STEP > /dev/null 2>&1
echo "traffic rows: $(grep -c dram__bytes_read "$OUT/${TAG}_traffic_c2.csv")"

ncu --set full --clock-control none --import-source on -k regex:k_ff_chain -c 3 \
    -o "$OUT/${TAG}_chain" -f $STEP > /dev/null 2>&1
echo "chain capture: $?"
# the largest launch (by grid) of each: next-fit round, shuffle kernels, radix
# pass -- skip the launches of that kernel before it in the launch list
for k in k_nf_round k_fy_lists k_fy_scatter k_fy_sources k_os_pass; do
  skip=$(python - "$OUT/${TAG}_launches_c2.csv" "$k" <<'PY'
import csv, sys
rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum" and sys.argv[2] in r["Kernel Name"]]
grid = [eval(r["Grid Size"])[0] for r in rows]
print(grid.index(max(grid)) if grid else 0)
PY
)
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip "$skip" -c 1 \
      -o "$OUT/${TAG}_$k" -f $STEP > /dev/null 2>&1
  echo "$k capture: $?"
done

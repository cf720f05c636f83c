#!/usr/bin/env bash
# Profiles one C2 step on the GPU box (run under gpurun, one GPU):
#   1. launch list (per-launch device time, clocks not pinned)
#   2. DRAM traffic of every launch of the scan family (roofline "traffic")
#   3. one full-set capture of the first-fit chain and of the hottest scan
# Outputs go to gpurun_out/; summaries are copied into profiles/.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p "$OUT"
STEP="python tools/profile_step.py --steps 1"

ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_launches_c2.csv" $STEP > /dev/null 2>&1
echo "launch list: $(grep -c '"gpu__time_duration.sum"' "$OUT/${TAG}_launches_c2.csv") launches"

ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:k_scan_lookback --csv --log-file "$OUT/${TAG}_scan_traffic.csv" $STEP > /dev/null 2>&1
echo "scan traffic rows: $(grep -c dram__bytes_read "$OUT/${TAG}_scan_traffic.csv")"

ncu --set full --clock-control none --import-source on -k regex:k_ff_chain -c 3 \
    -o "$OUT/${TAG}_chain" -f $STEP > /dev/null 2>&1
echo "chain capture: $?"
# the largest plain scan of the step: the prefix sums of group 0's first ISF
# round (9.7M u64 elements; launch index among the scans, this round's code)
ncu --set full --clock-control none --import-source on -k regex:k_scan_lookback -s ${SCAN_SKIP:-51} -c 1 \
    -o "$OUT/${TAG}_scan" -f $STEP > /dev/null 2>&1
echo "scan capture: $?"
for k in k_fy_lists k_radix_scatter k_nf_emit; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s ${BIG_SKIP:-8} -c 1 \
      -o "$OUT/${TAG}_$k" -f $STEP > /dev/null 2>&1
  echo "$k capture: $?"
done
# corpus parse + plan reader
ING="python tools/profile_ingest.py"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_launches_ingest.csv" $ING > /dev/null 2>&1
echo "ingest launch list: $?"
ncu --set full --clock-control none --import-source on -k regex:k_parse_jsonl -c 1 \
    -o "$OUT/${TAG}_k_parse_jsonl" -f $ING > /dev/null 2>&1
echo "k_parse_jsonl capture: $?"
ncu --set full --clock-control none --import-source on -k regex:k_plan_lines -c 1 \
    -o "$OUT/${TAG}_k_plan_lines" -f $ING > /dev/null 2>&1
echo "k_plan_lines capture: $?"

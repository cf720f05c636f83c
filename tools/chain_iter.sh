#!/bin/bash
# GPU iteration on the first-fit chain: parity at scale, then the chain
# timeline of one C2 step (HBP_TRACE) and the bench's device step time.
# Usage (on the GPU box): bash tools/chain_iter.sh [tag]
tag=${1:-it}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_plan.py tests/test_gpu_reference_scale.py -x -q > gpurun_out/$tag.tests.log 2>&1
tail -2 gpurun_out/$tag.tests.log
rm -f gpurun_out/$tag.tl.bin
HBP_TRACE=1 HBP_CHAIN_TL=gpurun_out/$tag.tl.bin python tools/profile_step.py --steps 1 > gpurun_out/$tag.trace.log 2>&1
python tools/chain_timeline.py gpurun_out/$tag.tl.bin > gpurun_out/$tag.tl.txt 2>&1
grep "fit chain" gpurun_out/$tag.trace.log
python bench.py --steps 10 --warmup 3 --no-cpu --no-sweep --no-c4 --no-ingest > gpurun_out/$tag.bench.log 2>&1
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/{tag}.bench.log") if x.startswith("{")][-1]
d = json.loads(l)
print("step ms", round(d["ms_per_step"], 3), "e2e ms", round(d["e2e"]["ms_per_step"], 3), "launches", d["gpu_launches"])
print({k: v for k, v in list(d["stages_ms"].items())[:10]})
PY

"""One JSONL load_lengths (2M records of the C2 spec) and one plan_from_json
(1M-sample C2 plan manifest), for ncu captures: python tools/profile_ingest.py"""
import sys
sys.path.insert(0, '.')
import bench
from paper_2503_07680_b200 import abi
lib = abi.load_library(); ctx = abi.Context(0)
L = bench.synth(lib, dict(bench.C2), 2_000_000)
text = "".join(f'{{"id":{i},"length":{v}}}\n' for i, v in enumerate(L.tolist())).encode()
plan = ctx.build_plan(None, L[:1_000_000], bench.C2_GROUPS, 16384, device_count=8, seed=1)
manifest = plan.to_json(None, L[:1_000_000])
plan = None
ctx.synchronize()
ctx.load_lengths(text, "jsonl", with_ids=True)
ctx.plan_from_json(manifest)
ctx.synchronize()

import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np
from paper_2503_07680_b200 import abi
ctx = abi.Context(0)
rng = np.random.default_rng(1)
for fmt, text in (("raw-lengths", b"5\n 7\n\n12"), ("csv", b"a,length\n1,5\n2,6,\n"), ("jsonl", b'{"id":3,"length":4}\n{"length":9,"x":[1,{"y":"\\u00e9"}]}\n')):
    print(fmt, ctx.load_lengths(text, fmt, with_ids=True))
for bad in (b"5\nx\n", b'{"length":5,}\n'):
    try: ctx.load_lengths(bad, "jsonl" if bad.startswith(b"{") else "raw")
    except Exception as e: print("err", e)
L = rng.integers(1, 65, size=5000)
for st in ("bfs", "spfhp"):
    for env in ("", "HBP_FIT_GLOBAL"):
        if env: os.environ[env] = "1"
        p = ctx.pack(None, L, 64, st, seed=3).flat(); print(st, env, len(p.pack_total))
        os.environ.pop("HBP_FIT_GLOBAL", None)
L2 = rng.integers(1, 20000, size=3000)
plan = ctx.build_plan(None, L2, [(16384, 1, 0), (65536, 2, 4)], l_best=16384, device_count=3, seed=11)
t = plan.to_json(None, L2)
b, i, l = ctx.plan_from_json(t)
print("reader", b.to_json(i, l) == t)
for bad in (t.replace(b'"version": 1', b'"version": 2'), t[:len(t)//2], b"{}"):
    try: ctx.plan_from_json(bad)
    except Exception as e: print("err", str(e)[:60])
print("done")

for reg in 0; do for w in 1 8 16 32; do
  if [ $reg = 1 ]; then export HBP_CHAIN_REGULAR=1; else unset HBP_CHAIN_REGULAR; fi
  HBP_SWEEP_STREAMS=$w timeout 120 python -c "
import sys,time; sys.path.insert(0,'.')
import numpy as np, bench
from paper_2503_07680_b200 import abi, sweep
lib=abi.load_library(); ctx=abi.Context(0)
L=np.maximum(bench.synth(lib, bench.C1),128); s,k=abi.make_samples(None,L,'c1')
c=sweep.make_candidates(ctx,131072,bench.SWEEP_SMALLER,bench.SWEEP_SP)
ctx.sweep_samples(s,c[:16],None,device_count=8,seed=7); ctx.synchronize()
t=time.perf_counter(); r=ctx.sweep_samples(s,c[:512],None,device_count=8,seed=7); ctx.synchronize(); el=time.perf_counter()-t
print('regular=$reg streams=$w', round(el,3),'s', round(512/el,1),'cand/s best', r[1])"
done; done

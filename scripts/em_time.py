"""EM iteration throughput at N=2048 (paper Table 2's workload is 100 EM
iterations over an N^3 volume): device time of `iters` steps on `batch`
slices of the synthetic stack (CUDA events). GPU probe for DESIGN.md."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from paper_1506_00014_b200 import phantoms  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
plan = lp.RadonPlan(g, max_batch=B)
f = phantoms.stack(N, B).clamp_min(0)
sino = lp.fast_radon(f, plan).clamp_min(0)
lp.em_run(sino, plan, 1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
est, ll = lp.em_run(sino, plan, iters)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(json.dumps({"N": N, "batch": B, "iters": iters, "ms": ms, "ms_per_iter_per_slice": ms / iters / B,
                  "slice_iters_per_s": B * iters / (ms / 1e3), "loglik_first_last": [ll[0][0], ll[0][-1]]}))

"""R and R# at N=2048 (the bench plan and batch, 16 slices) twice: the target
process for ncu captures (scripts/gpu_round.sh; -s 10 skips the first pair)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from paper_1506_00014_b200 import phantoms  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
plan = lp.RadonPlan(g, max_batch=B)
f = phantoms.stack(N, B)
for _ in range(2):
    s = lp.fast_radon(f, plan)
    b = lp.fast_backprojection(s, plan)
torch.cuda.synchronize()
print("done", float(s.abs().sum()), float(b.abs().sum()))

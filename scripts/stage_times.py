"""Per-stage CUDA-event times of R and R# for one plan variant (GPU A/B probe).

    python scripts/stage_times.py [N] [batch] [--tex] [--default-plan]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from paper_1506_00014_b200 import phantoms, roofline  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
N = int(args[0]) if args else 2048
B = int(args[1]) if len(args) > 1 else 8
tex = "--tex" in sys.argv
g = lp.sampling_plan(N, 3, 0, 0 if "--default-plan" in sys.argv else lp.smooth_n_rho(N))
plan = lp.RadonPlan(g, max_batch=B, texture_gather=tex)
f = phantoms.stack(N, B)
s = torch.empty(B, g.n_theta, N, device="cuda")
b = torch.empty(B, N, N, device="cuda")
out = {"N": N, "batch": B, "tex": tex, "n_rho": g.n_rho}
out["radon"] = roofline.profile_stages(plan, "radon", f.data_ptr(), s.data_ptr(), B, 5)
if not tex:
    out["backproject"] = roofline.profile_stages(plan, "backproject", s.data_ptr(), b.data_ptr(), B, 5)
print(json.dumps(out))

"""Driver for compute-sanitizer (tests/test_sanitizer.py): every kernel of R,
R#, R^T, the FBP filter and one EM step at N=64 through the host-buffer C ABI
(numpy buffers; torch only for the device-resident EM entry point), both plan kinds (default N_rho, 7-smooth N_rho)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_00014_b200 as lp  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
for n_rho in (0, lp.smooth_n_rho(N)):
    g = lp.sampling_plan(N, 3, 0, n_rho)
    plan = lp.RadonPlan(g, lp.zeta_spectrum(g), lp.zeta_bp_spectrum(g), max_batch=2)
    rng = np.random.default_rng(1)
    f = rng.uniform(0, 1, (3, N, N)).astype(np.float32)
    s = lp.fast_radon(f, plan)
    b = lp.fast_backprojection(s, plan)
    t = lp.radon_transpose(s, plan)
    fb = lp.fbp(s, plan, "ramp")
    em, _ = lp.em_run(torch.tensor(np.abs(s[0]), device="cuda:0"), plan, 1)
    em = em.cpu().numpy()
    assert np.isfinite(b).all() and np.isfinite(t).all() and np.isfinite(fb).all() and np.isfinite(em).all()
    plan.close()
print("sanitize driver ok")

"""Driver for compute-sanitizer over the bench kernels (tests/test_sanitizer.py):
one slice of R and R# on the N=2048 7-smooth plan, i.e. the compile-time
specialisations the bench runs (the fused fine theta kernel on the 2056
raster pitch, the TMA / mbarrier streamed rho pass for N_rho = 4374, the
N_theta = 3072 sinogram kernels), plus the default plan's padded rho
convolution. Spectra are passed in precomputed on the host so that only the
operators run under the tool."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_00014_b200 as lp  # noqa: E402

N = 2048
rng = np.random.default_rng(2)
f = rng.uniform(0, 1, (1, N, N)).astype(np.float32)
for n_rho in (lp.smooth_n_rho(N), 0):
    g = lp.sampling_plan(N, 3, 0, n_rho)
    plan = lp.RadonPlan(g, lp.zeta_spectrum(g), lp.zeta_bp_spectrum(g), max_batch=1)
    s = lp.fast_radon(f, plan)
    b = lp.fast_backprojection(s, plan)
    assert np.isfinite(s).all() and np.isfinite(b).all()
    plan.close()
print("sanitize driver ok")

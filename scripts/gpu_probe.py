"""Quick GPU probe: parity of R / R# against the oracle at small N and a
rough timing at N=2048. Development aid; the real checks live in tests/."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from oracle import lpo  # noqa: E402


def parity(N, n_rho=0, batch=2):
    g = lp.sampling_plan(N, 3, 0, n_rho)
    p = lpo.make_plan(N, 3, 0, n_rho)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=batch)
    f = np.stack([lpo.smooth_disc_image(N, 0.9, 7 + i) for i in range(batch)])
    f[0] = lpo.phantom_image(N)
    t0 = time.time()
    ref = lpo.fast_radon(p, z, f)
    t1 = time.time()
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device="cuda"), plan).cpu().numpy()
    e_r = [lpo.rel_l2(got[i], ref[i]) for i in range(batch)]
    sino = ref
    refb = lpo.fast_backprojection(p, zb, sino)
    gotb = lp.fast_backprojection(torch.tensor(sino, dtype=torch.float32, device="cuda"), plan).cpu().numpy()
    e_b = [lpo.rel_l2(gotb[i], refb[i]) for i in range(batch)]
    print(f"N={N} n_rho={g.n_rho} R rel_l2 {e_r}  R# rel_l2 {e_b}  (oracle R {t1 - t0:.2f}s)", flush=True)
    return max(e_r + e_b)


def timing(N, n_rho, batch, reps=5):
    g = lp.sampling_plan(N, 3, 0, n_rho)
    t = time.time()
    plan = lp.RadonPlan(g, max_batch=batch)
    print(f"plan N={N} n_rho={g.n_rho}: {time.time() - t:.1f}s", flush=True)
    f = torch.rand(batch, N, N, device="cuda")
    s = torch.rand(batch, g.n_theta, N, device="cuda")
    for name, fn, x in (("R", lp.fast_radon, f), ("R#", lp.fast_backprojection, s)):
        fn(x, plan)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn(x, plan)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"  {name}: {ms:.2f} ms per batch of {batch} -> {batch / ms * 1e3:.1f} slices/s", flush=True)


if __name__ == "__main__":
    worst = 0.0
    for N in (64, 128, 256):
        worst = max(worst, parity(N))
    worst = max(worst, parity(256, n_rho=lp.smooth_n_rho(256)))
    print("worst", worst)
    timing(2048, lp.smooth_n_rho(2048), 4)
    timing(2048, 0, 4)

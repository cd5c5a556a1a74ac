"""The paper's published timing tables (Table 1: R# seconds
per slice at N = 256 ... 2048; Table 2: 100 EM iterations
over an N^3 volume; both on a GeForce GTX 770, single precision, batched,
init excluded) re-measured on one B200 with this library: R, R# and one EM
iteration per slice, device time by CUDA events on the plan's launches,
B slices per launch, the reference's own sampling_plan (minimal N_rho) and
the 7-smooth plan. Writes one JSON object to stdout.

    python scripts/paper_tables.py [batch]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from paper_1506_00014_b200 import phantoms  # noqa: E402

PAPER_RSHARP_S = {256: 1.6e-3, 512: 6.1e-3, 1024: 2.5e-2, 2048: 9.9e-2}  # PAPER.md:575-578, log-polar, GTX 770
PAPER_EM100_VOLUME_S = {256: 88.0, 512: 690.0, 1024: 5.4e3, 2048: 4.2e4}

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


rows = []
for N in (256, 512, 1024, 2048):
    for smooth in (False, True):
        g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N) if smooth else 0)
        plan = lp.RadonPlan(g, max_batch=B)
        f = phantoms.stack(N, B).clamp_min(0)
        s = lp.fast_radon(f, plan)
        ms_r = timed(lambda: lp.fast_radon(f, plan))
        ms_b = timed(lambda: lp.fast_backprojection(s, plan))
        sp = s.clamp_min(0)
        iters = 5
        ms_em = timed(lambda: lp.em_run(sp, plan, iters), reps=2) / iters
        row = {"N": N, "n_theta": g.n_theta, "n_rho": g.n_rho, "plan": "smooth" if smooth else "reference",
               "batch": B, "radon_s_per_slice": ms_r / 1e3 / B, "backprojection_s_per_slice": ms_b / 1e3 / B,
               "em_iter_s_per_slice": ms_em / 1e3 / B,
               "em100_volume_s": ms_em / 1e3 / B * 100 * N}
        if not smooth:
            row["paper_gtx770_backprojection_s_per_slice"] = PAPER_RSHARP_S[N]
            row["paper_gtx770_em100_volume_s"] = PAPER_EM100_VOLUME_S[N]
            row["backprojection_speedup_vs_paper"] = PAPER_RSHARP_S[N] / row["backprojection_s_per_slice"]
        rows.append(row)
        plan.close()
print(json.dumps({"how": __doc__.split("\n\n")[0].replace("\n", " "), "device": torch.cuda.get_device_name(),
                  "rows": rows}))

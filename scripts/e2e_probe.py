"""Where the end-to-end time goes: the host-buffer C-ABI calls of the bench
(N=2048, 16 slices per call, pinned buffers) timed alone and together, next
to plain pinned copies of the same bytes (one direction, both directions)
and the device-only compute. GPU probe for DESIGN.md §6; one JSON line."""
import json
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import paper_1506_00014_b200 as lp  # noqa: E402
from paper_1506_00014_b200 import phantoms  # noqa: E402

N, B, K = 2048, 16, 8
g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
z, zb = lp.zeta_spectrum(g, device=0), lp.zeta_bp_spectrum(g, device=0)
pa = lp.RadonPlan(g, z, zb, max_batch=B)
pb = lp.RadonPlan(g, z, zb, max_batch=B)
L = lp._lib.lib()
imgs = phantoms.stack(N, B)
h_img = torch.empty(B, N, N, pin_memory=True)
h_img.copy_(imgs.cpu())
h_sino = torch.empty(B, g.n_theta, N, pin_memory=True)
h_sino2 = torch.empty(B, g.n_theta, N, pin_memory=True)
h_back = torch.empty(B, N, N, pin_memory=True)
d_img = torch.empty(B, N, N, device="cuda")
d_sino = torch.empty(B, g.n_theta, N, device="cuda")
lp._lib.check(L.lpr_gpu_radon_host(pa.handle, h_img.data_ptr(), h_sino.data_ptr(), B))
h_sino2.copy_(h_sino)


def wall(fn, k=K):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / k * 1e3


def r_call():
    lp._lib.check(L.lpr_gpu_radon_host(pa.handle, h_img.data_ptr(), h_sino.data_ptr(), B))


def b_call():
    lp._lib.check(L.lpr_gpu_backproject_host(pb.handle, h_sino2.data_ptr(), h_back.data_ptr(), B))


def both():
    t1, t2 = threading.Thread(target=r_call), threading.Thread(target=b_call)
    t1.start()
    t2.start()
    t1.join()
    t2.join()


def dev_r():
    lp.fast_radon(d_img, pa)


s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def copies(h2d_img=True, d2h_sino=True, h2d_sino=True, d2h_img=True):
    def f():
        with torch.cuda.stream(s1):
            if h2d_img:
                d_img.copy_(h_img, non_blocking=True)
            if h2d_sino:
                d_sino.copy_(h_sino2, non_blocking=True)
        with torch.cuda.stream(s2):
            if d2h_sino:
                h_sino.copy_(d_sino, non_blocking=True)
            if d2h_img:
                h_back.copy_(d_img, non_blocking=True)
        torch.cuda.synchronize()
    return f


d_img.copy_(imgs)
out = {
    "slices_per_call": B,
    "ms_R_host_call": wall(r_call),
    "ms_Rsharp_host_call": wall(b_call),
    "ms_both_calls_concurrent": wall(both),
    "ms_R_device": wall(dev_r),
    "ms_copy_h2d_img": wall(copies(True, False, False, False)),
    "ms_copy_d2h_sino": wall(copies(False, True, False, False)),
    "ms_copy_h2d_img_plus_sino": wall(copies(True, False, True, False)),
    "ms_copy_all_four_duplex": wall(copies(True, True, True, True)),
    "bytes_img_MB": B * N * N * 4 / 1e6,
    "bytes_sino_MB": B * g.n_theta * N * 4 / 1e6,
}
print(json.dumps(out))

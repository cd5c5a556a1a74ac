"""Host-side mirror of the reference's (specified) lp_ops interface.

Names, argument meaning and error behaviour follow SPEC.md:250-328 and the
reference headers (proj/include/lpradon/geometry.hpp, kernel.hpp):

    sampling_plan(N, M[, n_theta])          geometry.hpp:48-61
    zeta_spectrum / zeta_bp_spectrum(plan)  kernel.hpp:41-47
    RadonPlan(geometry)
    fast_radon(image, plan)                  SPEC.md:282-290   (Algorithm 1)
    fast_backprojection(sino, plan)          SPEC.md:291-299   (Algorithm 2)
    radon_transpose(sino, plan)              exact adjoint of fast_radon
    adjoint_gap(plan, trials)

Every call goes through the C ABI (``include/lpradon_gpu.h``) into the
sm_100a kernels; bad shapes raise ValueError (the reference's
std::invalid_argument), device failures RuntimeError. Torch CUDA tensors are
processed in place on their device and stream; numpy arrays take the host
entry points (H2D, compute, D2H inside the call).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from ._lib import Geometry, check, lib


def sampling_plan(N: int, M: int = 3, n_theta: int = 0, n_rho: int = 0) -> Geometry:
    g = Geometry()
    check(lib().lpr_geometry_make(int(N), int(M), int(n_theta), int(n_rho), ctypes.byref(g)))
    return g


def smooth_n_rho(N: int, M: int = 3) -> int:
    v = lib().lpr_smooth_n_rho(int(N), int(M))
    if v < 0:
        raise ValueError("smooth_n_rho: bad arguments")
    return v


def _spectrum(g: Geometry, kind: int, device) -> np.ndarray:
    out = np.zeros((2 * g.nts, g.n_rho), dtype=np.complex128)
    if device is None:
        check(lib().lpr_spectrum_quadrature(ctypes.byref(g), kind, out.ctypes.data))
    else:
        check(lib().lpr_gpu_spectrum_quadrature(int(device), ctypes.byref(g), kind, out.ctypes.data))
    return out


def set_spectrum_cache(directory) -> None:
    """Directory of the on-disk spectrum cache keyed by (kind, N, M, n_theta,
    n_rho); None disables it. Default: $LPR_SPECTRUM_CACHE."""
    check(lib().lpr_spectrum_cache_dir(None if directory is None else os.fsencode(directory)))


def spectrum_cache_counters() -> tuple:
    """(reads served from the cache, spectra written to it) since load."""
    return int(lib().lpr_spectrum_cache_hits()), int(lib().lpr_spectrum_cache_stores())


def zeta_spectrum(g: Geometry, device=None) -> np.ndarray:
    """Forward-kernel spectrum, (2 nts) x n_rho complex, theta rows in FFT order
    (kernel.cpp:341-439, quadrature). device=None: host fp64 threads; an int:
    the same quadrature on that GPU (fp64)."""
    return _spectrum(g, 0, device)


def zeta_bp_spectrum(g: Geometry, device=None) -> np.ndarray:
    return _spectrum(g, 1, device)


class RadonPlan:
    """Immutable per-device plan: geometry, uploaded spectra, scratch for
    ``max_batch`` slices (larger batches run in chunks)."""

    def __init__(self, geometry: Geometry, zeta=None, zeta_bp=None, max_batch: int = 1, device: int = 0,
                 texture_gather: bool = False):
        self.geometry = geometry
        self.max_batch = int(max_batch)
        self.device = int(device)
        z = None if zeta is None else np.ascontiguousarray(zeta, dtype=np.complex128)
        zb = None if zeta_bp is None else np.ascontiguousarray(zeta_bp, dtype=np.complex128)
        for a in (z, zb):
            if a is not None and a.shape != (2 * geometry.nts, geometry.n_rho):
                raise ValueError(f"spectrum shape {a.shape} does not match the plan")
        h = ctypes.c_void_p()
        self.texture_gather = bool(texture_gather)
        check(lib().lpr_gpu_plan_create_ex(self.device, ctypes.byref(geometry),
                                           None if z is None else z.ctypes.data,
                                           None if zb is None else zb.ctypes.data,
                                           self.max_batch, 1 if texture_gather else 0, ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    @property
    def N(self) -> int:
        return self.geometry.N

    @property
    def n_theta(self) -> int:
        return self.geometry.n_theta

    def launch_count(self) -> int:
        return int(lib().lpr_gpu_launch_count(self._h))

    def fft_count(self) -> int:
        return int(lib().lpr_gpu_fft_count(self._h))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().lpr_gpu_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _run(plan: RadonPlan, x, in_shape, out_shape, dev_fn, host_fn):
    if _is_torch(x) and not x.is_cuda:
        # host tensor (pinned ones take the pipelined H2D/compute/D2H path)
        import torch

        if x.dtype != torch.float32:
            raise ValueError("expected a float32 tensor")
        single = x.dim() == 2
        xb = (x.unsqueeze(0) if single else x).contiguous()
        if tuple(xb.shape[1:]) != in_shape:
            raise ValueError(f"input shape {tuple(x.shape)} does not match the plan {in_shape}")
        out = torch.empty((xb.shape[0],) + out_shape, dtype=torch.float32, pin_memory=x.is_pinned())
        check(host_fn(plan.handle, xb.data_ptr(), out.data_ptr(), xb.shape[0]))
        return out[0] if single else out
    if _is_torch(x):
        import torch

        if x.dtype != torch.float32 or not x.is_cuda:
            raise ValueError("expected a float32 CUDA tensor")
        single = x.dim() == 2
        xb = x.unsqueeze(0) if single else x
        if tuple(xb.shape[1:]) != in_shape:
            raise ValueError(f"input shape {tuple(x.shape)} does not match the plan {in_shape}")
        xb = xb.contiguous()
        out = torch.empty((xb.shape[0],) + out_shape, dtype=torch.float32, device=xb.device)
        stream = torch.cuda.current_stream(xb.device).cuda_stream
        check(dev_fn(plan.handle, xb.data_ptr(), out.data_ptr(), xb.shape[0], ctypes.c_void_p(stream)))
        return out[0] if single else out
    a = np.asarray(x)
    single = a.ndim == 2
    ab = a[None] if single else a
    if ab.shape[1:] != in_shape:
        raise ValueError(f"input shape {a.shape} does not match the plan {in_shape}")
    ab = np.ascontiguousarray(ab, dtype=np.float32)
    out = np.empty((ab.shape[0],) + out_shape, dtype=np.float32)
    check(host_fn(plan.handle, ab.ctypes.data, out.ctypes.data, ab.shape[0]))
    return out[0] if single else out


def fast_radon(image, plan: RadonPlan):
    """Algorithm 1: image [batch x] N x N -> sinogram [batch x] n_theta x N."""
    g = plan.geometry
    return _run(plan, image, (g.N, g.N), (g.n_theta, g.N), lib().lpr_gpu_radon, lib().lpr_gpu_radon_host)


def fast_backprojection(sino, plan: RadonPlan):
    """Algorithm 2: sinogram -> image (zero outside the unit disc)."""
    g = plan.geometry
    return _run(plan, sino, (g.n_theta, g.N), (g.N, g.N), lib().lpr_gpu_backproject,
                lib().lpr_gpu_backproject_host)


def radon_backproject(image, plan: RadonPlan):
    """R then R# of the same slices in one host-buffer call (the normal
    operator of iterative reconstruction): image [batch x] N x N host array or
    CPU tensor -> (R f, R# R f), the sinograms never re-uploaded."""
    import torch

    g = plan.geometry
    x = image if _is_torch(image) else torch.as_tensor(np.ascontiguousarray(image, dtype=np.float32))
    if x.is_cuda or x.dtype != torch.float32:
        raise ValueError("expected a float32 host array or CPU tensor")
    single = x.dim() == 2
    xb = (x.unsqueeze(0) if single else x).contiguous()
    if tuple(xb.shape[1:]) != (g.N, g.N):
        raise ValueError(f"image shape {tuple(x.shape)} does not match the plan")
    pin = xb.is_pinned()
    sino = torch.empty((xb.shape[0], g.n_theta, g.N), dtype=torch.float32, pin_memory=pin)
    back = torch.empty((xb.shape[0], g.N, g.N), dtype=torch.float32, pin_memory=pin)
    check(lib().lpr_gpu_radon_backproject_host(plan.handle, xb.data_ptr(), sino.data_ptr(), back.data_ptr(),
                                               xb.shape[0]))
    if not _is_torch(image):
        sino, back = sino.numpy(), back.numpy()
    return (sino[0], back[0]) if single else (sino, back)


def radon_transpose(sino, plan: RadonPlan):
    """Exact adjoint of fast_radon under the weighted inner products of adjoint_gap."""
    g = plan.geometry
    return _run(plan, sino, (g.n_theta, g.N), (g.N, g.N), lib().lpr_gpu_radon_transpose,
                lib().lpr_gpu_radon_transpose_host)


FILTER_KINDS = {"ramp": 0, "shepp-logan": 1, "cosine": 2}


def _kind(kind: str) -> int:
    if kind not in FILTER_KINDS:
        raise ValueError(f"unknown filter kind {kind!r} (ramp, shepp-logan, cosine)")
    return FILTER_KINDS[kind]


def apply_filter(sino, plan: RadonPlan, kind: str = "ramp"):
    """FBP filter along s: per-row linear convolution with the
    discrete band-limited ramp (optionally Shepp-Logan / cosine windowed)."""
    g, k = plan.geometry, _kind(kind)
    if not (_is_torch(sino) and sino.is_cuda):
        import torch

        t = torch.as_tensor(np.ascontiguousarray(sino, dtype=np.float32), device=f"cuda:{plan.device}")
        return apply_filter(t, plan, kind).cpu().numpy()
    return _run(plan, sino, (g.n_theta, g.N), (g.n_theta, g.N),
                lambda h, i, o, b, s: lib().lpr_gpu_filter(h, k, i, o, b, s), None)


def lp_convolve(data, spectrum, plan: RadonPlan, divide_bspline: bool = True):
    """Re IFFT2(FFT2(data) * spectrum [/ Bhat]) on the doubled
    grid, data [batch x] (2 nts) x n_rho real (CUDA tensor, or host array / tensor),
    spectrum (2 nts) x n_rho complex even in k_theta (zeta / zeta#), its
    theta-Nyquist row treated as zero (as in Algorithms 1-2)."""
    g = plan.geometry
    shape = (2 * g.nts, g.n_rho)
    s = np.ascontiguousarray(spectrum, dtype=np.complex128)
    if s.shape != shape:
        raise ValueError(f"spectrum shape {s.shape} does not match the plan {shape}")
    div = int(bool(divide_bspline))
    return _run(plan, data, shape, shape,
                lambda h, i, o, b, st: lib().lpr_gpu_lp_convolve(h, s.ctypes.data, div, i, o, b, st),
                lambda h, i, o, b: lib().lpr_gpu_lp_convolve_host(h, s.ctypes.data, div, i, o, b))


def fbp(sino, plan: RadonPlan, kind: str = "ramp"):
    """Filtered back-projection: c_norm R#(filter(g)), c_norm = 1/2."""
    g, k = plan.geometry, _kind(kind)
    return _run(plan, sino, (g.n_theta, g.N), (g.N, g.N),
                lambda h, i, o, b, s: lib().lpr_gpu_fbp(h, k, i, o, b, s),
                lambda h, i, o, b: lib().lpr_gpu_fbp_host(h, k, i, o, b))


def sensitivity_image(plan: RadonPlan):
    """R# chi_C: the back-projection of the all-lines
    indicator, N x N CUDA tensor on the plan's device."""
    import torch

    g = plan.geometry
    out = torch.empty(g.N, g.N, dtype=torch.float32, device=f"cuda:{plan.device}")
    stream = torch.cuda.current_stream(out.device).cuda_stream
    check(lib().lpr_gpu_sensitivity(plan.handle, out.data_ptr(), ctypes.c_void_p(stream)))
    return out


def em_run(sino, plan: RadonPlan, iters: int, f0=None):
    """EM reconstruction, device resident:
    f <- f R#(g / max(Rf, eps)) / R# chi_C. sino: [batch x] n_theta x N float32
    CUDA tensor (g >= 0); f0: same-batch N x N start (default: 1 inside the
    unit disc). Returns (estimate, loglik) with loglik[b, k] the Poisson
    log-likelihood of iterate k + 1 of slice b."""
    import torch

    g = plan.geometry
    if not (_is_torch(sino) and sino.is_cuda and sino.dtype == torch.float32):
        raise ValueError("expected a float32 CUDA tensor")
    single = sino.dim() == 2
    gb = (sino.unsqueeze(0) if single else sino).contiguous()
    if tuple(gb.shape[1:]) != (g.n_theta, g.N):
        raise ValueError(f"sinogram shape {tuple(sino.shape)} does not match the plan")
    B = gb.shape[0]
    if f0 is None:
        f = torch.empty(B, g.N, g.N, dtype=torch.float32, device=gb.device)
        init = 1
    else:
        f = (f0.unsqueeze(0) if f0.dim() == 2 else f0).to(device=gb.device, dtype=torch.float32).contiguous().clone()
        if tuple(f.shape) != (B, g.N, g.N):
            raise ValueError("f0 shape does not match the sinogram batch")
        init = 0
    ll = np.zeros((B, max(int(iters), 0)), dtype=np.float64)
    stream = torch.cuda.current_stream(gb.device).cuda_stream
    check(lib().lpr_gpu_em(plan.handle, gb.data_ptr(), f.data_ptr(), B, int(iters), init,
                           ll.ctypes.data if iters > 0 else None, ctypes.c_void_p(stream)))
    return (f[0] if single else f), (ll[0] if single else ll)


def inner_sinogram(g: Geometry, a, b) -> float:
    """<a, b>_Sigma = 2 dtheta ds sum(a b)  (test_oracle.cpp:198-212)."""
    return float(2.0 * g.dtheta_p * g.ds * np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)))


def inner_image(g: Geometry, a, b) -> float:
    """<a, b>_X = sum(a b) / N^2."""
    return float(np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)) / (g.N * g.N))


def adjoint_gap(plan: RadonPlan, trials: int = 20, exact: bool = False, seed: int = 0) -> float:
    """max over random (f, g) of |<Rf,g> - <f,R#g>| / (|f| |g|).
    exact=True pairs R with its exact transpose instead of Algorithm 2."""
    if trials < 1:
        raise ValueError("adjoint_gap: trials must be >= 1")
    g = plan.geometry
    rng = np.random.default_rng(seed)
    worst = 0.0
    for _ in range(trials):
        f = rng.uniform(-1, 1, (g.N, g.N)).astype(np.float32)
        s = rng.uniform(-1, 1, (g.n_theta, g.N)).astype(np.float32)
        rf = fast_radon(f, plan)
        bs = radon_transpose(s, plan) if exact else fast_backprojection(s, plan)
        num = abs(inner_sinogram(g, rf, s) - inner_image(g, f, bs))
        den = np.sqrt(inner_image(g, f, f) * inner_sinogram(g, s, s))
        worst = max(worst, num / den if den > 0 else 0.0)
    return worst

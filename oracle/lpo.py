"""ORACLE — test infrastructure only.

ctypes bindings for ``oracle/liblpo.so`` (our fp64 CPU restatement of the
reference path, see ``oracle/lpo.hpp``) and, when it has been built here, for
``oracle/_ref/liblpr_ref.so`` (the reference's own geometry / bspline / kernel
/ oracle sources compiled from /root/reference). Only ``tests/``,
``__graft_entry__.smoke()`` and the CPU legs of ``bench.py`` may import this
module, and only as the checker / CPU baseline — never on the product path.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LPO_PATH = os.path.join(HERE, "liblpo.so")
REF_PATH = os.path.join(HERE, "_ref", "liblpr_ref.so")

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LPO_PATH):
            raise RuntimeError(f"oracle library missing: {LPO_PATH} (run `make -C oracle`)")
        _lib = ctypes.CDLL(LPO_PATH)
        _lib.lpo_last_error.restype = ctypes.c_char_p
        _lib.lpo_fft2d_count.restype = ctypes.c_ulonglong
        L, P, C = ctypes.c_long, ctypes.c_void_p, ctypes.c_int
        sig = {
            "lpo_prefilter_1d": [P, L],
            "lpo_prefilter_2d": [P, L, L],
            "lpo_fft1d": [P, L, C],
            "lpo_fft2d": [P, L, L, C],
            "lpo_lp_convolve": [P, C, P, L, L],
            "lpo_eval_mirror_2d": [P, L, L, P, P, P, L],
            "lpo_eval_periodic_2d": [P, L, L, P, P, P, L],
        }
        for name, args in sig.items():
            getattr(_lib, name).argtypes = args
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError(f"reference build missing: {REF_PATH} (run `make -C oracle ref`)")
        _ref = ctypes.CDLL(REF_PATH)
        _ref.lpr_ref_last_error.restype = ctypes.c_char_p
        L, P, C = ctypes.c_long, ctypes.c_void_p, ctypes.c_int
        sig = {
            "lpr_ref_prefilter_1d": [P, L],
            "lpr_ref_prefilter_2d": [P, L, L],
            "lpr_ref_interp_cubic_2d": [P, L, L, P, P, P, L],
            "lpr_ref_eval_periodic_2d": [P, L, L, P, P, P, L],
            "lpr_ref_eval_zero_1d": [P, L, P, P, L],
        }
        for name, args in sig.items():
            getattr(_ref, name).argtypes = args
    return _ref


def _check(rc: int, which="lpo"):
    if rc != 0:
        msg = (lib().lpo_last_error() if which == "lpo" else ref().lpr_ref_last_error()).decode()
        raise RuntimeError(msg)


@dataclass(frozen=True)
class Plan:
    N: int
    M: int
    n_theta: int
    nts: int
    n_rho: int
    refine: int
    beta: float
    aR: float
    ar: float
    log_ar: float
    dtheta_p: float
    dtheta_lp: float
    drho: float
    ds: float

    @property
    def key(self):
        return (self.N, self.M, self.n_theta, self.n_rho)


def make_plan(N: int, M: int = 3, n_theta: int = 0, n_rho: int = 0) -> Plan:
    iv = (ctypes.c_int * 6)()
    dv = (ctypes.c_double * 8)()
    _check(lib().lpo_plan(N, M, n_theta, n_rho, iv, dv))
    return Plan(*list(iv), *list(dv))


def spectrum(p: Plan, kind: int) -> np.ndarray:
    out = np.zeros((2 * p.nts, p.n_rho), dtype=np.complex128)
    _check(lib().lpo_spectrum(*p.key, kind, out.ctypes.data_as(_D)))
    return out


def _batched(x, shape):
    x = np.ascontiguousarray(x, dtype=np.float64)
    single = x.ndim == 2
    if single:
        x = x[None]
    assert x.shape[1:] == shape, (x.shape, shape)
    return x, single


def fast_radon(p: Plan, zeta: np.ndarray, img: np.ndarray) -> np.ndarray:
    x, single = _batched(img, (p.N, p.N))
    out = np.zeros((x.shape[0], p.n_theta, p.N))
    z = np.ascontiguousarray(zeta, dtype=np.complex128)
    _check(lib().lpo_fast_radon(*p.key, z.ctypes.data_as(_D), _ptr(x), _ptr(out), x.shape[0]))
    return out[0] if single else out


def fast_backprojection(p: Plan, zeta_bp: np.ndarray, sino: np.ndarray) -> np.ndarray:
    x, single = _batched(sino, (p.n_theta, p.N))
    out = np.zeros((x.shape[0], p.N, p.N))
    z = np.ascontiguousarray(zeta_bp, dtype=np.complex128)
    _check(lib().lpo_fast_backprojection(*p.key, z.ctypes.data_as(_D), _ptr(x), _ptr(out), x.shape[0]))
    return out[0] if single else out


def radon_transpose(p: Plan, zeta: np.ndarray, sino: np.ndarray) -> np.ndarray:
    x, single = _batched(sino, (p.n_theta, p.N))
    out = np.zeros((x.shape[0], p.N, p.N))
    z = np.ascontiguousarray(zeta, dtype=np.complex128)
    _check(lib().lpo_radon_transpose(*p.key, z.ctypes.data_as(_D), _ptr(x), _ptr(out), x.shape[0]))
    return out[0] if single else out


def radon_sector_coeffs(p: Plan, zeta: np.ndarray, qf: np.ndarray, m: int) -> np.ndarray:
    out = np.zeros((p.nts + 1, p.n_rho), dtype=np.complex128)
    z = np.ascontiguousarray(zeta, dtype=np.complex128)
    q = np.ascontiguousarray(qf, dtype=np.float64)
    _check(lib().lpo_radon_sector_coeffs(*p.key, z.ctypes.data_as(_D), _ptr(q), m, out.ctypes.data_as(_D)))
    return out


def lp_convolve(spec: np.ndarray, data: np.ndarray, divide_bspline: bool = True) -> np.ndarray:
    d = np.array(data, dtype=np.float64, order="C")
    s = np.ascontiguousarray(spec, dtype=np.complex128)
    _check(lib().lpo_lp_convolve(s.ctypes.data_as(_D), int(divide_bspline), _ptr(d), d.shape[0], d.shape[1]))
    return d


def direct_radon(p: Plan, img: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(img, dtype=np.float64)
    out = np.zeros((p.n_theta, p.N))
    _check(lib().lpo_direct_radon(*p.key, _ptr(x), _ptr(out)))
    return out


def direct_backprojection(p: Plan, sino: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(sino, dtype=np.float64)
    out = np.zeros((p.N, p.N))
    _check(lib().lpo_direct_backprojection(*p.key, _ptr(x), _ptr(out)))
    return out


def phantom_image(N: int) -> np.ndarray:
    out = np.zeros((N, N))
    _check(lib().lpo_phantom_image(N, _ptr(out)))
    return out


def phantom_sinogram(p: Plan) -> np.ndarray:
    out = np.zeros((p.n_theta, p.N))
    _check(lib().lpo_phantom_sinogram(*p.key, _ptr(out)))
    return out


def prefilter_1d(x: np.ndarray) -> np.ndarray:
    y = np.array(x, dtype=np.float64)
    _check(lib().lpo_prefilter_1d(_ptr(y), y.size))
    return y


def prefilter_2d(x: np.ndarray) -> np.ndarray:
    y = np.array(x, dtype=np.float64, order="C")
    _check(lib().lpo_prefilter_2d(_ptr(y), y.shape[0], y.shape[1]))
    return y


def eval_mirror_2d(coef: np.ndarray, tr: np.ndarray, tc: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(coef, dtype=np.float64)
    tr = np.ascontiguousarray(tr, dtype=np.float64)
    tc = np.ascontiguousarray(tc, dtype=np.float64)
    out = np.zeros(tr.size)
    _check(lib().lpo_eval_mirror_2d(_ptr(c), c.shape[0], c.shape[1], _ptr(tr), _ptr(tc), _ptr(out), tr.size))
    return out


def eval_periodic_2d(coef: np.ndarray, tr: np.ndarray, tc: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(coef, dtype=np.float64)
    tr = np.ascontiguousarray(tr, dtype=np.float64)
    tc = np.ascontiguousarray(tc, dtype=np.float64)
    out = np.zeros(tr.size)
    _check(lib().lpo_eval_periodic_2d(_ptr(c), c.shape[0], c.shape[1], _ptr(tr), _ptr(tc), _ptr(out), tr.size))
    return out


def fft2d(x: np.ndarray, sign: int) -> np.ndarray:
    y = np.array(x, dtype=np.complex128, order="C")
    _check(lib().lpo_fft2d(y.ctypes.data_as(_D), y.shape[0], y.shape[1], sign))
    return y


def fft1d(x: np.ndarray, sign: int) -> np.ndarray:
    y = np.array(x, dtype=np.complex128, order="C")
    _check(lib().lpo_fft1d(y.ctypes.data_as(_D), y.size, sign))
    return y


def fft2d_count() -> int:
    return int(lib().lpo_fft2d_count())


def fft2d_count_reset() -> None:
    lib().lpo_fft2d_count_reset()


# ----------------------------------------------------------------- FBP

FILTER_KINDS = ("ramp", "shepp-logan", "cosine")


def filter_spectrum(N: int, kind: str = "ramp") -> np.ndarray:
    """Real, even transfer function on the 2N-point DFT grid used by
    apply_filter, normalised so that filtered = IDFT(DFT(pad(g)) * H)[:N].

    The ramp is the DFT of the band-limited discrete ramp kernel (Kak &
    Slaney): h(0) = 1/(4 ds^2), h(n odd) = -1/(n pi ds)^2, h(n even) = 0,
    times ds — this is the end-point corrected |sigma| whose sigma = 0 bin is
    the trapezoid value of the discrete kernel rather than 0.
    Shepp-Logan and cosine multiply it by sinc(sigma/N) and cos(pi sigma/N)
    (the cosine variant that vanishes at sigma = N/2,
    SPEC.md:377), sigma_k = k / (2 N ds) cycles per unit length."""
    if kind not in FILTER_KINDS:
        raise ValueError(f"unknown filter kind {kind!r}")
    ds = 1.0 / N
    n = np.arange(2 * N)
    lag = np.where(n < N, n, n - 2 * N)
    h = np.zeros(2 * N)
    h[lag == 0] = 1.0 / (4 * ds * ds)
    odd = (lag % 2) != 0
    h[odd] = -1.0 / (np.pi * lag[odd] * ds) ** 2
    H = np.real(np.fft.fft(h)) * ds
    sigma = np.abs(np.where(n <= N, n, n - 2 * N)) / (2 * N * ds)
    if kind == "shepp-logan":
        H = H * np.sinc(sigma / N)
    elif kind == "cosine":
        H = H * np.cos(np.pi * sigma / N)
    return H


def apply_filter(sino: np.ndarray, kind: str = "ramp") -> np.ndarray:
    """Per-theta-row linear convolution along s with 2N zero padding
    (SPEC.md:353-361)."""
    g = np.asarray(sino, dtype=np.float64)
    N = g.shape[-1]
    H = filter_spectrum(N, kind)
    G = np.fft.fft(np.concatenate([g, np.zeros_like(g)], axis=-1), axis=-1)
    return np.real(np.fft.ifft(G * H, axis=-1))[..., :N]


# fbp = C_NORM * fast_backprojection(apply_filter(g)): R# integrates over the
# full line set (factor 2), the inversion formula over a half
# turn, so C_NORM = 1/2; checked by the disc calibration of SPEC.md:368/378.
C_NORM = 0.5


def fbp(p: Plan, zeta_bp: np.ndarray, sino: np.ndarray, kind: str = "ramp") -> np.ndarray:
    return C_NORM * fast_backprojection(p, zeta_bp, apply_filter(sino, kind))


# ----------------------------------------------------------------- EM

def disc_mask(N: int) -> np.ndarray:
    """Pixels inside the unit disc: (2c - N)^2 + (2r - N)^2 <= N^2 (the R# support)."""
    i = 2 * np.arange(N) - N
    return (i[None, :] ** 2 + i[:, None] ** 2) <= N * N


def sensitivity_image(p: Plan, zeta_bp: np.ndarray) -> np.ndarray:
    """R# chi_C, chi_C = 1 on every detector bin (|s| <= 1/2)."""
    return fast_backprojection(p, zeta_bp, np.ones((p.n_theta, p.N)))


def em_run(p: Plan, zeta: np.ndarray, zeta_bp: np.ndarray, g: np.ndarray, iters: int, f0=None):
    """em_run / em_step: f <- f R#(g / max(Rf, eps)) / R# chi_C,
    eps = 1e-6 max g (bins with Rf <= eps give ratio 0), sensitivity clamped at
    1e-6 of its max, estimate >= 0 and 0 outside the unit disc; returns the
    estimate and the Poisson log-likelihood of every iterate f^1..f^iters."""
    g = np.asarray(g, dtype=np.float64)
    mask = disc_mask(p.N)
    f = mask.astype(np.float64) if f0 is None else np.array(f0, dtype=np.float64)
    sens = sensitivity_image(p, zeta_bp)
    inv = np.where(mask, 1.0 / np.maximum(sens, 1e-6 * sens.max()), 0.0)
    eps = 1e-6 * g.max()
    hist = []
    rf = fast_radon(p, zeta, f)
    for _ in range(iters):
        q = np.where(rf > eps, g / np.where(rf > eps, rf, 1.0), 0.0)
        f = np.maximum(f * fast_backprojection(p, zeta_bp, q) * inv, 0.0)
        if not np.isfinite(f).all():
            raise FloatingPointError("em: non-finite estimate")
        rf = fast_radon(p, zeta, f)
        ok = rf > eps
        hist.append(float(np.sum(g[ok] * np.log(rf[ok]) - rf[ok])))
    return f, np.array(hist)


# ----------------------------------------------------------------- inputs

def smooth_disc_image(N: int, support_radius: float, seed: int, blur_sigma: float = 3.0) -> np.ndarray:
    """Random phantom in the style of the reference's helpers.hpp:55-112:
    Gaussian-blurred noise, cosine taper to the physical support radius,
    max-normalised. (numpy RNG, so values differ from mt19937_64.)"""
    rng = np.random.default_rng(seed)
    img = rng.standard_normal((N, N))
    half = int(np.ceil(3 * blur_sigma))
    t = np.arange(-half, half + 1)
    k = np.exp(-0.5 * t * t / blur_sigma ** 2)
    k /= k.sum()
    img = np.apply_along_axis(lambda r: np.convolve(r, k, mode="same"), 1, img)
    img = np.apply_along_axis(lambda c: np.convolve(c, k, mode="same"), 0, img)
    idx = (np.arange(N) - N // 2) / N
    rad = np.hypot(idx[None, :], idx[:, None])
    r_raster = support_radius / 2.0
    edge = 0.85 * r_raster
    w = np.where(rad < edge, 1.0, np.where(rad < r_raster, 0.5 * (1 + np.cos(np.pi * (rad - edge) / (r_raster - edge))), 0.0))
    img *= w
    return np.ascontiguousarray(img / np.abs(img).max())


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.sqrt(((a - b) ** 2).sum() / (b ** 2).sum()))


def inner_sino(p: Plan, a, b) -> float:
    return float(2.0 * p.dtheta_p * p.ds * np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)))


def inner_img(p: Plan, a, b) -> float:
    return float(np.sum(np.asarray(a, np.float64) * np.asarray(b, np.float64)) / (p.N * p.N))

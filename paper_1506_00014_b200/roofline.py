"""Algorithmic byte model of each kernel and
the per-stage profiler binding.

§8(d): each stage of Algorithms 1-2 reads its per-slice input once and writes
its output once, fp32 reals (r = 4 B) and complex64 spectra (c = 8 B); plan
constants (the multiplier tables) are excluded. With P = N^2, S = N_theta N,
L = nts N_rho (one sector's Omega_p), H = (nts + 1) N_rho (its half theta
spectrum):

  R : prefilter 2rP | gather-in rP + rML | theta-fwd rML + cMH | rho 2cMH
      | theta-inv cMH + rML | gather-out rML + rS
  R#: prefilter 2rS | gather-in rS + rML | theta-fwd rML + cMH | rho 2cMH
      | theta-inv cMH + rML | gather-out rML + rP

A kernel that fuses two stages (the gather + theta forward of both
operators) is charged the sum of its stages (`bytes`, the figure the
roofline fraction uses); `compulsory` is what that fused kernel must move at
least (its input and its output, without the Omega_p round trip it
removes). Re-reads served by L1/L2 (spline taps, FFT passes) count in
neither.
"""
from __future__ import annotations

import ctypes

from ._lib import check, lib


def _sizes(g):
    N, M, nts, nr, nt = g.N, g.M, g.nts, g.n_rho, g.n_theta
    return N * N, nt * N, nts * nr, (nts + 1) * nr, M


def stage_model(g, op: str) -> dict:
    """Per slice: {kernel stage: (§8(d) bytes, compulsory bytes)}."""
    P, S, L, H, M = _sizes(g)
    r, c = 4, 8
    if op == "radon":
        gather_in, theta_fwd = r * P + r * M * L, r * M * L + c * M * H
        return {
            "prefilter_2d": (2 * r * P, 2 * r * P),
            "radon_theta_fwd": (gather_in + theta_fwd, r * P + c * M * H),
            "rho_pass": (2 * c * M * H, 2 * c * M * H),
            "theta_inv": (c * M * H + r * M * L, c * M * H + r * M * L),
            "radon_out": (r * M * L + r * S, r * M * L + r * S),
        }
    if op == "backproject":
        gather_in, theta_fwd = r * S + r * M * L, r * M * L + c * M * H
        return {
            "prefilter_sino": (2 * r * S, 2 * r * S),
            "bp_theta_fwd": (gather_in + theta_fwd, r * S + c * M * H),
            "rho_pass": (2 * c * M * H, 2 * c * M * H),
            "theta_inv": (c * M * H + r * M * L, c * M * H + r * M * L),
            "bp_out": (r * M * L + r * P, r * M * L + r * P),
        }
    raise ValueError(op)


def stage_bytes(g, op: str, batch: int) -> dict:
    """§8(d) bytes per launch of each kernel for a batch of `batch` slices."""
    return {k: v[0] * batch for k, v in stage_model(g, op).items()}


def compulsory_bytes(g, op: str, batch: int) -> dict:
    return {k: v[1] * batch for k, v in stage_model(g, op).items()}


def slice_bytes(g, op: str) -> int:
    """§8(d) bytes of one slice through the operator (714.8 MB for R at N=2048, N_rho=4333)."""
    return sum(v[0] for v in stage_model(g, op).values())


def profile_stages(plan, op: str, d_in, d_out, batch: int, reps: int = 5) -> dict:
    """Mean CUDA-event duration (ms) of each kernel of one chunk, measured on
    the plan's stream (lpr_gpu_profile_stages)."""
    ms = (ctypes.c_double * 8)()
    names = (ctypes.c_char_p * 8)()
    ns = ctypes.c_int(0)
    check(lib().lpr_gpu_profile_stages(plan.handle, 0 if op == "radon" else 1, ctypes.c_void_p(d_in),
                                       ctypes.c_void_p(d_out), int(batch), int(reps), ms, ctypes.byref(ns),
                                       names))
    return {names[i].decode(): ms[i] for i in range(ns.value)}

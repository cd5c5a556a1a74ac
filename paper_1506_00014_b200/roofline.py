"""Algorithmic byte model of each kernel and the per-stage
profiler binding. "Algorithmic" = each stage reads its per-slice input once
and writes its output once (fp32 real / complex64 spectra); re-reads served
by L1/L2 (spline taps, FFT passes) are not counted. The spectral multiplier
table is read once per launch and shared by the whole batch."""
from __future__ import annotations

import ctypes

from ._lib import check, lib

APRON = 4


def stage_bytes(g, op: str, batch: int) -> dict:
    """Bytes per launch of each stage for a batch of `batch` slices."""
    N, M, nts, nr, nt = g.N, g.M, g.nts, g.n_rho, g.n_theta
    P = N * N
    pitch = N + 2 * APRON
    H = (nts + 1) * nr          # half theta spectrum per sector
    W = (nts + 8) * nr          # theta-inverse window per sector
    S = nt * N
    if op == "radon":
        per = {
            # quad raster + its transpose (sector 0 reads the transposed one)
            "prefilter_2d": 4 * P + 32 * pitch * pitch,
            "radon_theta_fwd": 32 * pitch * pitch + 8 * M * H,
            "rho_pass": 16 * M * H,
            "theta_inv": 8 * M * H + 4 * M * W,
            "radon_out": 4 * M * nts * nr + 4 * S,
        }
    elif op == "backproject":
        per = {
            "prefilter_sino": 8 * S,
            "bp_theta_fwd": 4 * S + 8 * M * H,
            "rho_pass": 16 * M * H,
            "theta_inv": 8 * M * H + 4 * M * W,
            "bp_out": 4 * M * W + 4 * P,
        }
    else:
        raise ValueError(op)
    out = {k: v * batch for k, v in per.items()}
    out["rho_pass"] += 8 * H  # multiplier row table, once per launch
    return out


def slice_bytes(g, op: str) -> int:
    return sum(stage_bytes(g, op, 1).values())


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

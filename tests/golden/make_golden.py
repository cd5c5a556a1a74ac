"""Generate the golden fixtures in tests/golden/ from the REFERENCE's own
compiled building blocks (oracle/_ref/liblpr_ref.so, built from
/root/reference/proj/src/{geometry,bspline,kernel,oracle}.cpp by
`make -C oracle ref`). Run here, where /root/reference exists; the fixtures
are committed so the CPU tests can pin the oracle without the reference.

    python tests/golden/make_golden.py
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import lpo  # noqa: E402

D = ctypes.POINTER(ctypes.c_double)


def ptr(a):
    return a.ctypes.data_as(D)


def main():
    r = lpo.ref()
    out = {}
    for N in (16, 32, 64):
        iv = (ctypes.c_int * 7)()
        dv = (ctypes.c_double * 8)()
        assert r.lpr_ref_plan(N, 3, 0, iv, dv) == 0
        out[f"plan_ints_{N}"] = np.array(list(iv), dtype=np.int64)
        out[f"plan_dbls_{N}"] = np.array(list(dv))
        nts, nr = iv[3], iv[4]
        for kind in (0, 1):
            s = np.zeros((2 * nts, nr), complex)
            assert r.lpr_ref_spectrum(N, 3, 0, kind, 0, s.ctypes.data_as(D), None) == 0
            out[f"spectrum_{kind}_{N}"] = s
    # closed-form spectrum at N=16 (MPFR path) for the cross-validation test
    for kind in (0, 1):
        iv = out["plan_ints_16"]
        s = np.zeros((2 * iv[3], iv[4]), complex)
        fb = ctypes.c_long(0)
        assert r.lpr_ref_spectrum(16, 3, 0, kind, 1, s.ctypes.data_as(D), ctypes.byref(fb)) == 0
        out[f"spectrum_closed_{kind}_16"] = s
    rng = np.random.default_rng(20240817)
    x = rng.uniform(-1, 1, (40, 48))
    out["prefilter_in"] = x.copy()
    y = x.copy()
    assert r.lpr_ref_prefilter_2d(ptr(y), 40, 48) == 0
    out["prefilter_out"] = y
    pts_r = rng.uniform(-1.5, 40.5, 500)
    pts_c = rng.uniform(-1.5, 48.5, 500)
    v = np.zeros(500)
    assert r.lpr_ref_interp_cubic_2d(ptr(y), 40, 48, ptr(pts_r), ptr(pts_c), ptr(v), 500) == 0
    out["interp_r"], out["interp_c"], out["interp_v"] = pts_r, pts_c, v
    N = 32
    img = lpo.smooth_disc_image(N, 0.9, 3)
    out["direct_in"] = img
    nt = int(out["plan_ints_32"][2])
    s = np.zeros((nt, N))
    assert r.lpr_ref_direct_radon(N, 3, 0, ptr(img), ptr(s)) == 0
    out["direct_radon_out"] = s
    b = np.zeros((N, N))
    assert r.lpr_ref_direct_backprojection(N, 3, 0, ptr(s), ptr(b)) == 0
    out["direct_bp_out"] = b
    ph = np.zeros((64, 64))
    assert r.lpr_ref_phantom_image(64, ptr(ph)) == 0
    out["phantom_64"] = ph
    nt64 = int(out["plan_ints_64"][2])
    ps = np.zeros((nt64, 64))
    assert r.lpr_ref_phantom_sinogram(64, 3, 0, ptr(ps)) == 0
    out["phantom_sino_64"] = ps
    np.savez_compressed(os.path.join(HERE, "reference_blocks.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_blocks.npz"), sorted(out))


if __name__ == "__main__":
    main()

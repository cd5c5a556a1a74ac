"""CPU-side checks of the drop-in boundary (include/lpradon_gpu.h):
the library loads, exports every declared entry point, and its plan-time
host code (geometry, kernel spectra) agrees with the oracle and the
reference fixtures. No compute call needs a GPU here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lpradon_gpu.h")
GOLD = os.path.join(ROOT, "tests", "golden", "reference_blocks.npz")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lpr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(lp):
    import ctypes

    from paper_1506_00014_b200 import _lib

    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), f"missing export {n}"
    # and the Python binding covers all of them
    assert set(names) <= set(_lib.EXPORTS), set(names) - set(_lib.EXPORTS)
    assert isinstance(L.lpr_gpu_last_error(), (bytes, type(None)))
    del ctypes


def test_geometry_matches_oracle(lp, lpo):
    for N, nt, nr in [(16, 0, 0), (64, 0, 0), (96, 100, 0), (512, 0, 0), (2048, 0, 0), (2048, 0, 4374),
                      (4096, 0, 0)]:
        g = lp.sampling_plan(N, 3, nt, nr)
        p = lpo.make_plan(N, 3, nt, nr)
        assert (g.N, g.M, g.n_theta, g.nts, g.n_rho, g.refine) == (p.N, p.M, p.n_theta, p.nts, p.n_rho, p.refine)
        assert g.drho == p.drho and g.dtheta_lp == p.dtheta_lp and g.a_R == p.aR


def test_smooth_n_rho(lp):
    for N in (64, 256, 512, 2048, 4096):
        g = lp.sampling_plan(N)
        n = lp.smooth_n_rho(N)
        assert n >= g.n_rho
        m = n
        for f in (2, 3, 5, 7):
            while m % f == 0:
                m //= f
        assert m == 1
    assert lp.smooth_n_rho(2048) == 4374


def test_geometry_errors_mirror_reference(lp):
    # require() -> std::invalid_argument  (types.hpp:72-74) -> ValueError
    for args in [(15, 3), (14, 3), (64, 2), (64, 3, 0, 10)]:
        with pytest.raises(ValueError):
            lp.sampling_plan(*args)


@pytest.mark.parametrize("N", [16, 32, 64])
def test_product_spectrum_matches_reference_fixture(lp, N):
    gold = np.load(GOLD)
    g = lp.sampling_plan(N)
    for kind, fn in ((0, lp.zeta_spectrum), (1, lp.zeta_bp_spectrum)):
        want = gold[f"spectrum_{kind}_{N}"]
        assert np.abs(fn(g) - want).max() <= 1e-12 * np.abs(want).max()


def test_product_spectrum_matches_oracle_n256(lp, lpo):
    g = lp.sampling_plan(256, 3, 0, lp.smooth_n_rho(256))
    p = lpo.make_plan(256, 3, 0, g.n_rho)
    assert np.abs(lp.zeta_spectrum(g) - lpo.spectrum(p, 0)).max() <= 1e-11
    assert np.abs(lp.zeta_bp_spectrum(g) - lpo.spectrum(p, 1)).max() <= 1e-11


def test_plan_creation_fails_loudly_without_gpu(lp):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        lp.RadonPlan(lp.sampling_plan(64))

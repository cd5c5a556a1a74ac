"""On-disk spectrum cache keyed by (kind, N, M, n_theta, n_rho) (
SURVEY.md §8(f)3): the second request of a spectrum reads the file, the
cached spectrum is the computed one bit for bit, a damaged file is ignored and
rewritten, and different keys do not collide."""
import os

import numpy as np
import pytest


@pytest.fixture()
def cache(lp, tmp_path):
    lp.set_spectrum_cache(str(tmp_path))
    yield tmp_path
    lp.set_spectrum_cache(None)


def test_second_request_reads_the_cache(lp, cache):
    g = lp.sampling_plan(64)
    h0, s0 = lp.spectrum_cache_counters()
    z = lp.zeta_spectrum(g)
    h1, s1 = lp.spectrum_cache_counters()
    assert (h1, s1) == (h0, s0 + 1)
    files = sorted(os.listdir(cache))
    assert files == [f"zeta0_N64_M3_T{g.n_theta}_R{g.n_rho}.lpsc"]
    assert os.path.getsize(cache / files[0]) == 40 + 16 * 2 * g.nts * g.n_rho
    z2 = lp.zeta_spectrum(g)
    assert lp.spectrum_cache_counters() == (h1 + 1, s1)
    assert np.array_equal(z, z2)
    zb = lp.zeta_bp_spectrum(g)  # a different kind is a different key
    assert lp.spectrum_cache_counters() == (h1 + 1, s1 + 1)
    assert not np.array_equal(z, zb)


def test_damaged_or_foreign_files_are_recomputed(lp, cache):
    g = lp.sampling_plan(64)
    z = lp.zeta_spectrum(g)
    path = cache / f"zeta0_N64_M3_T{g.n_theta}_R{g.n_rho}.lpsc"
    raw = path.read_bytes()
    path.write_bytes(raw[:-8])  # truncated
    h, s = lp.spectrum_cache_counters()
    assert np.array_equal(lp.zeta_spectrum(g), z)
    assert lp.spectrum_cache_counters() == (h, s + 1)  # a miss, rewritten
    assert path.read_bytes() == raw
    path.write_bytes(b"XXXX" + raw[4:])  # bad magic
    assert np.array_equal(lp.zeta_spectrum(g), z)
    assert lp.spectrum_cache_counters()[0] == h
    # another n_rho is another key
    g2 = lp.sampling_plan(64, 3, 0, g.n_rho + 1)
    assert g2.n_rho != g.n_rho
    z3 = lp.zeta_spectrum(g2)
    assert z3.shape == (2 * g2.nts, g2.n_rho)
    assert len([f for f in os.listdir(cache) if f.endswith(".lpsc")]) == 2


def test_disabled_cache_writes_nothing(lp, tmp_path):
    lp.set_spectrum_cache(None)
    h, s = lp.spectrum_cache_counters()
    lp.zeta_spectrum(lp.sampling_plan(32))
    assert lp.spectrum_cache_counters() == (h, s)
    assert os.listdir(tmp_path) == []


@pytest.mark.gpu
def test_plan_creation_reads_the_cache(lp, lpo, cache, cuda):
    """Plans created without spectra compute them on the GPU once; the second
    plan of the same key reads both from the cache and computes the same R."""
    import torch

    g = lp.sampling_plan(256)
    h, s = lp.spectrum_cache_counters()
    p1 = lp.RadonPlan(g)
    assert lp.spectrum_cache_counters() == (h, s + 2)
    p2 = lp.RadonPlan(g)
    assert lp.spectrum_cache_counters() == (h + 2, s + 2)
    f = torch.tensor(lpo.phantom_image(256), dtype=torch.float32, device=cuda)
    assert torch.equal(lp.fast_radon(f, p1), lp.fast_radon(f, p2))

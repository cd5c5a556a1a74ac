"""GPU parity: the sm_100a path through the C ABI against the fp64 oracle.

Bar (BASELINE.json north_star): relative l2 <= 1e-4 in fp32 for R and R# on
the same inputs. Inputs are the reference's two synthetic families: the
modified Shepp-Logan phantom and smooth random discs. Plans cover the
default sampling_plan (non-smooth N_rho -> Bluestein rho FFT) and the
7-smooth N_rho variant used for throughput.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _setup(lp, lpo, N, n_rho=0, max_batch=2):
    g = lp.sampling_plan(N, 3, 0, n_rho)
    p = lpo.make_plan(N, 3, 0, n_rho)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    return g, p, z, zb, lp.RadonPlan(g, z, zb, max_batch=max_batch)


def _inputs(lpo, N, n):
    f = np.stack([lpo.smooth_disc_image(N, 0.9, 11 + i) for i in range(n)])
    f[0] = lpo.phantom_image(N)
    return f


@pytest.mark.parametrize("N,smooth", [(64, False), (128, False), (256, False), (256, True), (512, False),
                                      (512, True), (1024, False), (1024, True)])
def test_radon_and_backprojection_parity(lp, lpo, cuda, N, smooth):
    import torch

    n_rho = lp.smooth_n_rho(N) if smooth else 0
    g, p, z, zb, plan = _setup(lp, lpo, N, n_rho, max_batch=2)
    f = _inputs(lpo, N, 3)  # 3 slices through a plan of 2 -> exercises chunking
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    for i in range(3):
        assert lpo.rel_l2(got[i], want[i]) <= TOL, (i, lpo.rel_l2(got[i], want[i]))
    wantb = lpo.fast_backprojection(p, zb, want)
    gotb = lp.fast_backprojection(torch.tensor(want, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    for i in range(3):
        assert lpo.rel_l2(gotb[i], wantb[i]) <= TOL, (i, lpo.rel_l2(gotb[i], wantb[i]))


def test_random_sinogram_backprojection_parity(lp, lpo, cuda):
    import torch

    N = 128
    g, p, z, zb, plan = _setup(lp, lpo, N)
    rng = np.random.default_rng(3)
    s = rng.uniform(-1, 1, (g.n_theta, N))
    want = lpo.fast_backprojection(p, zb, s)
    got = lp.fast_backprojection(torch.tensor(s, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    assert lpo.rel_l2(got, want) <= TOL


@pytest.mark.parametrize("smooth", [False, True])
def test_parity_n2048(lp, lpo, cuda, smooth):
    """Config 3 (N=2048, 3072 angles) against the oracle on one slice each way."""
    import torch

    N = 2048
    n_rho = lp.smooth_n_rho(N) if smooth else 0
    g, p, z, zb, plan = _setup(lp, lpo, N, n_rho, max_batch=1)
    f = lpo.phantom_image(N) if smooth else lpo.smooth_disc_image(N, 0.9, 5)
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    assert lpo.rel_l2(got, want) <= TOL
    wantb = lpo.fast_backprojection(p, zb, want)
    gotb = lp.fast_backprojection(torch.tensor(want, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    assert lpo.rel_l2(gotb, wantb) <= TOL


def test_host_entry_points_match_device(lp, lpo, cuda):
    import torch

    N = 128
    g, p, z, zb, plan = _setup(lp, lpo, N, max_batch=2)
    f = _inputs(lpo, N, 3).astype(np.float32)
    dev = lp.fast_radon(torch.tensor(f, device=cuda), plan).cpu().numpy()
    host = lp.fast_radon(f, plan)  # numpy -> lpr_gpu_radon_host
    np.testing.assert_array_equal(dev, host)
    devb = lp.fast_backprojection(torch.tensor(dev, device=cuda), plan).cpu().numpy()
    hostb = lp.fast_backprojection(host, plan)
    np.testing.assert_array_equal(devb, hostb)
    # pinned host tensors take the chunked three-stream pipeline
    plan4 = lp.RadonPlan(g, z, zb, max_batch=4)
    f7 = np.concatenate([f, f, f[:1]]).astype(np.float32)  # 7 slices -> chunks of 2, ragged tail
    pinned = torch.tensor(f7).pin_memory()
    piped = lp.fast_radon(pinned, plan4)
    assert piped.is_pinned()
    np.testing.assert_array_equal(piped.numpy(), lp.fast_radon(torch.tensor(f7, device=cuda), plan4).cpu().numpy())
    pipedb = lp.fast_backprojection(piped, plan4)
    np.testing.assert_array_equal(pipedb.numpy(), lp.fast_backprojection(piped.to(cuda), plan4).cpu().numpy())


def test_two_plans_on_two_host_threads(lp, lpo, cuda):
    """The bench's pipelined e2e leg: R on plan 1 and R# on plan 2 from two
    host threads at once (pinned buffers, chunked pipelines on both) give the
    same bits as the calls one after the other."""
    import threading

    import torch

    N = 256
    g, p, z, zb, plan1 = _setup(lp, lpo, N, max_batch=4)
    plan2 = lp.RadonPlan(g, z, zb, max_batch=4)
    f = torch.tensor(_inputs(lpo, N, 6).astype(np.float32)).pin_memory()
    s_ref = lp.fast_radon(f, plan1)
    b_ref = lp.fast_backprojection(s_ref, plan1)
    out = {}
    for _ in range(3):
        t = threading.Thread(target=lambda: out.__setitem__("b", lp.fast_backprojection(s_ref, plan2)))
        t.start()
        out["s"] = lp.fast_radon(f, plan1)
        t.join()
        np.testing.assert_array_equal(out["s"].numpy(), s_ref.numpy())
        np.testing.assert_array_equal(out["b"].numpy(), b_ref.numpy())
    plan2.close()


def test_zero_linearity_and_edge_cases(lp, lpo, cuda):
    import torch

    N = 64
    g, p, z, zb, plan = _setup(lp, lpo, N)
    zero = torch.zeros(N, N, device=cuda)
    assert not lp.fast_radon(zero, plan).any()
    assert not lp.fast_backprojection(torch.zeros(g.n_theta, N, device=cuda), plan).any()
    f1 = torch.tensor(lpo.smooth_disc_image(N, 0.9, 1), dtype=torch.float32, device=cuda)
    f2 = torch.tensor(lpo.smooth_disc_image(N, 0.9, 2), dtype=torch.float32, device=cuda)
    lhs = lp.fast_radon(2.5 * f1 - 1.25 * f2, plan)
    rhs = 2.5 * lp.fast_radon(f1, plan) - 1.25 * lp.fast_radon(f2, plan)
    assert float((lhs - rhs).norm() / rhs.norm()) <= 1e-5
    # empty batch is a no-op; wrong shapes raise like std::invalid_argument
    assert lp.fast_radon(torch.zeros(0, N, N, device=cuda), plan).shape == (0, g.n_theta, N)
    with pytest.raises(ValueError):
        lp.fast_radon(torch.zeros(N, N + 2, device=cuda), plan)
    with pytest.raises(ValueError):
        lp.fast_backprojection(np.zeros((g.n_theta + 1, N), np.float32), plan)
    # back-projection is zero outside the unit disc
    s = torch.rand(g.n_theta, N, device=cuda)
    img = lp.fast_backprojection(s, plan).cpu().numpy()
    x = (np.arange(N) * 2 - N)
    outside = (x[None, :] ** 2 + x[:, None] ** 2) > N * N
    assert not img[outside].any()


def test_adjoint_gap_algorithm2_gpu(lp, lpo, cuda):
    # gap <= 2e-2 at N=64 over 20 random pairs
    g, p, z, zb, plan = _setup(lp, lpo, 64)
    assert lp.adjoint_gap(plan, trials=20) <= 2e-2


def test_counters_and_no_cpu_fallback(lp, lpo, cuda):
    import torch

    g, p, z, zb, plan = _setup(lp, lpo, 64)
    l0, f0 = plan.launch_count(), plan.fft_count()
    lp.fast_radon(torch.zeros(3, 64, 64, device=cuda), plan)
    assert plan.launch_count() > l0
    assert plan.fft_count() - f0 == 2 * g.M * 3  # 2M spectral transforms per slice


def test_sinogram_of_disc_is_rotation_invariant(lp, lpo, cuda):
    """Size-independent property at N=2048: a centred disc's sinogram is the
    same on every row and matches 2 sqrt(r^2 - s^2)."""
    import torch

    N = 2048
    g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
    plan = lp.RadonPlan(g, max_batch=1)
    x = (np.arange(N) - N / 2) / N
    f = (np.hypot(x[None, :], x[:, None]) <= 0.2).astype(np.float32)
    s = lp.fast_radon(torch.tensor(f, device=cuda), plan).cpu().numpy().astype(np.float64)
    want = 2 * np.sqrt(np.clip(0.04 - x ** 2, 0, None))
    assert lpo.rel_l2(s.mean(axis=0), want) <= 5e-3
    assert np.abs(s - s.mean(axis=0)).max() <= 1e-2 * want.max()


@pytest.mark.parametrize("N", [64, 256])
def test_exact_transpose_adjoint_identity(lp, lpo, cuda, N):
    """<R f, g>_Sigma = <f, R^T g>_X to 1e-5 (north star), fp64 inner products
    of fp32 GPU outputs; and R^T itself against the oracle's transpose."""
    import torch

    g, p, z, zb, plan = _setup(lp, lpo, N)
    rng = np.random.default_rng(7)
    for trial in range(3):
        f = lpo.smooth_disc_image(N, 0.9, 100 + trial) if trial else rng.uniform(-1, 1, (N, N))
        rf = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
        s = rf.astype(np.float64) + 0.3 * rng.uniform(-1, 1, rf.shape) * np.abs(rf).max()
        rts = lp.radon_transpose(torch.tensor(s, dtype=torch.float32, device=cuda), plan).cpu().numpy()
        f32 = f.astype(np.float32).astype(np.float64)
        s32 = s.astype(np.float32).astype(np.float64)
        a = lp.inner_sinogram(g, rf, s32)
        b = lp.inner_image(g, f32, rts)
        assert abs(a - b) <= 1e-5 * abs(a), (trial, a, b)
        gap = abs(a - b) / np.sqrt(lp.inner_image(g, f32, f32) * lp.inner_sinogram(g, s32, s32))
        assert gap <= 1e-5
    want = lpo.radon_transpose(p, z, s32)
    assert lpo.rel_l2(rts, want) <= TOL


def test_adjoint_gap_exact_gpu(lp, lpo, cuda):
    g, p, z, zb, plan = _setup(lp, lpo, 64)
    assert lp.adjoint_gap(plan, trials=5, exact=True) <= 1e-5


def test_cpp_dropin_against_reference_blocks(cuda):
    """The C++ drop-in (include/lpradon/lp_ops.hpp) driven by the reference's own
    compiled sampling_plan / zeta_spectrum / direct oracles (tests/dropin)."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "paper_1506_00014_b200", "_dropin", "dropin_smoke")
    if not os.path.exists(exe):
        pytest.skip("drop-in driver not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "adjoint gap" in r.stdout


@pytest.mark.parametrize("kind", ["ramp", "shepp-logan", "cosine"])
def test_fbp_parity_n512(lp, lpo, cuda, kind):
    """Config 2 (N=512, 768 angles): the FBP filter and FBP against the oracle."""
    import torch

    N = 512
    g, p, z, zb, plan = _setup(lp, lpo, N, lp.smooth_n_rho(N))
    s = lpo.phantom_sinogram(p)
    want_f = lpo.apply_filter(s, kind)
    got_f = lp.apply_filter(torch.tensor(s, dtype=torch.float32, device=cuda), plan, kind).cpu().numpy()
    assert lpo.rel_l2(got_f, want_f) <= TOL
    want = lpo.fbp(p, zb, s, kind)
    got = lp.fbp(torch.tensor(s, dtype=torch.float32, device=cuda), plan, kind).cpu().numpy()
    assert lpo.rel_l2(got, want) <= TOL
    host = lp.fbp(s.astype(np.float32), plan, kind)
    np.testing.assert_array_equal(host, got)


def test_texture_gather_ablation(lp, lpo, cuda):
    """Config 5 ablation: hardware bilinear texture filtering in R's gather is
    measurably less accurate than the fp32 software taps (its 9-bit weights)."""
    import torch

    N = 512
    g, p, z, zb, soft = _setup(lp, lpo, N, lp.smooth_n_rho(N))
    tex = lp.RadonPlan(g, z, zb, texture_gather=True)
    f = lpo.smooth_disc_image(N, 0.9, 21)
    want = lpo.fast_radon(p, z, f)
    t = torch.tensor(f, dtype=torch.float32, device=cuda)
    e_soft = lpo.rel_l2(lp.fast_radon(t, soft).cpu().numpy(), want)
    e_tex = lpo.rel_l2(lp.fast_radon(t, tex).cpu().numpy(), want)
    assert e_soft <= TOL
    assert e_soft < e_tex <= 5e-3, (e_soft, e_tex)
    with pytest.raises(ValueError):
        lp.radon_transpose(torch.zeros(g.n_theta, N, device=cuda), tex)


def _gaussian_case(N, n_theta):
    """An off-centre Gaussian blob, its analytic line integrals and its
    analytic back-projection R# R f (x) = 2 int_0^pi Rf(theta, x.theta) dtheta
    = 2 sigma sqrt(2 pi) pi e^-a I0(a), a = |x - x0|^2 / (4 sigma^2).
    Convention: s = x1 cos(theta) + x2 sin(theta), x1 along columns."""
    from scipy.special import i0e

    x = (np.arange(N) - N / 2) / N
    X1, X2 = np.meshgrid(x, x)
    x0, sig = (0.1, -0.05), 0.05
    f = np.exp(-((X1 - x0[0]) ** 2 + (X2 - x0[1]) ** 2) / (2 * sig ** 2))
    th = np.arange(n_theta) * np.pi / n_theta
    proj = x0[0] * np.cos(th) + x0[1] * np.sin(th)
    g = sig * np.sqrt(2 * np.pi) * np.exp(-(x[None, :] - proj[:, None]) ** 2 / (2 * sig ** 2))
    a = ((X1 - x0[0]) ** 2 + (X2 - x0[1]) ** 2) / (4 * sig ** 2)
    bp = 2 * sig * np.sqrt(2 * np.pi) * np.pi * i0e(a)
    inside = X1 ** 2 + X2 ** 2 <= 0.25
    return f, g, bp, inside


@pytest.mark.parametrize("N", [2048, 4096])
def test_gaussian_analytic(lp, lpo, cuda, N):
    """R and R# of a smooth Gaussian against their closed forms at the bench
    size and at config 5 (N=4096, 6144 angles): the discretisation error of
    the method is ~1e-6 here (oracle at N=128: 2e-6), so this pins the fp32
    GPU path at full size to the 1e-4 bar without a CPU run."""
    import torch

    g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
    assert g.n_theta == 3 * N // 2
    plan = lp.RadonPlan(g, max_batch=1)
    f, sino, bp, inside = _gaussian_case(N, g.n_theta)
    s = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    assert lpo.rel_l2(s, sino) <= TOL
    b = lp.fast_backprojection(torch.tensor(sino, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    assert lpo.rel_l2(b[inside], bp[inside]) <= TOL
    assert np.abs(b[~inside]).max() == 0.0


def test_config5_n4096_disc(lp, lpo, cuda):
    """Config 5 (N=4096, 6144 angles): R of a centred disc is rotation
    invariant and matches 2 sqrt(r^2 - s^2)."""
    import torch

    N = 4096
    g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
    assert g.n_theta == 6144
    plan = lp.RadonPlan(g, max_batch=1)
    x = (np.arange(N) - N / 2) / N
    rad = np.hypot(x[None, :], x[:, None])
    f = torch.tensor((rad <= 0.2).astype(np.float32), device=cuda)
    s = lp.fast_radon(f, plan).cpu().numpy().astype(np.float64)
    want = 2 * np.sqrt(np.clip(0.04 - x ** 2, 0, None))
    assert lpo.rel_l2(s.mean(axis=0), want) <= 5e-3
    assert np.abs(s - s.mean(axis=0)).max() <= 1e-2 * want.max()


def test_fbp_reconstructs_phantom(lp, lpo, cuda):
    """FBP of the analytic Shepp-Logan sinogram at N=512 approximates the phantom
    inside the head (ramp); disc calibration gives unit interior mean."""
    import torch

    N = 512
    g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
    plan = lp.RadonPlan(g)
    p = lpo.make_plan(N, 3, 0, g.n_rho)
    x = (np.arange(N) - N / 2) / N
    rad = np.hypot(x[None, :], x[:, None])
    s = -0.5 + np.arange(N) / N
    disc = np.where(np.abs(s) < 0.25, 2 * np.sqrt(np.clip(0.0625 - s * s, 0, None)), 0.0)[None].repeat(g.n_theta, 0)
    img = lp.fbp(torch.tensor(disc, dtype=torch.float32, device=cuda), plan, "ramp").cpu().numpy()
    assert 0.98 <= img[rad < 0.2].mean() <= 1.02
    ph = lpo.phantom_image(N)
    rec = lp.fbp(torch.tensor(lpo.phantom_sinogram(p), dtype=torch.float32, device=cuda), plan, "cosine").cpu().numpy()
    inside = rad < 0.4
    assert lpo.rel_l2(rec[inside], ph[inside]) <= 0.25


@pytest.mark.parametrize("N,smooth", [(256, False), (512, True)])
def test_gpu_spectrum_matches_oracle(lp, lpo, cuda, N, smooth):
    """Plan-time spectra computed on the GPU (fp64 samples + batched fp64 FFTs)
    equal the oracle's quadrature restatement (pinned to kernel.cpp) to 1e-11
    of the DC scale, both kernels, default (Bluestein-length) and smooth plans."""
    n_rho = lp.smooth_n_rho(N) if smooth else 0
    g = lp.sampling_plan(N, 3, 0, n_rho)
    p = lpo.make_plan(N, 3, 0, g.n_rho)
    for kind, fn in ((0, lp.zeta_spectrum), (1, lp.zeta_bp_spectrum)):
        want = lpo.spectrum(p, kind)
        got = fn(g, device=0)
        assert got.shape == want.shape
        assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max(), kind


def test_em_parity_and_properties(lp, lpo, cuda):
    """Device-resident EM against the oracle's restatement
    on the same plan: 5 steps from the default start on a noisy phantom
    sinogram agree to 1e-4 (estimate and every log-likelihood); the fixed
    point holds; estimates stay >= 0 and vanish outside the unit disc."""
    import torch

    N = 64
    g = lp.sampling_plan(N)
    p = lpo.make_plan(N)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=2)
    mask = lpo.disc_mask(N)
    rng = np.random.default_rng(11)
    clean = np.clip(lpo.phantom_sinogram(p), 0, None)
    noisy = rng.poisson(100 * clean) / 100.0
    sino = torch.tensor(np.stack([noisy, clean]), dtype=torch.float32, device=cuda)
    f, ll = lp.em_run(sino, plan, 5)
    f = f.cpu().numpy()
    for i, gi in enumerate((noisy, clean)):
        want, hist = lpo.em_run(p, z, zb, gi, 5)
        assert lpo.rel_l2(f[i], want) <= 1e-4
        assert np.abs(ll[i] - hist).max() <= 1e-4 * np.abs(hist).max()
    assert (f >= 0).all() and not f[:, ~mask].any()
    sens = lp.sensitivity_image(plan).cpu().numpy()
    assert lpo.rel_l2(sens, lpo.sensitivity_image(p, zb)) <= 1e-4
    assert (sens[mask] > 0).all()
    fstar = np.abs(lpo.smooth_disc_image(N, 0.9, 3)) + 0.1 * mask
    gs = lp.fast_radon(torch.tensor(fstar, dtype=torch.float32, device=cuda), plan).clamp_min(0)  # g >= 0
    f1, _ = lp.em_run(gs, plan, 1, f0=torch.tensor(fstar, dtype=torch.float32, device=cuda))
    assert lpo.rel_l2(f1.cpu().numpy()[mask], fstar[mask]) <= 1e-2
    with pytest.raises(ValueError):
        lp.em_run(-sino, plan, 1)


@pytest.mark.parametrize("M,n_theta", [(4, 0), (5, 0), (6, 0), (3, 200)])
def test_parity_other_sector_counts_and_angles(lp, lpo, cuda, M, n_theta):
    """Sector counts other than 3 and a non-default angle count (rounded up to
    a multiple of 2M, geometry.cpp:69-98) run through the generic FFT lengths."""
    import torch

    N = 128
    g = lp.sampling_plan(N, M, n_theta)
    p = lpo.make_plan(N, M, n_theta)
    assert g.n_theta == p.n_theta and g.n_rho == p.n_rho
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=2)
    f = _inputs(lpo, N, 2)
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    wantb = lpo.fast_backprojection(p, zb, want)
    gotb = lp.fast_backprojection(torch.tensor(want, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    for i in range(2):
        assert lpo.rel_l2(got[i], want[i]) <= TOL
        assert lpo.rel_l2(gotb[i], wantb[i]) <= TOL


def test_unaligned_buffers_take_the_general_path(lp, lpo, cuda):
    """Device buffers that are not 16-byte aligned (a view one float into its
    storage) give the same result as aligned ones: the vectorised staging
    paths check alignment and fall back to scalar loads."""
    import torch

    N = 256
    g, p, z, zb, plan = _setup(lp, lpo, N)
    f = torch.tensor(_inputs(lpo, N, 1)[0], dtype=torch.float32, device=cuda)
    big = torch.zeros(N * N + 1, device=cuda)
    big[1:] = f.flatten()
    fu = big[1:].view(N, N)
    assert fu.data_ptr() % 16 != 0
    s_al, s_un = lp.fast_radon(f, plan), lp.fast_radon(fu, plan)
    assert float((s_al - s_un).abs().max()) == 0.0
    bs = torch.zeros(g.n_theta * N + 1, device=cuda)
    bs[1:] = s_al.flatten()
    su = bs[1:].view(g.n_theta, N)
    assert float((lp.fast_backprojection(s_al, plan) - lp.fast_backprojection(su, plan)).abs().max()) == 0.0


def test_radon_backproject_one_call_matches_two(lp, lpo, cuda):
    """lpr_gpu_radon_backproject_host (R then R# in one host call, the sinograms
    kept on the device for R#) returns the bits of fast_radon then
    fast_backprojection, pinned (pipelined chunks) and pageable buffers, a
    batch above max_batch."""
    import torch

    N = 256
    plan = lp.RadonPlan(lp.sampling_plan(N), max_batch=4)
    f = _inputs(lpo, N, 7).astype(np.float32)
    s_ref = lp.fast_radon(f, plan)
    b_ref = lp.fast_backprojection(s_ref, plan)
    s1, b1 = lp.radon_backproject(f, plan)
    np.testing.assert_array_equal(s1, s_ref)
    np.testing.assert_array_equal(b1, b_ref)
    fp = torch.tensor(f).pin_memory()
    s2, b2 = lp.radon_backproject(fp, plan)
    np.testing.assert_array_equal(s2.numpy(), s_ref)
    np.testing.assert_array_equal(b2.numpy(), b_ref)


@pytest.mark.parametrize("N", [96, 100, 250, 1536])
def test_parity_sizes_off_the_power_of_two_grid(lp, lpo, cuda, N):
    """Image sizes that are not powers of two (even: sampling_plan requires it, geometry.cpp; raster pitch, prefilter
    tiles, spline aprons and the R / R# kernels' edge handling), against the
    oracle on the reference's own plan."""
    import torch

    g = lp.sampling_plan(N)
    p = lpo.make_plan(N)
    assert (g.n_theta, g.n_rho) == (p.n_theta, p.n_rho)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=2)
    f = _inputs(lpo, N, 3)
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    wantb = lpo.fast_backprojection(p, zb, want)
    gotb = lp.fast_backprojection(torch.tensor(want, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    for i in range(3):
        assert lpo.rel_l2(got[i], want[i]) <= TOL, (i, lpo.rel_l2(got[i], want[i]))
        assert lpo.rel_l2(gotb[i], wantb[i]) <= TOL, (i, lpo.rel_l2(gotb[i], wantb[i]))


def test_parity_n3072_reference_plan(lp, lpo, cuda):
    """N=3072 on the reference's own plan (N_rho = 6499 = 67 * 97): the rho
    convolution padded over 13122 = 2 * 3^8 through the runtime Stockham with
    the multiplier read from L2 (the padded row alone takes 210 KB of shared
    memory); one slice each way against the oracle."""
    import torch

    N = 3072
    g = lp.sampling_plan(N)
    assert g.n_rho == 6499
    p = lpo.make_plan(N)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=1)
    f = lpo.smooth_disc_image(N, 0.9, 3072)
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    wantb = lpo.fast_backprojection(p, zb, want)
    gotb = lp.fast_backprojection(torch.tensor(want, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    er, eb = lpo.rel_l2(got, want), lpo.rel_l2(gotb, wantb)
    print(f"N=3072 n_rho=6499: R rel_l2 {er:.3e}, R# rel_l2 {eb:.3e}")
    assert er <= TOL and eb <= TOL

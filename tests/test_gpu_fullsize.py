"""GPU parity at the bench configuration and at config 5.

The bench runs N=2048, 3072 angles, 16 slices per launch. Here the same
kernels run at that batch (max_batch=16) on a 17-slice stack, so the batch is
cut into a full chunk and a ragged 1-slice tail, the R output kernel sees
blocks with fewer than kOutSlices slices, and every blockIdx.z of the
N=2048 specialisations is exercised. Slices 0, 7 and 16 are compared with
the fp64 oracle (tests/ only; the checker, never the thing measured), for the
bench's 7-smooth plan (N_rho=4374) and the reference's default plan
(N_rho=4333). The measured relative l2 errors are printed (pytest -s).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4
CHECK = (0, 7, 16)


def _stack(lpo, N, n):
    f = np.stack([lpo.smooth_disc_image(N, 0.9, 0x5EED + i) for i in range(n)])
    f[0] = lpo.phantom_image(N)
    return f


@pytest.mark.parametrize("smooth", [True, False])
def test_bench_config_parity_batch17(lp, lpo, cuda, smooth):
    import torch

    N = 2048
    n_rho = lp.smooth_n_rho(N) if smooth else 0
    g = lp.sampling_plan(N, 3, 0, n_rho)
    assert (g.n_theta, g.n_rho) == (3072, 4374 if smooth else 4333)
    p = lpo.make_plan(N, 3, 0, n_rho)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=16)
    f = _stack(lpo, N, 17)
    sino = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan)
    back = lp.fast_backprojection(sino, plan).cpu().numpy()
    sino = sino.cpu().numpy()
    want = lpo.fast_radon(p, z, f[list(CHECK)])
    wantb = lpo.fast_backprojection(p, zb, sino[list(CHECK)].astype(np.float64))
    for j, i in enumerate(CHECK):
        er, eb = lpo.rel_l2(sino[i], want[j]), lpo.rel_l2(back[i], wantb[j])
        print(f"N=2048 n_rho={g.n_rho} slice {i}: R rel_l2 {er:.3e}, R# rel_l2 {eb:.3e}")
        assert er <= TOL and eb <= TOL, (i, er, eb)
    # the chunking is invisible: slice 16 alone through the same plan gives the same bits
    alone = lp.fast_radon(torch.tensor(f[16:], dtype=torch.float32, device=cuda), plan).cpu().numpy()
    np.testing.assert_array_equal(alone[0], sino[16])


def test_exact_transpose_identity_n2048(lp, lpo, cuda):
    """<R f, g>_Sigma = <f, R^T g>_X to 1e-5 at the bench size (fp64 inner
    products of the fp32 GPU outputs; R^T's fine-grid scatter uses fp32
    atomics, 16 per fine sample)."""
    import torch

    N = 2048
    g = lp.sampling_plan(N, 3, 0, lp.smooth_n_rho(N))
    plan = lp.RadonPlan(g, max_batch=2)
    rng = np.random.default_rng(11)
    f = np.stack([lpo.smooth_disc_image(N, 0.9, 3), rng.uniform(-1, 1, (N, N))])
    rf = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    s = (rf + 0.3 * rng.uniform(-1, 1, rf.shape) * np.abs(rf).max()).astype(np.float32)
    rts = lp.radon_transpose(torch.tensor(s, device=cuda), plan).cpu().numpy()
    f32 = f.astype(np.float32).astype(np.float64)
    for i in range(2):
        a = lp.inner_sinogram(g, rf[i], s[i])
        b = lp.inner_image(g, f32[i], rts[i])
        gap = abs(a - b) / np.sqrt(lp.inner_image(g, f32[i], f32[i]) * lp.inner_sinogram(g, s[i], s[i]))
        print(f"N=2048 R^T slice {i}: |<Rf,g>-<f,R^T g>| / |<Rf,g>| = {abs(a - b) / abs(a):.3e}, gap {gap:.3e}")
        assert abs(a - b) <= 1e-5 * abs(a) and gap <= 1e-5, (i, a, b, gap)


@pytest.mark.parametrize("smooth", [True, False])
def test_config5_n4096_against_oracle(lp, lpo, cuda, smooth):
    """Config 5 (N=4096, 6144 angles): one slice each way against the oracle,
    on the 7-smooth plan (N_rho=8748) and on the reference's own
    sampling_plan(4096, 3) (N_rho=8666 = 2 * 7 * 619, whose rho convolution
    runs zero-padded over 17496 = 2^3 3^7, geometry.cpp:85-88)."""
    import torch

    N = 4096
    n_rho = lp.smooth_n_rho(N) if smooth else 0
    g = lp.sampling_plan(N, 3, 0, n_rho)
    assert g.n_rho == (8748 if smooth else 8666)
    p = lpo.make_plan(N, 3, 0, n_rho)
    z, zb = lpo.spectrum(p, 0), lpo.spectrum(p, 1)
    plan = lp.RadonPlan(g, z, zb, max_batch=1)
    f = lpo.smooth_disc_image(N, 0.9, 4096)
    want = lpo.fast_radon(p, z, f)
    got = lp.fast_radon(torch.tensor(f, dtype=torch.float32, device=cuda), plan).cpu().numpy()
    er = lpo.rel_l2(got, want)
    wantb = lpo.fast_backprojection(p, zb, got.astype(np.float64))
    gotb = lp.fast_backprojection(torch.tensor(got, device=cuda), plan).cpu().numpy()
    eb = lpo.rel_l2(gotb, wantb)
    print(f"N=4096 n_rho={g.n_rho}: R rel_l2 {er:.3e}, R# rel_l2 {eb:.3e}")
    assert er <= TOL and eb <= TOL, (er, eb)


def test_mixed_device_and_host_calls_share_a_plan(lp, lpo, cuda):
    """a device call on the caller's stream followed at once by a
    host-buffer call (the plan's own stream) on the same plan, with no sync in
    between, must not race on the plan's scratch; and two host threads sharing
    one plan are serialised."""
    import threading

    import torch

    N = 256
    g = lp.sampling_plan(N)
    plan = lp.RadonPlan(g, max_batch=4)
    f = _stack(lpo, N, 4).astype(np.float32)
    f2 = f[::-1].copy()
    ref1 = lp.fast_radon(f, plan)
    ref2 = lp.fast_radon(f2, plan)
    side = torch.cuda.Stream()
    for _ in range(5):
        with torch.cuda.stream(side):
            dev = lp.fast_radon(torch.tensor(f, device=cuda), plan)  # enqueued, not synced
        host = lp.fast_radon(f2, plan)  # numpy: plan stream
        side.synchronize()
        np.testing.assert_array_equal(dev.cpu().numpy(), ref1)
        np.testing.assert_array_equal(host, ref2)
    out = {}

    def worker(k, x):
        out[k] = [lp.fast_radon(x, plan) for _ in range(3)]

    th = [threading.Thread(target=worker, args=(k, x)) for k, x in ((0, f), (1, f2))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for r in out[0]:
        np.testing.assert_array_equal(r, ref1)
    for r in out[1]:
        np.testing.assert_array_equal(r, ref2)

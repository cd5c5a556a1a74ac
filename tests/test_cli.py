"""The C++ CLI and LPT1 codec (csrc/cli, include/lpradon/lpt1.hpp; SPEC.md:524-556;
SURVEY.md §8(f)4): byte-identical round trips, byte identity with the Python
mirror (paper_1506_00014_b200/lpt1.py), the four distinct container errors,
usage errors, and on the GPU the file pipelines radon -> fbp / backproject /
em and the bench report."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1506_00014_b200 import lpt1

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1506_00014_b200", "bin", "lpradon")


@pytest.fixture(scope="module")
def cli():
    if not os.path.exists(CLI):
        from paper_1506_00014_b200 import build

        build.build()
    return CLI


def run(cli, *args, ok=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)
    if ok:
        assert r.returncode == 0, r.stderr
    return r


def test_phantom_matches_reference_definition_and_python_bytes(cli, lpo, tmp_path):
    out = tmp_path / "p.lpt"
    run(cli, "phantom", "--size", 64, "--out", out)
    raw = out.read_bytes()
    c = lpt1.read_container(out)
    assert c.kind == "image" and c.data.shape == (64, 64) and c.meta == {"phantom": "shepp-logan"}
    assert c.grid == lpt1.image_grid(64)
    assert len(raw) == 8 + int.from_bytes(raw[4:8], "little") + 4 * 64 * 64  # SPEC example: 4 N^2 payload bytes
    assert lpt1.encode(c) == raw  # the C++ header bytes are Python's json.dumps(sort_keys=True) bytes
    np.testing.assert_array_equal(c.data, lpo.phantom_image(64).astype(np.float32))


def test_python_containers_roundtrip_byte_identical_through_cpp(cli, tmp_path):
    rng = np.random.default_rng(3)
    cases = [
        lpt1.Container("image", rng.standard_normal((17, 33)).astype(np.float32), lpt1.image_grid(33),
                       {"seed": 3, "tiny": 1e-05, "big": 1.5e16, "neg": -0.0, "pi": np.pi, "flag": True,
                        "none": None, "list": [1, 2.5, "x"], "text": "µ-ray \"quoted\"\n\ttab", "e": 1e22}),
        lpt1.Container("sinogram", rng.standard_normal((96, 64)).astype(np.float32), lpt1.sinogram_grid(96, 64)),
        lpt1.Container("spectrum", (rng.standard_normal((8, 5)) + 1j * rng.standard_normal((8, 5))).astype(np.complex64)),
        lpt1.Container("image", np.zeros((0, 4), np.float32)),
    ]
    for k, c in enumerate(cases):
        a, b = tmp_path / f"a{k}.lpt", tmp_path / f"b{k}.lpt"
        lpt1.write_container(a, c)
        r = run(cli, "inspect", "--in", a, "--out", b)
        assert b.read_bytes() == a.read_bytes(), k
        hdr = json.loads(r.stdout)
        assert (hdr["kind"], hdr["rows"], hdr["cols"]) == (c.kind, *c.data.shape)


def test_distinct_container_errors(cli, tmp_path):
    good = lpt1.encode(lpt1.Container("image", np.zeros((64, 64), np.float32), lpt1.image_grid(64)))
    hdr = b'{"kind":"volume","rows":1,"cols":1,"dtype":"f32"}'
    bad = {
        "magic": (b"LPT2" + good[4:], 3, "BadMagicError"),
        "truncated": (good[:-3], 4, "TruncatedError"),
        "short": (good[:6], 4, "TruncatedError"),
        "rows": (good[:-4 * 64], 5, "ShapeError"),  # header says 64 x 64, payload holds 63 rows
        "long": (good + b"\0" * 4, 5, "ShapeError"),
        "schema": (b"LPT1" + len(hdr).to_bytes(4, "little") + hdr + b"\0" * 4, 6, "SchemaError"),
        "notjson": (b"LPT1" + (3).to_bytes(4, "little") + b"\xff\xfe{", 6, "SchemaError"),
    }
    for name, (blob, code, cls) in bad.items():
        f = tmp_path / f"{name}.lpt"
        f.write_bytes(blob)
        r = run(cli, "inspect", "--in", f, ok=False)
        assert r.returncode == code and cls in r.stderr, (name, r.returncode, r.stderr)


def test_usage_errors_exit_2(cli, tmp_path):
    assert run(cli, ok=False).returncode == 2
    r = run(cli, "transmogrify", ok=False)
    assert r.returncode == 2 and "usage:" in r.stderr
    r = run(cli, "phantom", "--size", 8, "--colour", "red", ok=False)
    assert r.returncode == 2 and "unknown flag --colour" in r.stderr
    r = run(cli, "phantom", "--out", tmp_path / "x.lpt", ok=False)
    assert r.returncode == 2 and "missing --size" in r.stderr


def test_kernel_dump_is_the_quadrature_spectrum(cli, lp, tmp_path):
    for kind, fn in (("radon", lp.zeta_spectrum), ("backprojection", lp.zeta_bp_spectrum)):
        out = tmp_path / f"{kind}.lpt"
        run(cli, "kernel-dump", "--size", 32, "--sectors", 3, "--kind", kind, "--out", out)
        c = lpt1.read_container(out)
        g = lp.sampling_plan(32)
        assert c.kind == "spectrum" and c.dtype == "c32" and c.data.shape == (2 * g.nts, g.n_rho)
        np.testing.assert_array_equal(c.data, fn(g).astype(np.complex64))
        assert c.meta["kernel"] == kind and c.meta["n_rho"] == g.n_rho


@pytest.mark.gpu
def test_file_pipelines_match_the_library(cli, lp, lpo, cuda, tmp_path):
    """phantom -> radon -> {backproject, fbp cosine, em} through files equals the
    library calls on the same arrays, bit for bit, and reruns are identical."""
    N = 128
    p, s = tmp_path / "p.lpt", tmp_path / "s.lpt"
    run(cli, "phantom", "--size", N, "--out", p)
    run(cli, "radon", "--in", p, "--sectors", 3, "--out", s)
    f = lpt1.read_container(p).data
    g = lp.sampling_plan(N)
    plan = lp.RadonPlan(g)
    sino = lp.fast_radon(f, plan)
    sc = lpt1.read_container(s)
    assert sc.kind == "sinogram" and sc.grid == lpt1.sinogram_grid(g.n_theta, N)
    np.testing.assert_array_equal(sc.data, sino)
    for sub, extra, want in (("backproject", (), lp.fast_backprojection(sino, plan)),
                             ("fbp", ("--filter", "cosine"), lp.fbp(sino, plan, "cosine"))):
        o = tmp_path / f"{sub}.lpt"
        run(cli, sub, "--in", s, *extra, "--out", o)
        np.testing.assert_array_equal(lpt1.read_container(o).data, want)
    # FBP quality of the pipeline (SPEC.md:549 example): cosine FBP of the phantom's sinogram
    rec = lpt1.read_container(tmp_path / "fbp.lpt").data
    inside = np.add.outer((np.arange(N) - N / 2) ** 2, (np.arange(N) - N / 2) ** 2) < (0.45 * N) ** 2
    assert np.linalg.norm((rec - f)[inside]) / np.linalg.norm(f[inside]) < 0.3
    # EM needs g >= 0: the clipped sinogram; a negative one is refused
    r = run(cli, "em", "--in", s, "--iters", 3, "--out", tmp_path / "bad.lpt", ok=False)
    assert r.returncode == 1 and "nonnegative" in r.stderr
    sp = tmp_path / "s_pos.lpt"
    lpt1.write_container(sp, lpt1.Container("sinogram", np.maximum(sc.data, 0), sc.grid, sc.meta))
    e1, e2 = tmp_path / "e1.lpt", tmp_path / "e2.lpt"
    run(cli, "em", "--in", sp, "--iters", 3, "--out", e1)
    run(cli, "em", "--in", sp, "--iters", 3, "--seed", 7, "--out", e2)
    c1, c2 = lpt1.read_container(e1), lpt1.read_container(e2)
    np.testing.assert_array_equal(c1.data, c2.data)  # deterministic
    ll = c1.meta["loglik"]
    assert len(ll) == 3 and ll[2] >= ll[0]
    # a rerun of the same command gives the same file
    s2 = tmp_path / "s2.lpt"
    run(cli, "radon", "--in", p, "--sectors", 3, "--out", s2)
    assert s2.read_bytes() == s.read_bytes()


@pytest.mark.gpu
def test_bench_report(cli, tmp_path, cuda):
    out = tmp_path / "b.json"
    run(cli, "bench", "--sizes", "128,256,512", "--json", out, "--reps", 3)
    rep = json.loads(out.read_text())
    sizes = rep["sizes"]
    assert [r["N"] for r in sizes] == [128, 256, 512]
    assert all(r["fft_count_per_transform"] == 2 * 3 for r in sizes)  # 2M
    dev = [sum(r["stages_ms"]["radon"].values()) for r in sizes]
    assert dev[0] < dev[1] < dev[2], dev  # device time grows with N
    assert set(sizes[0]["stages_ms"]["radon"]) >= {"prefilter_2d", "rho_pass", "theta_inv", "radon_out"}


@pytest.mark.gpu
def test_calibrate_cnorm(cli, cuda):
    """tools/calibrate_cnorm: FBP of the analytic disc sinogram at
    N=256 has interior mean 1 to 5 % with the built-in c_norm = 1/2."""
    r = run(cli, "calibrate-cnorm", "--size", 256)
    rep = json.loads(r.stdout)
    assert rep["within_spec"] and abs(rep["c_norm_calibrated"] - 0.5) <= 0.025, rep

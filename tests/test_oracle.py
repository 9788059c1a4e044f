"""CPU: pin the oracle before trusting it (no GPU needed).

1. The Eigen-free restatement (oracle/liboracle.so) equals the reference's own
   fastsum.cpp compiled by path (oracle/_ref/libref.so) and the committed
   golden fixtures made by it (tests/golden/make_golden.py).
2. The exact DFT used by both (the FFTW shim) agrees with numpy.fft.
3. The reference's own known-answer / tolerance tests for this path
   (P:tests/test_fastsum.cpp and acceptance criterion 3,
   P:tests/acceptance.cpp:195-226) hold for the oracle.
"""
import glob
import os

import numpy as np
import pytest

import oracle

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "ref_*.npz")))


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- 1. pins ---
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_reference_golden(oracle_lib, path):
    g = np.load(path)
    if str(g["kind"]) == "plan":
        p = oracle_lib.plan(g["points"], float(g["ell"]), int(g["N"]), int(g["m"]), int(g["sigma"]),
                            float(g["rT"]), float(g["fit"]))
        y = p.apply(g["v"])
        assert p.scaled_length() == float(g["scaled_length"])
        assert p.coefficient_sum() == pytest.approx(float(g["coefficient_sum"]), rel=1e-15)
        if "targets" in g:
            assert rel(p.apply_cross(g["targets"], g["v"]), g["y_cross"]) <= 1e-14
    else:
        sizes, flat = list(g["win_sizes"]), list(g["win_features"])
        wins, off = [], 0
        for s in sizes:
            wins.append(flat[off:off + s])
            off += s
        op = oracle_lib.anova(g["points"], wins, list(g["weights"]), list(g["ells"]), int(g["N"]),
                              int(g["m"]), int(g["sigma"]), float(g["rT"]), float(g["fit"]))
        y = op.apply(g["v"])
        assert op.entry(3, 8) == pytest.approx(float(g["entry_3_8"]), rel=1e-15)
    # same FFT and the same arithmetic order: agreement to a few ulp
    assert rel(y, g["y"]) <= 1e-14


def test_oracle_bit_identical_to_reference_build(oracle_lib, ref_lib):
    pts = oracle.random_points(700, 3, 91)
    v = oracle.random_vector(700, 92)
    a = oracle_lib.plan(pts).apply(v)
    b = ref_lib.plan(pts).apply(v)
    assert np.array_equal(a, b)
    w = [[0, 1], [2, 3, 4], [5]]
    pts = oracle.random_points(500, 6, 93)
    v = oracle.random_vector(500, 94)
    assert np.array_equal(oracle_lib.anova(pts, w, fit=1 / 1.2).apply(v),
                          ref_lib.anova(pts, w, fit=1 / 1.2).apply(v))


# ------------------------------------------------------------ 2. the DFT ---
@pytest.mark.parametrize("shape", [(64,), (32, 32), (16, 16, 16), (6, 10, 7), (24, 8), (5,)])
@pytest.mark.parametrize("sign", [-1, 1])
def test_fftw_shim_matches_numpy(oracle_lib, shape, sign):
    rng = np.random.default_rng(sum(shape) + sign)
    x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    ref = np.fft.fftn(x) if sign == -1 else np.fft.ifftn(x) * x.size
    assert np.abs(oracle.fft(x, sign) - ref).max() <= 1e-13 * np.abs(ref).max()


# ---------------------------- 3. reference known-answer tests (oracle) ---
def test_config_validation(oracle_lib):
    # P:tests/test_fastsum.cpp:29-40
    pts = oracle.random_points(10, 1, 1)
    for kw in (dict(N=15), dict(torus_radius=0.3), dict(m=1), dict(m=9), dict(sigma=0)):
        with pytest.raises(oracle.OracleError) as e:
            oracle_lib.plan(pts, **kw)
        assert e.value.code == 4


def test_evenness(oracle_lib):
    # P:tests/test_fastsum.cpp:42-56
    p = oracle_lib.plan(np.array([[-1.0], [0.0], [1.0]]), 0.5, N=16)
    f = p.apply_cross(np.array([[-0.5], [0.5]]), np.array([0.0, 1.0, 0.0]))
    assert f[0] == pytest.approx(f[1], rel=1e-12)


def test_coefficient_sum_and_scaled_length(oracle_lib):
    # P:tests/test_fastsum.cpp:58-67
    pts = (-1.0 + 0.2 * np.arange(11))[:, None]
    p = oracle_lib.plan(pts, 0.4)
    assert p.scaled_length() == pytest.approx(0.1, rel=1e-12)
    assert p.coefficient_sum() == pytest.approx(1.0, rel=1e-6)


def test_scaling_map_inside_ball(oracle_lib):
    # P:tests/test_fastsum.cpp:69-82
    pts = oracle.random_points(300, 3, 21, 4.0)
    s = oracle_lib.plan(pts).scale_points(pts)
    assert np.all(np.linalg.norm(s, axis=1) <= 0.25 * (1 + 1e-12))
    s = oracle_lib.plan(pts, fit=0.8).scale_points(pts)
    assert np.all(np.linalg.norm(s, axis=1) <= 0.8 * 0.25 * (1 + 1e-12))


def test_zero_and_dense_accuracy(oracle_lib):
    # P:tests/test_fastsum.cpp:84-106
    p = oracle_lib.plan(oracle.random_points(50, 2, 1))
    assert np.linalg.norm(p.apply(np.zeros(50))) == 0.0
    pts = oracle.random_points(500, 2, 31)
    v = oracle.random_vector(500, 32)
    ex = oracle.dense_gaussian(pts) @ v
    assert np.linalg.norm(oracle_lib.plan(pts).apply(v) - ex) <= 1e-4 * np.linalg.norm(ex)
    pts = oracle.random_points(200, 1, 41)
    e = np.zeros(200)
    e[17] = 1.0
    col = oracle.dense_gaussian(pts)[:, 17]
    assert np.abs(oracle_lib.plan(pts).apply(e) - col).max() <= 1e-4


def test_cross_transform(oracle_lib):
    # P:tests/test_fastsum.cpp:108-145
    pts = oracle.random_points(300, 2, 51)
    p = oracle_lib.plan(pts)
    v = oracle.random_vector(300, 52)
    assert np.abs(p.apply(v) - p.apply_cross(pts, v)).max() <= 1e-12
    e = np.zeros(300)
    e[42] = 1.0
    assert p.apply_cross(pts[42:43], e)[0] == pytest.approx(1.0, rel=1e-4)
    tg = oracle.random_points(100, 2, 53, 0.5)
    C = np.exp(-((tg[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    ex = C @ v
    assert np.linalg.norm(p.apply_cross(tg, v) - ex) <= 1e-4 * np.linalg.norm(ex)
    with pytest.raises(oracle.OracleError) as err:
        p.apply_cross(np.array([[1e3, 1e3]]), v)
    assert err.value.code == 2


def test_anova_operator(oracle_lib):
    # P:tests/test_fastsum.cpp:147-194
    pts = oracle.random_points(1000, 6, 61)
    v = oracle.random_vector(1000, 62)
    wins, eta, ell = [[0, 1, 2], [3, 4, 5]], [0.5, 0.5], [1.0, 1.3]
    op = oracle_lib.anova(pts, wins, eta, ell)
    K = sum(e * oracle.dense_gaussian(pts[:, w], l) for w, e, l in zip(wins, eta, ell))
    kv = K @ v
    y = op.apply(v)
    assert np.linalg.norm(y - kv) <= 1e-4 * np.linalg.norm(kv)
    one = oracle_lib.anova(pts, [[0, 1, 2]], [0.7], [1.0])
    direct = 0.7 * oracle_lib.plan(pts[:, :3]).apply(v)
    assert np.abs(one.apply(v) - direct).max() <= 1e-12
    w2 = oracle.random_vector(1000, 63)
    assert np.linalg.norm(op.apply(v + w2) - (y + op.apply(w2))) <= 1e-12 * np.linalg.norm(y + op.apply(w2))
    u = oracle.random_vector(1000, 64)
    assert abs(u @ y - op.apply(u) @ v) <= 1e-8 * np.linalg.norm(u) * np.linalg.norm(v)
    assert op.entry(3, 8) == pytest.approx(K[3, 8], rel=1e-14)


def test_error_decreases_with_bandwidth(oracle_lib):
    # P:tests/test_fastsum.cpp:196-206 and acceptance criterion 3 (:195-226, n reduced)
    for d, seed, n in ((2, 71, 400), (1, 201, 600), (3, 203, 600)):
        pts = oracle.random_points(n, d, seed)
        v = oracle.random_vector(n, 14)
        ex = oracle.dense_gaussian(pts) @ v
        prev = np.inf
        for N in (8, 16, 32):
            err = np.linalg.norm(oracle_lib.plan(pts, N=N).apply(v) - ex) / np.linalg.norm(ex)
            assert err < prev
            prev = err
        assert prev <= 1e-4


def test_plan_reuse_and_rejects(oracle_lib):
    # P:tests/test_fastsum.cpp:208-234
    p = oracle_lib.plan(oracle.random_points(200, 2, 81))
    v = oracle.random_vector(200, 82)
    assert np.array_equal(p.apply(v), p.apply(v))
    with pytest.raises(oracle.OracleError):
        oracle_lib.plan(oracle.random_points(10, 4, 1))
    with pytest.raises(oracle.OracleError):
        oracle_lib.plan(np.zeros((0, 2)))
    oracle_lib.plan(np.zeros((5, 2)))  # degenerate identical points are allowed

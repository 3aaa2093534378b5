"""BASELINE config 2 matrix-layer extras (paper_1902_04303_b200/matrix_ext.py) on the GPU.

These operations have no reference counterpart (SURVEY §0 reconciliation table), so parity
is unpinned: each decrypted result is checked against a float64 replay of the same
approximate computation, within CKKS noise at scale 2^45 (tolerances written per test).
Config-2 shapes: X 245 x 5 with N(0,1) entries (intercept column of ones), 5 x 5 matrices,
W diagonal in (0, 0.25)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_1902_04303_b200 as hg

    params = hg.CkksParams(log_n=12, log_l=1700, log_p=45, log_p_small=30, h=64)
    sk, pk, evk, rot = hg.keygen(params, seed=11)
    eng = hg.HeEngine(params, evk, rot)
    rs = np.random.default_rng(5)
    x = rs.standard_normal((245, 5))
    x[:, 0] = 1.0
    w = rs.uniform(0.0, 0.25, 245)
    return dict(hg=hg, params=params, sk=sk, pk=pk, eng=eng, x=x, w=w, rng=random.Random(3))


def _dec(env, ct, n):
    return env["hg"].decrypt_values(ct, env["sk"])[:n]


def test_row_major_pack_roundtrip(env):
    from paper_1902_04303_b200.matrix_ext import pack_row_major, unpack_row_major

    m = pack_row_major(env["x"], env["pk"], env["params"], env["rng"])
    assert m.stride == 8
    assert np.max(np.abs(unpack_row_major(m, env["sk"]) - env["x"])) < 1e-7


def test_diag_matvec_rectangular_encrypted(env):
    """X beta (245 x 5 padded to 256 x 8) by the diagonal method with encrypted diagonals."""
    from paper_1902_04303_b200.matrix_ext import diag_matvec, pack_diagonals, periodic_vector

    hg, params = env["hg"], env["params"]
    beta = np.random.default_rng(1).standard_normal(5)
    diags, period = pack_diagonals(env["x"], env["pk"], params, env["rng"])
    assert period == 8 and len(diags) == 8
    v = hg.encrypt_values(periodic_vector(beta, period, params.slot_count), params.log_p, env["pk"],
                          params, env["rng"])
    y = diag_matvec(env["eng"], diags, v)
    got = hg.decrypt_values(y, env["sk"]).real
    want = env["x"] @ beta
    assert np.max(np.abs(got[:245] - want)) < 1e-5
    assert np.max(np.abs(got[256:256 + 245] - want)) < 1e-5   # 256-periodic output


def test_diag_matvec_plain_square(env):
    from paper_1902_04303_b200.matrix_ext import diag_matvec_plain, periodic_vector

    hg, params = env["hg"], env["params"]
    a = np.random.default_rng(2).standard_normal((5, 5))
    v0 = np.random.default_rng(3).standard_normal(5)
    v = hg.encrypt_values(periodic_vector(v0, 8, params.slot_count), params.log_p, env["pk"], params,
                          env["rng"])
    y = diag_matvec_plain(env["eng"], a, v)
    got = hg.decrypt_values(y, env["sk"]).real
    assert np.max(np.abs(got[:5] - a @ v0)) < 1e-5
    assert np.max(np.abs(got[8:13] - a @ v0)) < 1e-5


def test_xt_w_x_and_xt_vec(env):
    from paper_1902_04303_b200.matrix import pack_cp, unpack_cp
    from paper_1902_04303_b200.matrix_ext import xt_vec, xt_w_x

    hg, params = env["hg"], env["params"]
    xcp = pack_cp(env["x"], env["pk"], params, env["rng"])
    w = hg.encrypt_values(env["w"], params.log_p, env["pk"], params, env["rng"])
    a = xt_w_x(env["eng"], xcp, w)
    want = env["x"].T @ np.diag(env["w"]) @ env["x"]
    got = unpack_cp(a, env["sk"])[:5, :5]
    assert np.max(np.abs(got - want) / (1 + np.abs(want))) < 1e-5
    r = np.random.default_rng(4).uniform(-1, 1, 245)
    g = xt_vec(env["eng"], xcp, hg.encrypt_values(r, params.log_p, env["pk"], params, env["rng"]))
    assert np.max(np.abs(_dec(env, g, 5).real - env["x"].T @ r)) < 1e-4


@pytest.mark.parametrize("degree", [3, 5, 7])
def test_sigmoid_least_squares(env, degree):
    from paper_1902_04303_b200.matrix_ext import sigmoid_ls_coeffs, sigmoid_poly, sigmoid_poly_eval

    hg, params = env["hg"], env["params"]
    xs = np.linspace(-8, 8, params.slot_count)
    ct = hg.encrypt_values(xs, params.log_p, env["pk"], params, env["rng"])
    coeffs = sigmoid_ls_coeffs(degree)
    out = sigmoid_poly(env["eng"], ct, degree)
    got = hg.decrypt_values(out, env["sk"]).real
    want = sigmoid_poly_eval(xs, coeffs)
    assert np.max(np.abs(got - want)) < 1e-5                          # vs the replay
    fit_err = np.max(np.abs(want - 1 / (1 + np.exp(-xs))))           # the fit itself
    assert fit_err < {3: 0.12, 5: 0.07, 7: 0.05}[degree]
    assert out.level_bits < ct.level_bits


def test_newton_matrix_inverse(env):
    """A = X^T W X (encrypted end to end), 7 Newton steps from alpha = 1/(0.25 n (d+1))."""
    from paper_1902_04303_b200.matrix import pack_cp, unpack_cp
    from paper_1902_04303_b200.matrix_ext import newton_alpha, newton_inverse, newton_inverse_replay, xt_w_x

    hg, params = env["hg"], env["params"]
    xcp = pack_cp(env["x"], env["pk"], params, env["rng"])
    w = hg.encrypt_values(env["w"], params.log_p, env["pk"], params, env["rng"])
    a = xt_w_x(env["eng"], xcp, w)
    a_clear = env["x"].T @ np.diag(env["w"]) @ env["x"]
    alpha = newton_alpha(245, 5)
    iters = 7
    inv = newton_inverse(env["eng"], a, alpha, iters)
    got = unpack_cp(inv, env["sk"])[:5, :5]
    want = newton_inverse_replay(a_clear, alpha, iters)
    assert np.max(np.abs(got - want)) < 1e-5 * max(1.0, np.max(np.abs(want)))
    # the iteration converges quadratically toward the true inverse
    assert np.linalg.norm(got @ a_clear - np.eye(5)) < 1e-3

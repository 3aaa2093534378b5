"""Matrix-layer operations of BASELINE config 2 that the reference package does not have.

SURVEY §0 (reconciliation table) and §8(d) config 2: the reference implements Algorithms
1-8 (CP / CCP / RP / REP layouts, matrix.py:79-218), sigma7 with fixed coefficients
(logreg.py:32-46) and a *slotwise* Newton reciprocal (gwas.py:148-162).  Config 2 also names
X^T W X for a diagonal W, the diagonal-method matrix-vector product, least-squares sigmoid
fits of degree 3-7 and a Newton-iteration *matrix* inverse; SPEC.md:250 lists the diagonal
method as a non-goal.  They are built here on the same HeEngine operations (every ring
operation runs in the sm_100a kernels), with the reference's layouts and conventions:

  diag_matvec        Halevi-Shoup diagonal method for an r x c matrix (c | r, powers of two)
                     against a c-periodic vector: y = sum_i diag_i * rot(v, i)
  xt_w_x / xt_vec    X^T W X (symmetric: (d+1)(d+2)/2 dot products) and X^T v, as the
                     rp_matvec (Alg. 6) of the rows w * x_a -- results in CP layout
  sigmoid_poly       0.5 + sum_k c_k u^k, u = x/8, odd least-squares fit on [-8, 8]
  newton_inverse     X_{k+1} = X_k (2I - A X_k), X_1 = 2 alpha I - alpha^2 A, via cp_matmul

Parity with the reference is UNPINNED for these (no reference semantics); tests check the
decrypted results against a float64 replay of the same approximate computation
(tests/test_gpu_matrix_ext.py), and the integer ops underneath are the bit-exact ones.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .ckks import Ciphertext, HeEngine, add_plain, decrypt_values, encrypt_values, negate
from .errors import DimensionError, ParameterError
from .keys import PublicKey, SecretKey
from .matrix import CPMatrix, RPMatrix, cp_matmul, next_pow2, rp_matvec, sum_terms
from .params import CkksParams


# -- row-major packing (config 2: "packed row-major into N/2 slots") ---------------------------

@dataclass
class RowMajorMatrix:
    """A[i][j] at slot i*stride + j, stride = next_pow2(cols)."""

    ct: Ciphertext
    rows: int
    cols: int
    stride: int


def pack_row_major(matrix, pk: PublicKey, params: CkksParams, rng, scale_bits: int | None = None
                   ) -> RowMajorMatrix:
    mat = np.asarray(matrix, dtype=float)
    if mat.ndim != 2:
        raise DimensionError("expected a 2-D matrix")
    r, c = mat.shape
    stride = next_pow2(c)
    if r * stride > params.slot_count:
        raise DimensionError(f"{r}x{c} matrix needs {r * stride} slots > {params.slot_count}")
    vec = np.zeros(params.slot_count)
    for i in range(r):
        vec[i * stride:i * stride + c] = mat[i]
    ct = encrypt_values(vec, scale_bits or params.log_p, pk, params, rng)
    return RowMajorMatrix(ct=ct, rows=r, cols=c, stride=stride)


def unpack_row_major(m: RowMajorMatrix, sk: SecretKey) -> np.ndarray:
    vals = decrypt_values(m.ct, sk).real
    return np.stack([vals[i * m.stride:i * m.stride + m.cols] for i in range(m.rows)])


# -- diagonal method ---------------------------------------------------------------------------

def generalized_diagonals(matrix, slots: int) -> tuple[list[np.ndarray], int, int]:
    """Diagonals of an r x c matrix padded to R x C (powers of two, C <= R):
    diag_i[s] = A[s mod R][(s - i) mod C], tiled over all slots (period R).  With a
    C-periodic v, y[s] = sum_i diag_i[s] v[(s - i) mod C] = (A v)[s mod R]."""
    mat = np.asarray(matrix, dtype=float)
    r, c = mat.shape
    big_r, big_c = next_pow2(r), next_pow2(c)
    if big_c > big_r:
        big_r = big_c
    if big_r > slots:
        raise DimensionError(f"{big_r} padded rows exceed {slots} slots")
    pad = np.zeros((big_r, big_c))
    pad[:r, :c] = mat
    s = np.arange(slots)
    diags = [pad[s % big_r, (s - i) % big_c] for i in range(big_c)]
    return diags, big_r, big_c


def periodic_vector(v, period: int, slots: int) -> np.ndarray:
    """v (length <= period) zero-padded to `period` and tiled over all slots."""
    v = np.asarray(v, dtype=complex).ravel()
    if v.size > period or slots % period:
        raise DimensionError("vector longer than its period, or period does not divide slots")
    base = np.zeros(period, dtype=complex)
    base[:v.size] = v
    return np.tile(base, slots // period)


def pack_diagonals(matrix, pk: PublicKey, params: CkksParams, rng,
                   scale_bits: int | None = None) -> tuple[list[Ciphertext], int]:
    """Encrypted generalized diagonals (client side); returns (diagonals, column period C)."""
    diags, _, big_c = generalized_diagonals(matrix, params.slot_count)
    return [encrypt_values(d, scale_bits or params.log_p, pk, params, rng) for d in diags], big_c


def diag_matvec(engine: HeEngine, diags: list[Ciphertext], v: Ciphertext) -> Ciphertext:
    """A v by the diagonal method: v is C-periodic (C = len(diags)); rot_i = rot(v, i) by a
    ladder of unit rotations (C - 1 key switches, one key), then sum_i diag_i * rot_i
    (C ct-mults, one level).  The output is R-periodic (R = the diagonals' period)."""
    if not diags:
        raise DimensionError("no diagonals")
    rots = [v]
    for _ in range(1, len(diags)):
        rots.append(engine.rotate(rots[-1], 1))
    return sum_terms(engine, [engine.mult(d, r) for d, r in zip(diags, rots)])


def diag_matvec_plain(engine: HeEngine, matrix, v: Ciphertext,
                      scale_bits: int | None = None) -> Ciphertext:
    """Plaintext matrix x encrypted C-periodic vector: the diagonals are encoded, not
    encrypted (mult_plain: one plaintext level instead of a ciphertext level)."""
    from .encoding import encode

    params = engine.params
    scale = scale_bits or params.log_p_small
    diags, _, _ = generalized_diagonals(matrix, params.slot_count)
    rots = [v]
    for _ in range(1, len(diags)):
        rots.append(engine.rotate(rots[-1], 1))
    terms = [engine.mult_plain(r, encode(d, scale, params)) for d, r in zip(diags, rots)]
    return sum_terms(engine, terms)


# -- X^T W X and X^T v (CP in, CP out) -------------------------------------------------------------

def xt_vec(engine: HeEngine, x: CPMatrix, v: Ciphertext) -> Ciphertext:
    """X^T v with v in the first x.rows slots: entry a at slot a (rp_matvec of X^T)."""
    return rp_matvec(engine, RPMatrix(rows_ct=x.cols, rows=x.cols_logical, cols_logical=x.rows), v)


def xt_w_x(engine: HeEngine, x: CPMatrix, w: Ciphertext) -> CPMatrix:
    """X^T diag(w) X as a (d+1) x (d+1) CP matrix (entry (a, b) at slot a of column b).
    u_a = w * x_a; entry (a, b) = <u_a, x_b> (Alg. 5) computed once per unordered pair and
    masked into slot a of column b and slot b of column a (Alg. 6's masking)."""
    from .matrix import dot_prod

    d1 = x.cols_logical
    u = [engine.mult(col, w) for col in x.cols]
    dots = {}
    for a in range(d1):
        for b in range(a, d1):
            dots[(a, b)] = dot_prod(engine, u[a], x.cols[b], x.rows)
    cols = []
    for b in range(d1):
        terms = [engine.mult_plain(dots[(min(a, b), max(a, b))], engine.mask(("slot", a)))
                 for a in range(d1)]
        cols.append(sum_terms(engine, terms))
    return CPMatrix(cols=cols, rows=d1, cols_logical=d1)


# -- least-squares sigmoid fits -----------------------------------------------------------------

def sigmoid_ls_coeffs(degree: int, lo: float = -8.0, hi: float = 8.0, points: int = 4001) -> list[float]:
    """Odd least-squares fit sigma(x) - 0.5 ~ sum_k c_k u^k (k odd <= degree, u = x/hi) on a
    uniform grid of [lo, hi]; returns [c_1, c_3, ...]."""
    if degree < 1 or degree % 2 == 0:
        raise ParameterError("sigmoid fit degree must be odd and >= 1")
    x = np.linspace(lo, hi, points)
    u = x / hi
    powers = np.stack([u ** k for k in range(1, degree + 1, 2)], axis=1)
    coef, *_ = np.linalg.lstsq(powers, 1.0 / (1.0 + np.exp(-x)) - 0.5, rcond=None)
    return [float(c) for c in coef]


def sigmoid_poly_eval(x, coeffs, hi: float = 8.0) -> np.ndarray:
    """Cleartext value of the fitted polynomial (the replay of sigmoid_poly)."""
    u = np.asarray(x, dtype=float) / hi
    return 0.5 + sum(c * u ** (2 * k + 1) for k, c in enumerate(coeffs))


def sigmoid_poly(engine: HeEngine, ct: Ciphertext, degree: int = 3, coeffs=None,
                 hi: float = 8.0) -> Ciphertext:
    """0.5 + u (c_1 + c_3 u^2 + ... ), u = x/hi: the even part in u^2 is evaluated by
    Horner on u^2 with plaintext-constant coefficients (degree 3: 2 ct levels, degree 5:
    3, degree 7: 4).  `coeffs` defaults to sigmoid_ls_coeffs(degree)."""
    coeffs = list(coeffs) if coeffs is not None else sigmoid_ls_coeffs(degree, -hi, hi)
    u = engine.mult_const(ct, 1.0 / hi)
    if len(coeffs) == 1:
        return engine.add_const(engine.mult_const(u, coeffs[0]), 0.5)
    u2 = engine.mult(u, u)
    acc = engine.add_const(engine.mult_const(u2, coeffs[-1]), coeffs[-2])
    for c in reversed(coeffs[:-2]):
        acc = engine.add_const(engine.mult(acc, u2), c)
    return engine.add_const(engine.mult(u, acc), 0.5)


# -- Newton matrix inverse -------------------------------------------------------------------------

def newton_alpha(n: int, d1: int, w_max: float = 0.25) -> float:
    """A public step size for A = X^T W X with standardised columns: 1 / (w_max n d1) bounds
    1 / trace(A) >= 1 / lambda_max, so I - alpha A is a contraction."""
    return 1.0 / (w_max * n * d1)


def _scaled_identity_minus(engine: HeEngine, m: CPMatrix, value: float) -> CPMatrix:
    """value * I - M (value * e_j added through a range_value mask at M's scale)."""
    cols = []
    for j, col in enumerate(m.cols):
        t = negate(col)
        cols.append(add_plain(t, engine.mask(("range_value", j, j + 1, value), t.scale_bits)))
    return CPMatrix(cols=cols, rows=m.rows, cols_logical=m.cols_logical)


def newton_inverse(engine: HeEngine, a: CPMatrix, alpha: float, iters: int = 4) -> CPMatrix:
    """Approximate A^-1 for a square CP matrix: X_1 = alpha (2I - alpha A) (constants only),
    then X_{k+1} = X_k (2I - A X_k) with cp_matmul (Alg. 3).  Each later iteration costs
    two matrix products (2 ct + 2 pt levels)."""
    if a.rows != a.cols_logical:
        raise DimensionError("newton_inverse needs a square matrix")
    if iters < 1:
        raise ParameterError("iters must be >= 1")
    t = CPMatrix(cols=[engine.mult_const(c, alpha) for c in a.cols], rows=a.rows,
                 cols_logical=a.cols_logical)
    r = _scaled_identity_minus(engine, t, 2.0)                       # 2I - alpha A
    x = CPMatrix(cols=[engine.mult_const(c, alpha) for c in r.cols], rows=a.rows,
                 cols_logical=a.cols_logical)                        # X_1
    for _ in range(iters - 1):
        ax = cp_matmul(engine, a, x)
        x = cp_matmul(engine, x, _scaled_identity_minus(engine, ax, 2.0))
    return x


def newton_inverse_replay(a, alpha: float, iters: int = 4) -> np.ndarray:
    """float64 replay of newton_inverse."""
    a = np.asarray(a, dtype=float)
    eye = np.eye(a.shape[0])
    x = alpha * (2 * eye - alpha * a)
    for _ in range(iters - 1):
        x = x @ (2 * eye - a @ x)
    return x

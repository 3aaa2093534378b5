"""Float64 replay of the encrypted GWAS circuit -- TEST INFRASTRUCTURE ONLY.

The package's own cleartext oracle (reference oracle.py:128-159) uses the exact 1/w,
while the encrypted circuit uses 3 Newton steps from the guess 3 (gwas.py:148-162), so
encrypted outputs differ from it by the paper's approximation error, not by crypto noise
(SURVEY F11).  This replay evaluates the *same approximate circuit* in float64:

  beta, p : kappa steps of p = sigma7(-X beta), beta += 4 (X^T X)^-1 X^T (y - p)
            (logreg.py:54-80, sigma7 per logreg.py:32-46 / oracle.py:18-34)
  w       : p (1 - p)                                            (gwas.py:302)
  w^-1    : x1 = g (2 - g w), x <- x (2 - w x)                   (gwas.py:148-162)
  z       : X beta + w^-1 (y - p)                                (gwas.py:165-170)
  M       : I - X (X^T X)^-1 X^T                                 (gwas.py:173-180)
  num_j   : (w z')^T S'_j,   den_j : w^T (S'_j)^2,  z' = M z, S' = M S   (gwas.py:197-229)
"""
from __future__ import annotations

import math

import numpy as np

C1, C3, C5, C7 = -1.73496, 4.19407, -5.43402, 2.50739


def sigma7(x):
    u = np.asarray(x, dtype=float) / 8.0
    u2 = u * u
    return 0.5 + u * (C1 + u2 * (C3 + u2 * (C5 + u2 * C7)))


def replay_gwas(X, y, S, kappa: int = 3, inverse_iters: int = 3, guess: float = 3.0,
                xtx_inv=None):
    X = np.asarray(X, dtype=float)
    y = np.asarray(y, dtype=float)
    S = np.asarray(S, dtype=float)
    if xtx_inv is None:
        xtx_inv = np.linalg.inv(X.T @ X)
    beta = np.zeros(X.shape[1])
    p = None
    for _ in range(kappa):
        p = sigma7(-(X @ beta))
        beta = beta + 4.0 * (xtx_inv @ (X.T @ (y - p)))
    w = p * (1.0 - p)
    x = guess * (2.0 - guess * w)
    for _ in range(inverse_iters - 1):
        x = x * (2.0 - w * x)
    z = X @ beta + x * (y - p)
    M = np.eye(X.shape[0]) - X @ xtx_inv @ X.T
    zp = M @ z
    Sp = M @ S
    num = (w * zp) @ Sp
    den = w @ (Sp * Sp)
    return {"beta": beta, "p": p, "w": w, "w_inv": x, "z": z, "z_prime": zp,
            "numerator": num, "denominator": den}


def finalize(num, den):
    """b' = num/den, stderr = sqrt(1/den), two-sided normal p (gwas.py:365-377)."""
    num = np.asarray(num, dtype=float)
    den = np.asarray(den, dtype=float)
    eff = np.full(num.shape, np.nan)
    se = np.full(num.shape, np.nan)
    pv = np.full(num.shape, np.nan)
    ok = den > 0
    eff[ok] = num[ok] / den[ok]
    se[ok] = np.sqrt(1.0 / den[ok])
    pv[ok] = [math.erfc(abs(e) * math.sqrt(d) / math.sqrt(2.0)) for e, d in zip(eff[ok], den[ok])]
    return eff, se, pv


def oracle_modified(X, y, S, beta, p):
    """Cleartext semi-parallel statistics with the exact 1/w and the unweighted projector
    M = I - X (X^T X)^-1 X^T (reference oracle.py:141-153 gwas_modified_parts /
    oracle_gwas_modified); returns (numerator, denominator)."""
    X, y, S, p = (np.asarray(a, dtype=float) for a in (X, y, S, p))
    w = p * (1.0 - p)
    z = X @ beta + (y - p) / w
    M = np.eye(X.shape[0]) - X @ np.linalg.inv(X.T @ X) @ X.T
    zp, sp = M @ z, M @ S
    return (w * zp) @ sp, w @ (sp * sp)


def oracle_original(X, y, S, beta, p):
    """The original (weighted) semi-parallel statistics: S* = S - X (X^T W X)^-1 X^T W S
    (reference oracle.py:128-138); returns (numerator, denominator)."""
    X, y, S, p = (np.asarray(a, dtype=float) for a in (X, y, S, p))
    w = p * (1.0 - p)
    z = X @ beta + (y - p) / w
    proj = X @ (np.linalg.inv(X.T @ (w[:, None] * X)) @ (X.T * w))
    zs, ss = z - proj @ z, S - proj @ S
    return (w * zs) @ ss, w @ (ss * ss)


def accuracy(reference, test, thresholds=(0.1, 0.01, 0.005)) -> dict:
    """Entry-difference counts per threshold and the least-squares fit line (the paper's
    accuracy methodology, reference oracle.py:207-220)."""
    reference = np.asarray(reference, dtype=float)
    test = np.asarray(test, dtype=float)
    diff = np.abs(test - reference)
    slope, intercept = np.polyfit(reference, test, 1) if reference.size >= 2 else (1.0, 0.0)
    return {"entries": int(reference.size),
            "above": {str(t): int(np.sum(diff > t)) for t in thresholds},
            "pct_within": {str(t): round(100.0 * float(np.mean(diff <= t)), 2) for t in thresholds},
            "max_abs_diff": float(diff.max()) if diff.size else 0.0,
            "fit": {"slope": float(slope), "intercept": float(intercept)}}

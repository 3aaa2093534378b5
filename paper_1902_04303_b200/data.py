"""Synthetic GWAS inputs with the shapes and value distributions of BASELINE.json's configs.

The paper's iDASH 2018 dataset is not distributed, so seeded synthetic data
stands in for it:

  X = [1, sex ~ Bernoulli(0.5), age ~ N(50, 10), c3 ~ N(0, 1), c4 ~ N(0, 1)], covariates
      z-scored (reference data.preprocess semantics, data.py:143-161);
  y ~ Bernoulli(sigmoid(X beta*)), beta* ~ N(0, 0.5) ("0.5" read as a standard deviation);
  S: MAF_j ~ U(maf_lo, 0.5), s_ij ~ Binomial(2, MAF_j) (Hardy-Weinberg), z-scored columns.

Everything here is cleartext numpy preprocessing (out of the GPU hot path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionError, InputError


@dataclass
class CleartextDataset:
    """Standardized design: X has a leading ones column, y is 0/1 (reference oracle.py:47-64)."""

    X: np.ndarray
    S: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        self.X = np.asarray(self.X, dtype=float)
        self.S = np.asarray(self.S, dtype=float)
        self.y = np.asarray(self.y, dtype=float)
        if not np.allclose(self.X[:, 0], 1.0):
            raise InputError("first column of X must be the intercept (all ones)")
        if not np.all(np.isin(self.y, (0.0, 1.0))):
            raise InputError("response must be binary")
        if self.X.shape[0] != self.S.shape[0] or self.X.shape[0] != self.y.shape[0]:
            raise DimensionError("X, S and y disagree on the sample count")


def standardize_columns(mat) -> np.ndarray:
    """Z-score each column; constant columns become zeros."""
    mat = np.asarray(mat, dtype=float)
    mean = mat.mean(axis=0)
    std = mat.std(axis=0)
    out = np.zeros_like(mat)
    keep = std > 0
    out[:, keep] = (mat[:, keep] - mean[keep]) / std[keep]
    return out


def synth_gwas_dataset(n: int, d: int, k: int, seed: int = 0, maf_lo: float = 0.05,
                       beta_sd: float = 0.5) -> CleartextDataset:
    """Seeded config-0/3/4 style dataset (seeds seed, seed+1, seed+2 for X, y, S)."""
    if d < 1:
        raise InputError("need at least one covariate")
    rx = np.random.default_rng(seed)
    cov = np.empty((n, d))
    cov[:, 0] = rx.binomial(1, 0.5, size=n)
    if d > 1:
        cov[:, 1] = rx.normal(50.0, 10.0, size=n)
    if d > 2:
        cov[:, 2:] = rx.normal(0.0, 1.0, size=(n, d - 2))
    x = np.column_stack([np.ones(n), standardize_columns(cov)])
    ry = np.random.default_rng(seed + 1)
    beta = ry.normal(0.0, beta_sd, size=d + 1)
    prob = 1.0 / (1.0 + np.exp(-(x @ beta)))
    y = (ry.uniform(size=n) < prob).astype(float)
    rs = np.random.default_rng(seed + 2)
    maf = rs.uniform(maf_lo, 0.5, size=k)
    dos = rs.binomial(2, maf, size=(n, k)).astype(float)
    return CleartextDataset(X=x, S=standardize_columns(dos), y=y)

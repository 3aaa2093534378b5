"""BASELINE config 4: the encrypted semi-parallel GWAS beyond the reference's sample limit.

The reference materialises the n x n projector M = I - X (X^T X)^-1 X^T as n CP columns and
replicates every column next_pow2(n) times (gwas.py:173-194, 293-333), which needs
next_pow2(n) * n <= N/2 slots: n = 6000 would need 2^26 slots, so config 4 has no
reference execution and its parity is UNPINNED.  This module reformulates Algorithm 10 so M
is never formed.  With H = X G (G = (X^T X)^-1, the client's encrypted
inverse), r = w^-1 (y - p), z' = M z = z - H X^T z, a = w z' (w masked to the samples):

    num_j = (w z')^T M S_j        = a^T S_j - b^T t_j,             b = H^T a,  t_j = X^T S_j
    den_j = (M S_j)^T W (M S_j)   = q_j - 2 u_j^T c_j + c_j^T A2 c_j
            q_j = S_j^T W S_j,  u_j = X^T W S_j,  c_j = G t_j,  A2 = X^T W X

-- algebraically the reference's statistics (oracle/replay.replay_gwas is the checker).

Layout.  SNP group g holds slots/B SNPs (B = `block`, a power of two); for each sample block
b (B samples) the client encrypts one ciphertext with S[b B + i][g slots/B + pos] at slot
pos B + i.  Every per-sample weight vector v (X columns, W X columns, w, a) is turned once into
block weights V_b (slots pos B + i = v[b B + i]: range mask, left rotation, duplicate), so a
weighted sum over samples is sum_b V_b * ct_b followed by a log2(B)-step rotate-and-sum: the
result for SNP pos sits at slot pos B + B - 1.  Per group: 12 weighted sums (5 t, 5 u, q, a^T S)
and the per-SNP (d+1)-dimensional algebra slotwise (replicated entries of G, A2, b).

Depth (log_p = 40, log_p_small = 30 recommended at log_l = 1700): logistic fit and w^-1 as in
the reference, then z' at ~230 bits, a at ~190, b at ~120 and the numerator at ~50 bits.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .ckks import Ciphertext, HeEngine, decrypt_values, encrypt_values, mult_integer
from .errors import DimensionError, InputError
from .gwas import assemble_result, compute_z, inverse_slots
from .keys import PublicKey, SecretKey
from .logreg import LogRegInputs, hom_logreg
from .matrix import (CPMatrix, cp_matmul, cp_matvec, duplicate_many, pack_cp, replicate, rotate_sum,
                     rotate_sum_many, sum_terms)
from .matrix_ext import xt_vec, xt_w_x
from .params import CkksParams


@dataclass
class ScaleConfig:
    n: int
    d: int
    k: int
    block: int = 128          # samples per ciphertext block (power of two)
    kappa: int = 3
    inverse_iters: int = 3
    inverse_guess: float = 3.0

    def check(self, params: CkksParams) -> "ScaleConfig":
        if self.block & (self.block - 1) or self.block > params.slot_count:
            raise DimensionError("block must be a power of two within the slot count")
        if self.n > params.slot_count:
            raise DimensionError(f"{self.n} samples exceed {params.slot_count} slots (CP columns)")
        if self.d + 1 > self.n:
            raise InputError("more covariates than samples")
        return self

    def snps_per_group(self, params: CkksParams) -> int:
        return params.slot_count // self.block

    def num_blocks(self) -> int:
        return -(-self.n // self.block)

    def num_groups(self, params: CkksParams) -> int:
        return -(-self.k // self.snps_per_group(params))


@dataclass
class ScaleInputs:
    logreg: LogRegInputs
    config: ScaleConfig
    group_source: Callable[[int], list[Ciphertext]]   # g -> num_blocks ciphertexts


@dataclass
class ScaleSetup:
    beta: Ciphertext
    p: Ciphertext
    w: Ciphertext          # masked to the samples
    z_prime: Ciphertext
    a: Ciphertext          # w z'
    b_rep: list[Ciphertext]         # b = H^T a, entries replicated
    g_rep: list[list[Ciphertext]]   # G[r][c] replicated
    a2_rep: list[list[Ciphertext]]  # (X^T W X)[r][c] replicated
    v_x: list[list[Ciphertext]]     # block weights of X columns   [d+1][blocks]
    v_wx: list[list[Ciphertext]]    # block weights of W X columns [d+1][blocks]
    v_w: list[Ciphertext]           # block weights of w           [blocks]
    v_a: list[Ciphertext]           # block weights of a           [blocks]
    # fused path (HeEngine.inner_product): the same block weights as HBM-resident NTT residues,
    # X / W X weights brought down to one level (their sums only feed the (d+1)-dim algebra)
    fused: bool = False
    p_xwx: list | None = None       # [2(d+1)][blocks] at level_xwx
    p_w: list | None = None         # [1][blocks] at level_xwx - log_p (the squares' level)
    p_a: list | None = None         # [1][blocks]
    level_xwx: int = 0


@dataclass
class GroupOutput:
    index: int
    num_ct: Ciphertext
    den_ct: Ciphertext


# -- client side --------------------------------------------------------------------------------

def group_slots(s_mat: np.ndarray, g: int, b: int, config: ScaleConfig, slots: int) -> np.ndarray:
    """Slot vector of SNP group g, sample block b: S[b B + i][g slots/B + pos] at pos B + i."""
    blk = config.block
    per = slots // blk
    rows = s_mat[b * blk:(b + 1) * blk, g * per:(g + 1) * per]     # (<= B) x (<= per)
    tile = np.zeros((per, blk))
    tile[:rows.shape[1], :rows.shape[0]] = rows.T
    return tile.reshape(-1)


def pack_snp_group(s_mat: np.ndarray, g: int, config: ScaleConfig, params: CkksParams,
                   pk: PublicKey, rng) -> list[Ciphertext]:
    """Ciphertexts of SNP group g, one per sample block.  With a CUDA torch.Generator the
    encoding runs on the GPU too (encoding.encode_device; config 4 has no reference run)."""
    from .ckks import _is_torch_generator, encrypt
    from .encoding import encode_device

    slots = [group_slots(s_mat, g, b, config, params.slot_count) for b in range(config.num_blocks())]
    if _is_torch_generator(rng):
        return [encrypt(encode_device(v, params.log_p, params), pk, params, rng) for v in slots]
    return [encrypt_values(v, params.log_p, pk, params, rng) for v in slots]


def encrypt_scale_inputs(X: np.ndarray, y: np.ndarray, s_mat: np.ndarray, config: ScaleConfig,
                         params: CkksParams, pk: PublicKey, rng) -> ScaleInputs:
    config.check(params)
    xtx_inv = np.linalg.inv(X.T @ X)
    if np.abs(X.T @ X @ xtx_inv - np.eye(X.shape[1])).max() >= 1e-8:
        raise InputError("inverse verification failed")
    logreg = LogRegInputs(X=pack_cp(X, pk, params, rng), Xt_rep=None,
                          XtX_inv=pack_cp(xtx_inv, pk, params, rng),
                          y=encrypt_values(y, params.log_p, pk, params, rng))
    return ScaleInputs(logreg=logreg, config=config,
                       group_source=lambda g: pack_snp_group(s_mat, g, config, params, pk, rng))


# -- server side ----------------------------------------------------------------------------------

def block_weights(engine: HeEngine, v: Ciphertext, config: ScaleConfig) -> list[Ciphertext]:
    """V_b (b < num_blocks): v[b B .. b B + B) moved to slots [0, B) and tiled over all slots."""
    blk = config.block
    slots = engine.params.slot_count
    masked = [engine.mult_plain(v, engine.mask(("range", b * blk, min((b + 1) * blk, config.n))))
              for b in range(config.num_blocks())]
    moved = [engine.rotate_left(m, b * blk) if b else m for b, m in enumerate(masked)]
    if blk == slots:
        return moved
    return duplicate_many(engine, moved, blk)


def weighted_sum(engine: HeEngine, weights: list[Ciphertext], cts: list[Ciphertext],
                 block: int, square: bool = False) -> Ciphertext:
    """sum_i v_i s_i per SNP (sum_i v_i s_i^2 with `square`): sum_b V_b * ct_b, then the
    within-block rotate-and-sum; SNP pos lands at slot pos B + B - 1."""
    terms = []
    for v, c in zip(weights, cts):
        t = engine.mult(v, c)
        terms.append(engine.mult(t, c) if square else t)
    return rotate_sum(engine, sum_terms(engine, terms), 1, block)


def _replicated_entries(engine: HeEngine, m: CPMatrix) -> list[list[Ciphertext]]:
    """rep[r][c] = entry (r, c) of a CP matrix broadcast to every slot (Alg. 1 per column)."""
    cols = [replicate(engine, col, m.rows) for col in m.cols]
    return [[cols[c][r] for c in range(m.cols_logical)] for r in range(m.rows)]


def compute_scale_setup(engine: HeEngine, inputs: ScaleInputs, fused: bool = True) -> ScaleSetup:
    """Logistic fit, w, z', a, b = H^T a, replicated G / A2 / b entries and the block weights.
    With ``fused`` (default) the block weights are kept as resident NTT residues for
    HeEngine.inner_product (one relinearisation per weighted sum instead of one per block)."""
    cfg = inputs.config.check(engine.params)
    lr = inputs.logreg
    beta, p = hom_logreg(engine, lr, cfg.kappa)
    w = engine.mult(p, engine.sub_from_const(1.0, p))
    w_inv = inverse_slots(engine, w, cfg.inverse_iters, cfg.inverse_guess)
    z = compute_z(engine, lr.X, beta, lr.y, p, w_inv)
    w_m = engine.mult_plain(w, engine.mask(("range", 0, cfg.n)))        # garbage beyond n -> 0
    h = cp_matmul(engine, lr.X, lr.XtX_inv)                            # H = X G, from fresh inputs
    z_prime = engine.sub(z, cp_matvec(engine, h, xt_vec(engine, lr.X, z)))
    a = engine.mult(w_m, z_prime)
    b = xt_vec(engine, h, a)
    wx = [engine.mult(col, w_m) for col in lr.X.cols]
    a2 = xt_w_x(engine, lr.X, w_m)
    setup = ScaleSetup(
        beta=beta, p=p, w=w_m, z_prime=z_prime, a=a,
        b_rep=replicate(engine, b, cfg.d + 1),
        g_rep=_replicated_entries(engine, lr.XtX_inv),
        a2_rep=_replicated_entries(engine, a2),
        v_x=[block_weights(engine, col, cfg) for col in lr.X.cols],
        v_wx=[block_weights(engine, col, cfg) for col in wx],
        v_w=block_weights(engine, w_m, cfg),
        v_a=block_weights(engine, a, cfg),
    )
    if fused and hasattr(engine, "inner_product"):
        from .ckks import mod_down

        nb = cfg.num_blocks()
        lvl = min(setup.v_wx[0][0].level_bits, setup.v_w[0].level_bits)
        setup.level_xwx = lvl
        setup.p_xwx = [[engine.prepare_sum(mod_down(v, lvl), nb) for v in row]
                       for row in setup.v_x + setup.v_wx]
        lw = lvl - engine.params.log_p
        setup.p_w = [[engine.prepare_sum(mod_down(v, lw), nb) for v in setup.v_w]]
        setup.p_a = [[engine.prepare_sum(v, nb) for v in setup.v_a]]
        setup.v_x = setup.v_wx = setup.v_w = setup.v_a = None   # the prepared copies replace them
        setup.fused = True
    return setup


def compute_scale_group(engine: HeEngine, setup: ScaleSetup, cts: list[Ciphertext], config: ScaleConfig,
                        index: int = 0) -> GroupOutput:
    """num and den of one SNP group (SNP pos at slot pos B + B - 1)."""
    blk = config.block
    d1 = config.d + 1
    if setup.fused:
        from .ckks import _mod_down_view

        tu = engine.inner_product(setup.p_xwx, cts)                      # 2(d+1) sums, one pass
        views = [_mod_down_view(c, setup.level_xwx) for c in cts]
        sq = _mults(engine, views, views)
        q_raw = engine.inner_product(setup.p_w, sq)[0]
        a_raw = engine.inner_product(setup.p_a, cts)[0]
        tu = rotate_sum_many(engine, tu, 1, blk)
        t, u = tu[:d1], tu[d1:]
        q, at_s = (rotate_sum(engine, x, 1, blk) for x in (q_raw, a_raw))
    else:
        t = [weighted_sum(engine, setup.v_x[a], cts, blk) for a in range(d1)]
        u = [weighted_sum(engine, setup.v_wx[a], cts, blk) for a in range(d1)]
        q = weighted_sum(engine, setup.v_w, cts, blk, square=True)
        at_s = weighted_sum(engine, setup.v_a, cts, blk)
    # c = G t ; den = q - 2 u.c + c^T A2 c ; num = a^T S - b.t   (independent products batched)
    gt = _mults(engine, [setup.g_rep[r][s] for r in range(d1) for s in range(d1)],
                [t[s] for r in range(d1) for s in range(d1)])
    c = [sum_terms(engine, gt[r * d1:(r + 1) * d1]) for r in range(d1)]
    uc = sum_terms(engine, _mults(engine, u, c))
    idx = [(r, s) for r in range(d1) for s in range(r, d1)]
    cc = _mults(engine, [c[r] for r, _ in idx], [c[s] for _, s in idx])
    terms = _mults(engine, [setup.a2_rep[r][s] for r, s in idx], cc)
    quad = [mult_integer(term, 2) if r != s else term for (r, s), term in zip(idx, terms)]
    den = engine.add(engine.sub(q, mult_integer(uc, 2)), sum_terms(engine, quad))
    num = engine.sub(at_s, sum_terms(engine, _mults(engine, setup.b_rep, t)))
    return GroupOutput(index=index, num_ct=num, den_ct=den)


def _mults(engine: HeEngine, lhs, rhs) -> list[Ciphertext]:
    many = getattr(engine, "mult_many", None)
    return many(list(lhs), list(rhs)) if many else [engine.mult(a, b) for a, b in zip(lhs, rhs)]


def compute_scale_gwas(engine: HeEngine, inputs: ScaleInputs, fused: bool = True):
    setup = compute_scale_setup(engine, inputs, fused)
    cfg = inputs.config
    outs = [compute_scale_group(engine, setup, inputs.group_source(g), cfg, g)
            for g in range(cfg.num_groups(engine.params))]
    return setup, outs


def decrypt_scale_statistics(outs: list[GroupOutput], config: ScaleConfig, params: CkksParams,
                             sk: SecretKey):
    """(numerators, denominators) for the k SNPs, then the reference's finale (gwas.py:365-377)."""
    per = config.snps_per_group(params)
    pos = np.arange(per) * config.block + config.block - 1
    num, den = np.zeros(config.k), np.zeros(config.k)
    for o in outs:
        lo = o.index * per
        hi = min(lo + per, config.k)
        num[lo:hi] = decrypt_values(o.num_ct, sk).real[pos][:hi - lo]
        den[lo:hi] = decrypt_values(o.den_ct, sk).real[pos][:hi - lo]
    return num, den, assemble_result(num, den)

"""Multi-GPU execution of the encrypted GWAS: one process per GPU.

After the setup (logistic fit, w, w^-1, z, M, z', M_dup) every SNP batch is independent
(reference gwas.py:313-331; "batch processing may run concurrently"), so batches
are sharded round-robin over ranks with no data-path collective.  The setup itself splits too:
its 245-way loops -- ccp_to_cp's projector columns (matrix.py:196-209), identity_minus
(:212-218), replicate's one-hot chains of z' = M z (:79-106) and the M_dup duplicate ladders
(:159-170) -- are column-sharded, followed by one all-gather of the duplicated projector columns
(every rank's batches need all of them) and of the ranks' partial sums of z'.  Sums are exact
mod 2^l, so the gathered results are bit-identical to the single-GPU run.  The logistic fit
(sequential, data-dependent) and the 5x5 products before the column split are replicated.

Collectives: NCCL moves device tensors directly (NVLink / NVSwitch); any other backend (gloo,
used by the CPU and shared-device tests) is staged through host memory.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_batches(num_batches: int, rank: int, world: int) -> list[int]:
    """Round-robin batch indices owned by `rank` (balanced to within one batch)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return list(range(rank, num_batches, world))


def batch_owner(index: int, world: int) -> int:
    return index % world


# the setup's projector columns are split the same way (column j -> rank j % world)
owned_columns = shard_batches


@dataclass
class ShardPlan:
    num_batches: int
    world: int

    def owned(self, rank: int) -> list[int]:
        return shard_batches(self.num_batches, rank, self.world)

    def per_rank_counts(self) -> list[int]:
        return [len(self.owned(r)) for r in range(self.world)]


def ciphertext_payload(ct) -> np.ndarray:
    """Flatten a ciphertext's two polys to one uint32 host array (for gathers)."""
    a = ct.c0.numpy_words().ravel()
    b = ct.c1.numpy_words().ravel()
    return np.concatenate([a, b])


def gather_to_root(local: dict[int, np.ndarray], world: int, root: int = 0, group=None):
    """Gather {batch index: payload} dicts to `root` with torch.distributed (any backend).
    Returns the merged dict on root, None elsewhere."""
    import torch.distributed as dist

    if world == 1:
        return dict(local)
    objs = [None] * world if dist.get_rank(group) == root else None
    dist.gather_object(local, objs, dst=root, group=group)
    if objs is None:
        return None
    merged: dict[int, np.ndarray] = {}
    for part in objs:
        merged.update(part)
    return merged


def _meta(ct) -> tuple:
    return (ct.level_bits, ct.scale_bits, ct.depth_ct, ct.depth_pt, ct.pending)


def all_gather_ciphertexts(local: dict, total: int, world: int, group=None, params=None) -> list:
    """{index: Ciphertext} owned round-robin (index -> rank index % world), all at one level,
    -> the full list of `total` ciphertexts on every rank.  One all-gather of the packed words
    (device tensors over NCCL; host-staged for other backends) plus one of the metadata."""
    import torch
    import torch.distributed as dist

    from .ckks import Ciphertext
    from .ring import RingElement

    if world == 1:
        return [local[i] for i in range(total)]
    rank = dist.get_rank(group)
    mine = shard_batches(total, rank, world)
    if sorted(local) != mine:
        raise ValueError(f"rank {rank} holds {sorted(local)}, owns {mine}")
    kmax = len(shard_batches(total, 0, world))
    metas = [None] * world
    proto = local[mine[0]] if mine else None
    dist.all_gather_object(metas, ({i: _meta(local[i]) for i in mine},
                                   None if proto is None else (proto.c0.n, proto.level_bits)), group=group)
    shape = next(m[1] for m in metas if m[1] is not None)
    n, level = shape
    w = (level + 31) // 32
    nccl = dist.get_backend(group) == "nccl"
    # device words on a GPU; host tensors only in the CPU tests of this exchange logic
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    buf = torch.zeros((kmax, 2, w, n), dtype=torch.int32, device=dev)
    for k, i in enumerate(mine):
        ct = local[i]
        if ct.level_bits != level or ct.c0.n != n:
            raise ValueError("all gathered ciphertexts must share ring degree and level")
        buf[k, 0].copy_(ct.c0.words)
        buf[k, 1].copy_(ct.c1.words)
    if nccl:
        out = torch.empty((world * kmax, 2, w, n), dtype=torch.int32, device=dev)
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        host = buf.cpu()
        parts = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(parts, host, group=group)
        out = torch.cat(parts).to(dev)
    allmeta = {}
    for m, _ in metas:
        allmeta.update(m)
    res = []
    params = proto.params if proto is not None else params
    if params is None:
        raise ValueError(f"rank {rank} owns no ciphertext: pass params")
    slots = params.slot_count
    for i in range(total):
        r, k = i % world, i // world
        lv, sc, dct, dpt, pend = allmeta[i]
        res.append(Ciphertext(c0=RingElement(n, lv, words=out[r * kmax + k, 0]),
                              c1=RingElement(n, lv, words=out[r * kmax + k, 1]),
                              level_bits=lv, scale_bits=sc, slots=slots, params=params,
                              depth_ct=dct, depth_pt=dpt, pending=pend))
    return res


def compute_setup_sharded(engine, inputs, rank: int, world: int, group=None, gather_m: bool = True,
                          prepare_left: bool = True):
    """compute_setup with the 245-way column loops split over `world` ranks (see module doc).
    Returns (beta, p_prev, GwasIntermediate, m_dup) identical to the single-GPU setup; with
    ``gather_m=False`` the intermediate's M holds only this rank's columns (the batch loop needs
    M_dup, not M)."""
    from . import gwas
    from .ckks import add_many
    from .matrix import (CPMatrix, ccp_to_cp, cp_matmul, cp_rep_matmul, duplicate_many,
                         identity_minus, next_pow2, replicate)

    if world == 1:
        return gwas.compute_setup(engine, inputs, prepare_left=prepare_left)
    config, lr = inputs.config, inputs.logreg
    gwas.plan_setup(engine, config)
    beta, p_prev = gwas.hom_logreg(engine, lr, config.kappa)
    w = engine.mult(p_prev, engine.sub_from_const(1.0, p_prev))
    w_inv = gwas.inverse_slots(engine, w, config.inverse_iters, config.inverse_guess)
    z = gwas.compute_z(engine, lr.X, beta, lr.y, p_prev, w_inv)
    # compute_M (gwas.py:173-180) up to the column split, replicated (D + D^2 products)
    hat = cp_matmul(engine, lr.X, lr.XtX_inv)
    prod = cp_rep_matmul(engine, hat, lr.Xt_rep)
    n = config.n
    own = owned_columns(n, rank, world)
    m_own = identity_minus(engine, ccp_to_cp(engine, prod, own), lr.X.rows, own)
    # z' = M z = sum_j M_j * rep(z)_j: this rank's terms, then the exact sum of all partials
    partial = None
    if own:
        reps = replicate(engine, z, n, own)
        many = getattr(engine, "mult_many", None)
        terms = many(m_own.cols, reps) if many else [engine.mult(c, r) for c, r in zip(m_own.cols, reps)]
        partial = add_many(engine.align(*terms)) if len(terms) > 1 else terms[0]
    parts = all_gather_ciphertexts({rank: partial} if partial is not None else {}, world, world, group) \
        if all(len(owned_columns(n, r, world)) for r in range(world)) else None
    if parts is None:
        raise ValueError(f"world size {world} exceeds the {n} projector columns")
    z_prime = add_many(engine.align(*parts))
    cs = next_pow2(n)
    dup_own = duplicate_many(engine, m_own.cols, cs)
    m_dup = all_gather_ciphertexts(dict(zip(own, dup_own)), n, world, group)
    del dup_own
    if gather_m:
        m = CPMatrix(cols=all_gather_ciphertexts(dict(zip(own, m_own.cols)), n, world, group),
                     rows=m_own.rows, cols_logical=n)
    else:
        m = m_own
    inter = gwas.GwasIntermediate(w=w, w_inv=w_inv, z=z, M=m, z_prime=z_prime)
    if prepare_left and hasattr(engine, "prepare"):
        m_dup = [engine.prepare(ct, keep_words=False) for ct in m_dup]
    return beta, p_prev, inter, m_dup


def compute_gwas_encrypted_sharded(engine, inputs, rank: int, world: int, group=None,
                                   split_setup: bool = True, batches=None):
    """The setup (column-split with one all-gather, or replicated) and this rank's share of
    the batches.  ``batches``: an iterable of SnpBatch (e.g. a SnpBatchStream of this rank's
    host batches); default: the inputs' own batches, filtered to the ones this rank owns."""
    from .gwas import compute_batch, compute_setup

    if split_setup:
        beta, p_prev, inter, m_dup = compute_setup_sharded(engine, inputs, rank, world, group)
    else:
        beta, p_prev, inter, m_dup = compute_setup(engine, inputs)
    owned = set(shard_batches(inputs.config.num_batches, rank, world))
    source = batches if batches is not None else (b for b in inputs.iter_batches() if b.index in owned)
    outs = [compute_batch(engine, inputs, inter, m_dup, b) for b in source]
    return outs, inter, beta, p_prev

"""Multi-GPU execution of the per-batch hot loop.

After the setup (logistic fit, w, w^-1, z, M, z', M_dup) every SNP batch is independent
(gwas.py:314-331), so batches are sharded round-robin over ranks with no data-path
collective; each rank either replicates the setup (no communication) or receives the setup
ciphertexts once.  The only exchange is the final gather of the tiny per-batch result
ciphertexts (num, den_even, den_odd at levels ~95/425 bits) to the rank that decrypts.

The sharding logic is pure host code and is tested on CPU with the gloo backend
(tests/test_parallel.py); on B200 nodes the same calls run over NCCL.
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


def compute_gwas_encrypted_sharded(engine, inputs, rank: int, world: int):
    """Run the setup (replicated) and this rank's share of the batches."""
    from .gwas import compute_batch, compute_setup

    beta, p_prev, inter, m_dup = compute_setup(engine, inputs)
    owned = set(shard_batches(inputs.config.num_batches, rank, world))
    outs = []
    for batch in inputs.iter_batches():
        if batch.index in owned:
            outs.append(compute_batch(engine, inputs, inter, m_dup, batch))
    return outs, inter, beta, p_prev

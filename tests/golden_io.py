"""Readers for the committed golden fixtures (tests/golden/*.npz, made by
tools/make_golden.py from the reference package)."""
from __future__ import annotations

import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def words_to_ints(arr) -> list[int]:
    arr = np.asarray(arr, dtype=np.uint32)
    w, n = arr.shape
    raw = np.ascontiguousarray(arr.T).astype("<u4").tobytes()
    return [int.from_bytes(raw[i * 4 * w:(i + 1) * 4 * w], "little") for i in range(n)]


class Golden:
    def __init__(self, name: str):
        self.path = os.path.join(HERE, "golden", name + ".npz")
        self.z = np.load(self.path, allow_pickle=False)

    def __contains__(self, key):
        return key in self.z.files

    def arr(self, key):
        return self.z[key]

    def words(self, key):
        return np.asarray(self.z[key], dtype=np.uint32), int(self.z[key + "__bits"])

    def ints(self, key):
        w, bits = self.words(key)
        return words_to_ints(w), bits

    def meta(self, key):
        lv, sc, dct, dpt, pend = (int(x) for x in self.z[key + ".meta"])
        return {"level_bits": lv, "scale_bits": sc, "depth_ct": dct, "depth_pt": dpt,
                "pending": {0: None, 1: "ct", 2: "pt"}[pend]}

    def params_tuple(self):
        return tuple(int(x) for x in self.z["params"])

    def key_hashes(self) -> dict:
        return dict(zip([str(s) for s in self.z["key_hash_names"]],
                        [str(s) for s in self.z["key_hash_values"]]))


def words_hash(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr, dtype=np.uint32)).tobytes()).hexdigest()


def random_words(seed, bits: int, n: int) -> np.ndarray:
    """Uniform residues mod 2^bits as limb-major [W][N] uint32 words from a seeded numpy
    generator (seed: an int or a tuple of ints) -- the inputs of the scale goldens
    (tools/make_scale_golden.py), rebuilt identically by the GPU tests."""
    seq = list(seed) if isinstance(seed, (tuple, list)) else [seed]
    rng = np.random.default_rng(seq)
    w = (bits + 31) // 32
    arr = rng.integers(0, 1 << 32, size=(w, n), dtype=np.uint64).astype(np.uint32)
    top = bits - 32 * (w - 1)
    if top < 32:
        arr[w - 1] &= np.uint32((1 << top) - 1)
    return arr


def ints_to_words(coeffs, bits: int) -> np.ndarray:
    """Coefficients mod 2^bits -> limb-major [W][N] uint32 words (inverse of words_to_ints)."""
    w = (bits + 31) // 32
    mask = (1 << bits) - 1
    buf = b"".join((c & mask).to_bytes(4 * w, "little") for c in coeffs)
    return np.ascontiguousarray(np.frombuffer(buf, dtype="<u4").reshape(len(coeffs), w).T)

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

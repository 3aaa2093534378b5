"""Helpers for GPU parity tests: golden fixtures -> device objects and back."""
from __future__ import annotations

import numpy as np

from tests.golden_io import words_hash


def params_from(g):
    from paper_1902_04303_b200 import CkksParams

    log_n, log_l, log_p, log_p_small, h = g.params_tuple()
    return CkksParams(log_n=log_n, log_l=log_l, log_p=log_p, log_p_small=log_p_small, h=h)


def ring_from(g, key):
    from paper_1902_04303_b200.ring import RingElement, upload_words

    w, bits = g.words(key)
    return RingElement(w.shape[1], bits, words=upload_words(w))


def ct_from(g, name, params):
    from paper_1902_04303_b200 import Ciphertext

    meta = g.meta(name)
    return Ciphertext(c0=ring_from(g, name + ".c0"), c1=ring_from(g, name + ".c1"),
                      slots=params.slot_count, params=params, **meta)


def assert_ring_equal(elem, g, key):
    w, bits = g.words(key)
    assert elem.mod_bits == bits, f"{key}: modulus {elem.mod_bits} != {bits}"
    got = elem.numpy_words()
    if not np.array_equal(got, w):
        bad = np.argwhere(got != w)
        raise AssertionError(f"{key}: {len(bad)} words differ, first at (word, coeff) {bad[0].tolist()}")


def assert_ct_equal(ct, g, name):
    assert_ring_equal(ct.c0, g, name + ".c0")
    assert_ring_equal(ct.c1, g, name + ".c1")
    meta = g.meta(name)
    got = {"level_bits": ct.level_bits, "scale_bits": ct.scale_bits, "depth_ct": ct.depth_ct,
           "depth_pt": ct.depth_pt, "pending": ct.pending}
    assert got == meta, f"{name}: metadata {got} != {meta}"


def ring_hash(elem) -> str:
    return words_hash(elem.numpy_words())


def keys_from_golden(g, params):
    """Full key set stored in the fixture (unit_ops)."""
    from paper_1902_04303_b200.keys import EvaluationKey, PublicKey, RotationKeySet, SecretKey

    sk = SecretKey(s=ring_from(g, "sk.s"))
    pk = PublicKey(b=ring_from(g, "pk.b"), a=ring_from(g, "pk.a"))
    evk = EvaluationKey(b=ring_from(g, "evk.b"), a=ring_from(g, "evk.a"))
    rot = {}
    amt = 1
    while f"rot{amt}.b" in g:
        rot[amt] = (ring_from(g, f"rot{amt}.b"), ring_from(g, f"rot{amt}.a"))
        amt <<= 1
    conj = (ring_from(g, "conj.b"), ring_from(g, "conj.a"))
    return sk, pk, evk, RotationKeySet(keys=rot, conj=conj)

"""Reference-run golden HASHES at the ring sizes the product path runs at (config-1 corners and
the P17 parity preset), by running the REFERENCE package (hegwas) itself.

Full ciphertexts at N=2^16 are tens of MB each, so the fixture keeps, per output ciphertext,
the sha256 of its limb-major words ([W][N] uint32, c0 then c1) and its metadata.  Inputs are
uniform random residues drawn from a seeded numpy generator (tests/golden_io.random_words),
so the GPU test rebuilds the same inputs without the reference.  Keys come from the
reference's own keygen(params, seed); the fixture records their hashes, so the GPU test also
pins the client keygen at these sizes.

The reference runs with tools/gmpy2_shim on sys.path (libgmp's mpz_mul for its one big
multiply, hegwas/ring.py:55): exact, ~40x faster than CPython ints, results unchanged.

    python tools/make_scale_golden.py [case ...]      -> tests/golden/scale_hashes.json
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools", "gmpy2_shim"))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

OUT = os.path.join(REPO, "tests", "golden", "scale_hashes.json")

# (name, log_n, log_l, level, key seed): config-1 corners log_n 13..16 x log_l {240, 1440}
# at the top level, and P17 (log_n 17, log_l 1700) at the batch product's level 1550 and the
# setup's z' level 230 (SURVEY §8 level table).
CASES = [(f"n{ln}_l{ll}", ln, ll, ll, 100 + ln) for ln in (13, 14, 15, 16) for ll in (240, 1440)]
CASES += [("p17_1550", 17, 1700, 1550, 17), ("p17_230", 17, 1700, 230, 17)]


def ring_words(elem):
    import numpy as np

    w = (elem.mod_bits + 31) // 32
    buf = b"".join(c.to_bytes(4 * w, "little") for c in elem.coeffs)
    return np.ascontiguousarray(np.frombuffer(buf, dtype="<u4").reshape(len(elem.coeffs), w).T)


def ct_record(ct) -> dict:
    h = hashlib.sha256()
    h.update(ring_words(ct.c0).tobytes())
    h.update(ring_words(ct.c1).tobytes())
    return {"sha256": h.hexdigest(),
            "meta": [ct.level_bits, ct.scale_bits, ct.depth_ct, ct.depth_pt,
                     {None: 0, "ct": 1, "pt": 2}[ct.pending]]}


def pair_record(e0, e1) -> dict:
    h = hashlib.sha256()
    h.update(ring_words(e0).tobytes())
    h.update(ring_words(e1).tobytes())
    return {"sha256": h.hexdigest(), "meta": [e0.mod_bits]}


def key_hash(elem) -> str:
    return hashlib.sha256(ring_words(elem).tobytes()).hexdigest()


def run_case(case):
    import gmpy2

    import hegwas
    from hegwas import ckks as rck
    from hegwas.ring import RingElement

    from tests.golden_io import random_words, words_to_ints

    name, log_n, log_l, level, seed = case
    params = hegwas.CkksParams(log_n=log_n, log_l=log_l, log_p=45, log_p_small=30, h=64)
    n, slots = params.n, params.slot_count
    t0 = time.time()
    sk, pk, evk, rot = hegwas.keygen(params, seed)
    t_key = time.time() - t0
    keys = {"sk.s": key_hash(sk.s), "pk.b": key_hash(pk.b), "pk.a": key_hash(pk.a),
            "evk.b": key_hash(evk.b), "evk.a": key_hash(evk.a),
            "conj.b": key_hash(rot.conj[0]), "conj.a": key_hash(rot.conj[1])}
    for amt, (b, a) in rot.keys.items():
        keys[f"rot{amt}.b"] = key_hash(b)
        keys[f"rot{amt}.a"] = key_hash(a)

    def ct(tag):
        c0 = RingElement(n, level, words_to_ints(random_words((seed, level, tag, 0), level, n)))
        c1 = RingElement(n, level, words_to_ints(random_words((seed, level, tag, 1), level, n)))
        return rck.Ciphertext(c0=c0, c1=c1, level_bits=level, scale_bits=params.log_p, slots=slots,
                              params=params)

    a, b, a2, b2 = ct(0), ct(1), ct(2), ct(3)
    eng = hegwas.HeEngine(params, evk, rot)
    out = {}
    t0 = time.time()
    out["mult_ab"] = ct_record(eng.mult(a, b))
    out["mult_a2b2"] = ct_record(eng.mult(a2, b2))
    e0, e1 = rck._keyswitch(a.c1, (evk.b, evk.a), level, params.log_l)
    out["keyswitch_a1"] = pair_record(e0, e1)
    rot_a1 = eng.rotate(a, 1)
    out["rot1_a"] = ct_record(rot_a1)
    out["rot1_b"] = ct_record(eng.rotate(b, 1))
    out["add_a_rot1_a"] = ct_record(eng.add(a, rot_a1))
    out["rot_half_a"] = ct_record(eng.rotate(a, slots // 2))
    out["rot5_a"] = ct_record(eng.rotate(a, 5))
    out["rotl_quarter_a"] = ct_record(eng.rotate_left(a, slots // 4))
    out["rotl_half_b"] = ct_record(eng.rotate_left(b, slots // 2))
    out["conj_a"] = ct_record(eng.conjugate(a))
    out["rescale30_a"] = ct_record(rck.rescale(a, 30))
    out["mult_plain_range_a"] = ct_record(eng.mult_plain(a, eng.mask(("range", 0, 256))))
    out["mult_const_a"] = ct_record(eng.mult_const(a, 0.125))
    t_ops = time.time() - t0
    print(f"{name}: keygen {t_key:.1f}s ops {t_ops:.1f}s", flush=True)
    return name, {"log_n": log_n, "log_l": log_l, "log_p": 45, "log_p_small": 30, "h": 64,
                  "level": level, "seed": seed, "keys": keys, "outputs": out,
                  "reference_seconds": {"keygen": round(t_key, 1), "ops": round(t_ops, 1)},
                  "gmpy2": "tools/gmpy2_shim (libgmp mpz_mul)" if getattr(gmpy2, "SHIM", False) else "gmpy2"}


def main():
    want = set(sys.argv[1:])
    cases = [c for c in CASES if not want or c[0] in want]
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    # largest first so the pool's tail is short
    cases.sort(key=lambda c: -(c[1] * 10000 + c[2]))
    with Pool(min(len(cases), os.cpu_count() or 1)) as pool:
        for name, rec in pool.imap_unordered(run_case, cases):
            data[name] = rec
            with open(OUT, "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()

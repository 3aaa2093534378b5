"""Bit-exact parity at the ring sizes the product path actually runs at, against the REFERENCE.

tests/golden/scale_hashes.json holds, for every config-1 corner (log_n 13..16 x log_l 240 /
1440, top level) and the P17 parity preset at levels 1550 and 230, the sha256 of each output
ciphertext the reference package computed (tools/make_scale_golden.py: hegwas itself, its one
big multiply through libgmp).  The GPU rebuilds the same uniform random input ciphertexts from
their seeds, derives the keys with its own keygen (their hashes are pinned too), and must
reproduce every output word for word: ckks.mult + rescale (hegwas ckks.py:166-224, 310-313),
_keyswitch (:187-194), rotate by 1, by slots/2 and by 5 (composite), rotate_left (:256-273,
322-323), conjugate (:276-279), rescale (:197-224), mult_plain with a range mask and
mult_const (:147-163, 315-317, 351-356) -- and the batched entry points (mult_many,
mult_prepared_many, rotate_many, rotate_add_many, rotate_left_each) must give the same words
as the one-by-one reference ops.  Each selects different NTT / ModUp / CRT instantiations than
the toy goldens (log_n <= 9) do."""
from __future__ import annotations

import hashlib
import json
import os

import pytest

from tests.golden_io import HERE, random_words

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(HERE, "golden", "scale_hashes.json")))
CASES = sorted(GOLD, key=lambda c: (GOLD[c]["log_n"], GOLD[c]["log_l"], GOLD[c]["level"]))



def _ct_sha(ct) -> str:
    h = hashlib.sha256()
    h.update(ct.c0.numpy_words().tobytes())
    h.update(ct.c1.numpy_words().tobytes())
    return h.hexdigest()


def _meta(ct) -> list:
    return [ct.level_bits, ct.scale_bits, ct.depth_ct, ct.depth_pt, {None: 0, "ct": 1, "pt": 2}[ct.pending]]


def _check(case, name, ct):
    want = GOLD[case]["outputs"][name]
    assert _meta(ct) == want["meta"], f"{case}/{name}: metadata {_meta(ct)} != {want['meta']}"
    assert _ct_sha(ct) == want["sha256"], f"{case}/{name}: ciphertext words differ from the reference"


@pytest.fixture(scope="module", params=CASES)
def st(request):
    """Keys (own keygen, same seed), engine and the four input ciphertexts of a case (module
    scope: pytest runs every test of one case before building the next)."""
    import gc

    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.ring import RingElement, upload_words

    gc.collect()
    case = request.param
    g = GOLD[case]
    params = hg.CkksParams(log_n=g["log_n"], log_l=g["log_l"], log_p=g["log_p"],
                           log_p_small=g["log_p_small"], h=g["h"])
    keys = hg.keygen(params, g["seed"])
    n, level, seed = params.n, g["level"], g["seed"]

    def ct(tag):
        c0 = RingElement(n, level, words=upload_words(random_words((seed, level, tag, 0), level, n)))
        c1 = RingElement(n, level, words=upload_words(random_words((seed, level, tag, 1), level, n)))
        return hg.Ciphertext(c0=c0, c1=c1, level_bits=level, scale_bits=params.log_p,
                             slots=params.slot_count, params=params)

    yield dict(case=case, params=params, keys=keys, engine=hg.HeEngine(params, keys[2], keys[3]),
               cts=[ct(i) for i in range(4)])


def test_keygen_hashes(st):
    from tests.gpu_helpers import ring_hash

    case = st["case"]
    sk, pk, evk, rot = st["keys"]
    got = {"sk.s": ring_hash(sk.s), "pk.b": ring_hash(pk.b), "pk.a": ring_hash(pk.a),
           "evk.b": ring_hash(evk.b), "evk.a": ring_hash(evk.a),
           "conj.b": ring_hash(rot.conj[0]), "conj.a": ring_hash(rot.conj[1])}
    for amt, (b, a) in rot.keys.items():
        got[f"rot{amt}.b"] = ring_hash(b)
        got[f"rot{amt}.a"] = ring_hash(a)
    assert got == GOLD[case]["keys"]


def test_scheme_ops(st):
    from paper_1902_04303_b200 import ckks

    case = st["case"]
    eng, (a, b, a2, b2), params = st["engine"], st["cts"], st["params"]
    slots = params.slot_count
    _check(case, "mult_ab", eng.mult(a, b))
    _check(case, "mult_a2b2", eng.mult(a2, b2))
    evk = st["keys"][2]
    e0, e1 = ckks._keyswitch(a.c1, (evk.b, evk.a), a.level_bits, params.log_l)
    h = hashlib.sha256()
    h.update(e0.numpy_words().tobytes())
    h.update(e1.numpy_words().tobytes())
    want = GOLD[case]["outputs"]["keyswitch_a1"]
    assert [e0.mod_bits] == want["meta"] and h.hexdigest() == want["sha256"], f"{case}: _keyswitch differs"
    _check(case, "rot1_a", eng.rotate(a, 1))
    _check(case, "rot_half_a", eng.rotate(a, slots // 2))
    _check(case, "rot5_a", eng.rotate(a, 5))
    _check(case, "rotl_quarter_a", eng.rotate_left(a, slots // 4))
    _check(case, "conj_a", eng.conjugate(a))
    _check(case, "rescale30_a", ckks.rescale(a, 30))
    _check(case, "mult_plain_range_a", eng.mult_plain(a, eng.mask(("range", 0, 256))))
    _check(case, "mult_const_a", eng.mult_const(a, 0.125))


def test_batched_entry_points(st):
    case = st["case"]
    eng, (a, b, a2, b2), params = st["engine"], st["cts"], st["params"]
    slots = params.slot_count
    m1, m2 = eng.mult_many([a, a2], [b, b2])
    _check(case, "mult_ab", m1)
    _check(case, "mult_a2b2", m2)
    p1, p2 = eng.mult_prepared_many([eng.prepare(a), eng.prepare(a2)], [b, b2])
    _check(case, "mult_ab", p1)
    _check(case, "mult_a2b2", p2)
    r1, r2 = eng.rotate_many([a, b], 1)
    _check(case, "rot1_a", r1)
    _check(case, "rot1_b", r2)
    (s1,) = eng.rotate_add_many([a], 1)
    _check(case, "add_a_rot1_a", s1)
    l1, l2 = eng.rotate_left_each([a, b], [slots // 4, slots // 2])
    _check(case, "rotl_quarter_a", l1)
    _check(case, "rotl_half_b", l2)

"""The batched / fused ciphertext entry points added on top of the reference's op set must give,
word for word and event for event, what the one-by-one reference ops give:

  HeEngine.mult_plain_each(ct, pts)  (hg_ct_mult_plain_many: one ciphertext, many plaintexts --
                                      replicate's masks, ccp_to_cp's ranges; matrix.py:79-96, 196-209)
  HeEngine.mult_plain_many(cts, pt)  (hg_ct_mult_plain_batch)
  HeEngine.mult_const_many(cts, v)   (hg_ct_mult_const_rescale_batch)
  HeEngine.rescale_many / add_each / sub_each  (hg_ct_rescale_batch / hg_ct_add_batch)

against rescale(mult_plain(ct, pt), pt.scale_bits) etc. through the unfused module functions
(ckks.py:108-163, 197-224; pinned to the reference's goldens by test_gpu_ckks) and, for one
case, against the CPU oracle."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_1902_04303_b200 as hg

    params = hg.CkksParams(log_n=10, log_l=700, log_p=45, log_p_small=30, h=32)
    sk, pk, evk, rot = hg.keygen(params, 4)
    eng = hg.HeEngine(params, evk, rot)
    rng = random.Random(9)
    cts = []
    for s in range(3):
        vals = [complex(rng.uniform(-1, 1), rng.uniform(-1, 1)) for _ in range(params.slot_count)]
        cts.append(hg.mod_down(hg.encrypt_values(vals, params.log_p, pk, params, rng), 600))
    return hg, params, eng, cts


def _same(a, b):
    assert (a.level_bits, a.scale_bits, a.depth_ct, a.depth_pt, a.pending) == \
        (b.level_bits, b.scale_bits, b.depth_ct, b.depth_pt, b.pending)
    assert np.array_equal(a.c0.numpy_words(), b.c0.numpy_words())
    assert np.array_equal(a.c1.numpy_words(), b.c1.numpy_words())


def _unfused(hg, ct, pt):
    return hg.rescale(hg.mult_plain(ct, pt), pt.scale_bits)


def test_mult_plain_each_matches_one_by_one(env):
    hg, params, eng, (a, b, c) = env
    pts = [eng.mask(("slot", 3)), eng.mask(("range", 0, 64)), eng.mask(("range_value", 5, 90, 0.5)),
           eng.mask(("slot", 7), params.log_p), eng.constant(0.125), eng.constant(-3.0)]
    with hg.track_ops() as ops_b:
        got = eng.mult_plain_each(a, pts)
    with hg.track_ops() as ops_r:
        want = [_unfused(hg, a, pt) for pt in pts]
    assert ops_b.snapshot() == ops_r.snapshot()
    for g, w in zip(got, want):
        _same(g, w)


def test_mult_plain_many_and_const_match_one_by_one(env):
    hg, params, eng, cts = env
    pt = eng.mask(("range", 16, 200))
    for g, ct in zip(eng.mult_plain_many(cts, pt), cts):
        _same(g, _unfused(hg, ct, pt))
    for v in (0.5, -2.0, 3.0):
        for g, ct in zip(eng.mult_const_many(cts, v), cts):
            _same(g, _unfused(hg, ct, eng.constant(v)))


def test_rescale_and_add_batches_match_one_by_one(env):
    hg, params, eng, (a, b, c) = env
    for g, ct in zip(eng.rescale_many([a, b, c], 30), (a, b, c)):
        _same(g, hg.rescale(ct, 30))
    for g, (x, y) in zip(eng.add_each([a, b, c], [c, a, b]), ((a, c), (b, a), (c, b))):
        _same(g, hg.add(x, y))
    for g, (x, y) in zip(eng.sub_each([a, b], [c, c]), ((a, c), (b, c))):
        _same(g, hg.sub(x, y))


def test_fused_mult_plain_matches_oracle(env):
    from oracle import ckks_oracle as C

    hg, params, eng, (a, b, c) = env
    pt = eng.mask(("range", 0, 300))
    got = eng.mult_plain_each(a, [pt])[0]
    m = pt.m.coeffs
    p0, p1 = C.mult_plain(a.c0.coeffs, a.c1.coeffs, m, pt.m.mod_bits, a.level_bits, params.n)
    r0, r1 = C.rescale(p0, p1, pt.scale_bits, a.level_bits)
    assert (got.c0.coeffs, got.c1.coeffs) == (r0, r1)

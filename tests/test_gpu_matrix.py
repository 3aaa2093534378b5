"""The properties the reference's own tests pin for the ring, scheme and matrix layers
(reference pkg/tests/test_ring.py, test_ckks.py, test_matrix.py; SURVEY §4 item i), run on
the GPU path: Algorithms 1-8 against numpy, their level / depth / rotation contracts, and
the exact ring identities (wraparound sign, automorphism group law, divide_round
representative independence, centered lift).  UNIT parameters as in the reference's
conftest (log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def unit():
    import paper_1902_04303_b200 as hg

    params = hg.CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)
    sk, pk, evk, rot = hg.keygen(params, seed=7)
    return hg, params, sk, pk, hg.HeEngine(params, evk, rot)


def _rand(shape, seed):
    return np.random.default_rng(seed).uniform(-1, 1, shape)


def test_replicate_and_cp_matvec_contracts(unit):
    from paper_1902_04303_b200 import matrix as mx

    hg, params, sk, pk, eng = unit
    a, v = _rand((6, 4), 1), _rand(4, 2)
    acp = mx.pack_cp(a, pk, params, random.Random(1))
    vct = hg.encrypt_values(v, params.log_p, pk, params, random.Random(2))
    reps = mx.replicate(eng, vct, 4)
    for i, r in enumerate(reps):    # entry i in every slot
        assert np.max(np.abs(hg.decrypt_values(r, sk) - v[i])) < 1e-5
    with hg.track_ops() as ops:
        y = mx.cp_matvec(eng, acp, vct)
    assert np.max(np.abs(hg.decrypt_values(y, sk)[:6].real - a @ v)) < 1e-4
    # level contract: one plaintext level (replicate's mask) and one ciphertext level
    assert y.level_bits == params.log_l - params.log_p_small - params.log_p
    assert (y.depth_ct, y.depth_pt) == (1, 1)
    assert ops.all_rotations_power_of_two()


def test_cp_matmul_col_sum_dot_prod_rp_matvec(unit):
    from paper_1902_04303_b200 import matrix as mx

    hg, params, sk, pk, eng = unit
    rng = random.Random(3)
    a, b = _rand((4, 3), 3), _rand((3, 2), 4)
    prod = mx.cp_matmul(eng, mx.pack_cp(a, pk, params, rng), mx.pack_cp(b, pk, params, rng))
    assert np.max(np.abs(mx.unpack_cp(prod, sk).real - a @ b)) < 1e-4
    c = _rand((8, 5), 5)
    cs = mx.col_sum(eng, mx.pack_ccp(c, pk, params, rng))
    got = hg.decrypt_values(cs, sk).real
    assert np.max(np.abs(got[[8 * j for j in range(5)]] - c.sum(axis=0))) < 1e-4
    x, w = _rand(10, 6), _rand(10, 7)
    d = mx.dot_prod(eng, hg.encrypt_values(x, 45, pk, params, rng), hg.encrypt_values(w, 45, pk, params, rng), 10)
    assert np.max(np.abs(hg.decrypt_values(d, sk).real - x @ w)) < 1e-4   # replicated everywhere
    r = _rand((3, 6), 8)
    y = mx.rp_matvec(eng, mx.pack_rp(r, pk, params, rng), hg.encrypt_values(_rand(6, 9), 45, pk, params, rng))
    assert np.max(np.abs(hg.decrypt_values(y, sk)[:3].real - r @ _rand(6, 9))) < 1e-4


def test_duplicate_cp_rep_ccp_to_cp_identity_minus(unit):
    from paper_1902_04303_b200 import matrix as mx

    hg, params, sk, pk, eng = unit
    rng = random.Random(11)
    v = _rand(5, 10)
    dup = mx.duplicate(eng, hg.encrypt_values(v, 45, pk, params, rng), 5)
    got = hg.decrypt_values(dup, sk).real
    assert np.max(np.abs(got[:40].reshape(5, 8)[:, :5] - v)) < 1e-5       # tiles of next_pow2(5)=8
    a, b = _rand((6, 3), 12), _rand((3, 4), 13)
    acp = mx.pack_cp(a, pk, params, rng)
    ccp = mx.cp_rep_matmul(eng, acp, mx.pack_rep(b, 8, pk, params, rng))
    assert ccp.col_size == 8 and ccp.ct.level_bits == params.log_l - params.log_p   # one ct level
    assert np.max(np.abs(mx.unpack_ccp(ccp, sk, rows=6).real - a @ b)) < 1e-4
    cols = mx.ccp_to_cp(eng, ccp)
    assert np.max(np.abs(mx.unpack_cp(cols, sk)[:6].real - a @ b)) < 1e-4
    sq = _rand((4, 4), 14)
    im = mx.identity_minus(eng, mx.pack_cp(sq, pk, params, rng), 4)
    assert np.max(np.abs(mx.unpack_cp(im, sk).real - (np.eye(4) - sq))) < 1e-5


def test_rotation_key_switch_counts(unit):
    """A rotation costs one key switch per set bit, recorded ascending (the reference's
    245 -> {1, 4, 16, 32, 64, 128} contract, here 45 -> {1, 4, 8, 32} at 128 slots), and right
    rotations compose (reference test_ckks.py:262-300)."""
    hg, params, sk, pk, eng = unit
    v = _rand(params.slot_count, 15)
    ct = hg.encrypt_values(v, 45, pk, params, random.Random(5))
    with hg.track_ops() as ops:
        r = eng.rotate(ct, 45)                         # slots = 128: 45 = 32 + 8 + 4 + 1
    assert ops.keyswitches == 4 and ops.rotation_amounts == [1, 4, 8, 32]
    assert np.max(np.abs(hg.decrypt_values(r, sk) - np.roll(v, 45))) < 1e-5
    two = eng.rotate(eng.rotate(ct, 3), 5)
    assert np.max(np.abs(hg.decrypt_values(two, sk) - np.roll(v, 8))) < 1e-5


def test_exact_ring_identities(unit):
    """Wraparound sign, automorphism group law, divide_round representative independence,
    centered lift (reference test_ring.py:39-95), bit-exact on the GPU."""
    from paper_1902_04303_b200.ring import RingElement

    hg, params, *_ = unit
    n, bits = 64, 200
    xs = [0] * n
    xs[n - 1] = 1
    x1 = [0] * n
    x1[1] = 1
    prod = RingElement(n, bits, xs).mul(RingElement(n, bits, x1)).coeffs
    assert prod == [(1 << bits) - 1] + [0] * (n - 1)           # x^(n-1) * x = -1
    rng = random.Random(17)
    a = RingElement(n, bits, [rng.getrandbits(bits) for _ in range(n)])
    for k1, k2 in [(3, 5), (7, 9), (5, 2 * n - 1)]:
        assert a.automorphism(k1).automorphism(k2).coeffs == a.automorphism((k1 * k2) % (2 * n)).coeffs
    wide = a.lift_centered_to(bits + 40)                       # another representative of a
    assert wide.divide_round(30, bits - 30).coeffs == a.divide_round(30, bits - 30).coeffs
    small = RingElement(n, 16, [rng.getrandbits(16) for _ in range(n)])
    lifted = small.lift_centered_to(bits).coeffs
    for c, l in zip(small.coeffs, lifted):
        cen = c - (1 << 16) if c > (1 << 15) else c
        assert l == cen % (1 << bits)

"""Pin the CPU oracle against golden vectors produced by the reference package itself.

Every case recomputes a reference output from the golden inputs with oracle/ and demands
bit equality (these run without a GPU)."""
import pytest

from oracle import ckks_oracle as C
from oracle import ring_oracle as R


def _ct(g, name):
    c0, lv = g.ints(name + ".c0")
    c1, _ = g.ints(name + ".c1")
    return c0, c1, lv


@pytest.fixture(params=["unit_ops", "deep_ops"])
def case(request, golden):
    g = golden(request.param)
    log_n, log_l, log_p, log_p_small, h = g.params_tuple()
    return g, log_n, log_l, log_p, log_p_small


def _keys(g, log_n, log_l):
    if "evk.b" in g:
        return {k: g.ints(k)[0] for k in ("evk.b", "evk.a", "rot1.b", "rot1.a", "conj.b", "conj.a")}
    return None


def test_kronecker_matches_schoolbook_known_answer():
    # ring.py:29-58 property at the reference's test sizes (test_ring.py:23-36)
    import random

    for n, bits in ((16, 1), (32, 77), (64, 200), (64, 2400)):
        rng = random.Random(n * bits)
        a = [rng.getrandbits(bits) for _ in range(n)]
        b = [rng.getrandbits(bits) for _ in range(n)]
        assert R.negacyclic_mul(a, b, n, bits, bits) == R.schoolbook_negacyclic(a, b, n)


def test_wraparound_sign():
    n = 16
    a = [0] * n
    a[n - 1] = 1
    b = [0] * n
    b[1] = 1
    out = R.schoolbook_negacyclic(a, b, n)
    assert out[0] == -1 and not any(out[1:])


def test_oracle_rescale_and_moddown(case):
    g, log_n, log_l, log_p, _ = case
    a0, a1, lv = _ct(g, "ct_a")
    r0, r1 = C.rescale(a0, a1, 30, lv)
    assert (r0, r1) == (g.ints("rescale30.c0")[0], g.ints("rescale30.c1")[0])
    md0, md1, md_lv = _ct(g, "mod_down")
    assert R.reduce_to(a0, md_lv) == md0 and R.reduce_to(a1, md_lv) == md1


def test_oracle_integer_and_negation(case):
    g, *_ = case
    a0, a1, lv = _ct(g, "ct_a")
    assert R.scalar_mul(a0, 4, lv) == g.ints("mult_int_4.c0")[0]
    assert R.scalar_mul(a1, -1, lv) == g.ints("mult_int_m1.c1")[0]


def test_oracle_mult_and_keyswitch_unit(golden):
    g = golden("unit_ops")
    log_n, log_l, log_p, _, _ = g.params_tuple()
    n = 1 << log_n
    a0, a1, lv = _ct(g, "ct_a")
    b0, b1, _ = _ct(g, "ct_b")
    evb, _ = g.ints("evk.b")
    eva, _ = g.ints("evk.a")
    e0, e1 = C.keyswitch(a1, evb, eva, lv, log_l, n)
    assert e0 == g.ints("keyswitch.e0")[0] and e1 == g.ints("keyswitch.e1")[0]
    m0, m1 = C.mult(a0, a1, b0, b1, lv, evb, eva, log_l, n)
    assert (m0, m1) == (g.ints("mult_raw.c0")[0], g.ints("mult_raw.c1")[0])
    r0, r1 = C.engine_mult(a0, a1, b0, b1, lv, evb, eva, log_l, log_p, n)
    assert (r0, r1) == (g.ints("eng_mult.c0")[0], g.ints("eng_mult.c1")[0])


def test_oracle_rotations_unit(golden):
    g = golden("unit_ops")
    log_n, log_l, *_ = g.params_tuple()
    n = 1 << log_n
    a0, a1, lv = _ct(g, "ct_a")
    kb, _ = g.ints("rot1.b")
    ka, _ = g.ints("rot1.a")
    k = C.rotation_exponent(log_n, 1)
    o = C.apply_automorphism(a0, a1, k, kb, ka, lv, log_l, n)
    assert o == (g.ints("rot1.c0")[0], g.ints("rot1.c1")[0])
    cb, _ = g.ints("conj.b")
    ca, _ = g.ints("conj.a")
    o = C.apply_automorphism(a0, a1, 2 * n - 1, cb, ca, lv, log_l, n)
    assert o == (g.ints("conj.c0")[0], g.ints("conj.c1")[0])
    # composite right rotation by 5 = 1 then 4 (ckks.py:264-272)
    k4b, _ = g.ints("rot4.b")
    k4a, _ = g.ints("rot4.a")
    c0, c1 = C.apply_automorphism(a0, a1, k, kb, ka, lv, log_l, n)
    c0, c1 = C.apply_automorphism(c0, c1, C.rotation_exponent(log_n, 4), k4b, k4a, lv, log_l, n)
    assert (c0, c1) == (g.ints("rot5.c0")[0], g.ints("rot5.c1")[0])


def test_oracle_mult_plain_mask(case):
    g, log_n, log_l, log_p, log_p_small = case
    n = 1 << log_n
    a0, a1, lv = _ct(g, "ct_a")
    m, mbits = g.ints("mask_slot3")
    p0, p1 = C.mult_plain(a0, a1, m, mbits, lv, n)
    r0, r1 = C.rescale(p0, p1, log_p_small, lv)
    assert (r0, r1) == (g.ints("mult_plain_mask.c0")[0], g.ints("mult_plain_mask.c1")[0])


def test_oracle_decrypt_unit(golden):
    g = golden("unit_ops")
    log_n, *_ = g.params_tuple()
    n = 1 << log_n
    c0, c1, lv = _ct(g, "eng_mult")
    s, sbits = g.ints("sk.s")
    s_l = R.reduce_to(s, lv)
    m = R.add(c0, R.mul(c1, s_l, lv, n), lv)
    assert m == g.ints("decrypt_eng_mult")[0]


@pytest.mark.parametrize("name", ["gwas_toy", "gwas_toy_ragged", "gwas_toy_real"])
def test_replay_oracle_matches_reference_encrypted_run(golden, name):
    """The float64 replay of the approximate circuit (oracle/replay.py) agrees with the
    reference's decrypted encrypted-GWAS statistics (~1e-8), for a full batch,
    a ragged last batch and real packing."""
    import numpy as np

    from oracle.replay import replay_gwas

    g = golden(name)
    rep = replay_gwas(g.arr("X"), g.arr("y"), g.arr("S"))
    num, den = g.arr("num"), g.arr("den")
    assert np.max(np.abs(rep["numerator"] - num)) < 1e-6
    assert np.max(np.abs(rep["denominator"] - den)) < 1e-6


def test_cleartext_oracles_restate_reference_definitions():
    """oracle_modified is the replay with the exact 1/w (Newton from a good guess converges to
    it); oracle_original equals oracle_modified when W is constant (weighted == unweighted
    projector); accuracy() counts as the paper's methodology does."""
    import numpy as np

    from oracle.replay import accuracy, oracle_modified, oracle_original, replay_gwas
    from paper_1902_04303_b200.data import synth_gwas_dataset

    ds = synth_gwas_dataset(60, 4, 12, seed=9)
    rep = replay_gwas(ds.X, ds.y, ds.S, inverse_iters=40, guess=1.0)
    num, den = oracle_modified(ds.X, ds.y, ds.S, rep["beta"], rep["p"])
    assert np.allclose(num, rep["numerator"], rtol=1e-9) and np.allclose(den, rep["denominator"], rtol=1e-9)
    p_const = np.full(60, 0.3)
    a = oracle_modified(ds.X, ds.y, ds.S, rep["beta"], p_const)
    b = oracle_original(ds.X, ds.y, ds.S, rep["beta"], p_const)
    assert np.allclose(a[0], b[0]) and np.allclose(a[1], b[1])
    rep_acc = accuracy([0.0, 1.0, 2.0], [0.0, 1.02, 2.2])
    assert rep_acc["above"] == {"0.1": 1, "0.01": 2, "0.005": 2}


@pytest.mark.parametrize("case", ["n13_l240", "n13_l1440"])
def test_oracle_against_reference_hashes_at_n8192(case):
    """The oracle at N=2^13 against the reference-run hashes of tests/golden/scale_hashes.json
    (tools/make_scale_golden.py): rescale and mult_plain + rescale of the seeded inputs."""
    import hashlib
    import json
    import os

    from paper_1902_04303_b200.encoding import encode_coefficients, mask_vector
    from paper_1902_04303_b200.params import CkksParams
    from tests.golden_io import HERE, random_words, words_to_ints

    g = json.load(open(os.path.join(HERE, "golden", "scale_hashes.json")))[case]
    params = CkksParams(log_n=g["log_n"], log_l=g["log_l"], log_p=g["log_p"],
                        log_p_small=g["log_p_small"], h=g["h"])
    n, lv, seed = params.n, g["level"], g["seed"]
    a0 = words_to_ints(random_words((seed, lv, 0, 0), lv, n))
    a1 = words_to_ints(random_words((seed, lv, 0, 1), lv, n))

    def sha(*polys_bits):
        from tests.golden_io import ints_to_words

        h = hashlib.sha256()
        for coeffs, bits in polys_bits:
            h.update(ints_to_words(coeffs, bits).tobytes())
        return h.hexdigest()

    r0, r1 = C.rescale(a0, a1, 30, lv)
    assert sha((r0, lv - 30), (r1, lv - 30)) == g["outputs"]["rescale30_a"]["sha256"]
    mask = [c % (1 << params.log_l) for c in
            encode_coefficients(mask_vector(("range", 0, 256), params.slot_count), params.log_p_small, params)]
    m0, m1 = C.mult_plain(a0, a1, mask, params.log_l, lv, n)
    p0, p1 = C.rescale(m0, m1, params.log_p_small, lv)
    out_bits = lv - params.log_p_small
    assert sha((p0, out_bits), (p1, out_bits)) == g["outputs"]["mult_plain_range_a"]["sha256"]

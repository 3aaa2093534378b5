"""Drop-in check: the GPU package imported under the reference's name, used exactly as a
`hegwas` caller would (top-level names of hegwas/__init__.py:4-96 and the behaviours the
reference's own unit tests hold for them: tests/test_ckks.py and tests/test_matrix.py of the
reference package) -- keygen shape and determinism, the encrypt / decrypt noise bound, the
additive and multiplicative homomorphisms with their level / scale bookkeeping, rotation and
conjugation, the error classes for misaligned or exhausted ciphertexts and missing keys, op
tracking, and the matrix layer (replicate, duplicate, col_sum, cp_matvec, dot_prod).  Every
ring operation behind these names runs in libhegwas_b200.so."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hegwas():
    import paper_1902_04303_b200 as hegwas

    return hegwas


@pytest.fixture(scope="module")
def unit(hegwas):
    params = hegwas.CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)
    sk, pk, evk, rot = hegwas.keygen(params, seed=7)
    return params, sk, pk, evk, rot, hegwas.HeEngine(params, evk, rot)


def _vec(seed, n):
    g = np.random.default_rng(seed)
    return g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n)


def _err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


def test_keygen_shapes_and_determinism(hegwas, unit):
    params, sk, pk, evk, rot, _ = unit
    nz = [c for c in sk.s.centered() if c]
    assert len(nz) == params.h and set(nz) <= {-1, 1}
    assert evk.b.mod_bits == 2 * params.log_l
    assert set(rot.keys) == {1 << j for j in range((params.n // 4).bit_length())}
    again = hegwas.keygen(params, seed=7)
    assert again[0].s == sk.s and again[1].b == pk.b and again[2].a == evk.a
    assert hegwas.keygen(params, seed=8)[0].s != sk.s
    with pytest.raises(hegwas.ParameterError):
        hegwas.CkksParams(log_n=4, log_l=120, log_p=45, log_p_small=10, h=99)


def test_encrypt_decrypt_noise_bound(hegwas, unit):
    params, sk, pk, *_ = unit
    rng = random.Random(0)
    worst = 0.0
    for t in range(20):
        v = _vec(t, params.slot_count)
        ct = hegwas.encrypt_values(v, 45, pk, params, rng)
        worst = max(worst, _err(hegwas.decrypt_values(ct, sk), v))
    assert worst < 2.0 ** (-(45 - params.log_n - 4))


def test_wrong_key_and_exhausted_budget(hegwas, unit):
    params, sk, pk, *_ = unit
    v = _vec(1, params.slot_count)
    ct = hegwas.encrypt_values(v, 45, pk, params, random.Random(1))
    other = hegwas.keygen(params, seed=999)[0]
    assert np.max(np.abs(hegwas.decrypt_values(ct, other) - v)) > 1.0
    low = hegwas.mod_down(ct, 45)
    assert _err(hegwas.decrypt_values(low, sk), v) < 1e-6
    from dataclasses import replace

    with pytest.raises(hegwas.BudgetDepletedError):
        hegwas.decrypt(replace(low, scale_bits=46), sk)


def test_additive_ops_and_alignment(hegwas, unit):
    params, sk, pk, *_ = unit
    rng = random.Random(2)
    v, w = _vec(2, params.slot_count), _vec(3, params.slot_count)
    a = hegwas.encrypt_values(v, 45, pk, params, rng)
    b = hegwas.encrypt_values(w, 45, pk, params, rng)
    assert _err(hegwas.decrypt_values(hegwas.add(a, b), sk), v + w) < 1e-9
    assert np.max(np.abs(hegwas.decrypt_values(hegwas.sub(a, a), sk))) == 0.0
    assert _err(hegwas.decrypt_values(hegwas.negate(a), sk), -v) < 1e-9
    four = hegwas.mult_integer(a, 4)
    assert (four.level_bits, four.scale_bits) == (a.level_bits, a.scale_bits)
    assert _err(hegwas.decrypt_values(four, sk), 4 * v) < 1e-8
    with pytest.raises(hegwas.AlignmentError):
        hegwas.add(a, hegwas.mod_down(b, 200))


def test_mult_rescale_bookkeeping(hegwas, unit):
    params, sk, pk, evk, *_ = unit
    rng = random.Random(3)
    a = hegwas.encrypt_values([2.0, 3.0], 45, pk, params, rng)
    b = hegwas.encrypt_values([4.0, 5.0], 45, pk, params, rng)
    m = hegwas.rescale(hegwas.mult(a, b, evk), 45)
    got = hegwas.decrypt_values(m, sk).real
    assert abs(got[0] - 8.0) < 1e-5 and abs(got[1] - 15.0) < 1e-5
    assert m.level_bits == a.level_bits - 45 and m.scale_bits == 45
    pt = hegwas.encode([10.0, 10.0], 30, params)
    out = hegwas.rescale(hegwas.mult_plain(a, pt), 30)
    got = hegwas.decrypt_values(out, sk).real
    assert abs(got[0] - 20.0) < 1e-5 and abs(got[1] - 30.0) < 1e-5
    assert out.level_bits == a.level_bits - 30 and out.scale_bits == 45


def test_rotation_and_conjugation(hegwas, unit):
    params, sk, pk, evk, rot, eng = unit
    v = _vec(4, params.slot_count)
    ct = hegwas.encrypt_values(v, 45, pk, params, random.Random(4))
    for r in (1, 2, 5, params.slot_count - 1):   # right rotations, one key switch per set bit
        got = hegwas.decrypt_values(hegwas.rotate(ct, r, rot), sk)
        assert _err(got, np.roll(v, r)) < 1e-6, r
        assert _err(hegwas.decrypt_values(eng.rotate(ct, r), sk), got) < 1e-9
    half = params.slot_count // 2
    back = hegwas.rotate(hegwas.rotate(ct, half, rot), half, rot)
    assert _err(hegwas.decrypt_values(back, sk), v) < 1e-6
    conj = hegwas.conjugate(ct, rot.conj_key())
    assert _err(hegwas.decrypt_values(conj, sk), np.conj(v)) < 1e-6
    twice = hegwas.conjugate(conj, rot.conj_key())
    assert _err(hegwas.decrypt_values(twice, sk), v) < 1e-6


def test_missing_key_raises(hegwas, unit):
    from paper_1902_04303_b200.keys import RotationKeySet

    params, sk, pk, evk, rot, _ = unit
    ct = hegwas.encrypt_values([1.0], 45, pk, params, random.Random(5))
    with pytest.raises(hegwas.MissingKeyError):
        hegwas.rotate(ct, 1, RotationKeySet(keys={}, conj=None))


def test_track_ops_counts(hegwas, unit):
    params, sk, pk, evk, rot, eng = unit
    rng = random.Random(6)
    a = hegwas.encrypt_values([0.1], 45, pk, params, rng)
    b = hegwas.encrypt_values([0.2], 45, pk, params, rng)
    with hegwas.track_ops() as ops:
        hegwas.mult(a, b, evk)
        hegwas.rotate(a, 5, rot)        # 5 = 101b: two key switches
    assert ops.ct_mults == 1 and ops.rotations == 2 and ops.keyswitches == 3
    assert ops.rotation_amounts == [1, 4]


def test_matrix_layer(hegwas, unit):
    params, sk, pk, evk, rot, eng = unit
    slots = params.slot_count
    rng = random.Random(7)
    v = np.zeros(slots)
    v[:8] = np.arange(1, 9) / 10
    ct = hegwas.encrypt_values(v, 45, pk, params, rng)
    reps = hegwas.replicate(eng, ct, 3)
    for i, r in enumerate(reps):
        assert _err(hegwas.decrypt_values(r, sk).real, np.full(slots, v[i])) < 1e-4
    dup = hegwas.duplicate(eng, ct, 8)
    assert _err(hegwas.decrypt_values(dup, sk).real, np.tile(v[:8], slots // 8)) < 1e-5
    a = np.arange(16, dtype=float).reshape(4, 4) / 20
    x = np.array([0.3, -0.2, 0.1, 0.4])
    cp = hegwas.pack_cp(a, pk, params, rng)
    xv = np.zeros(slots)
    xv[:4] = x
    got = hegwas.decrypt_values(hegwas.cp_matvec(eng, cp, hegwas.encrypt_values(xv, 45, pk, params, rng)), sk).real
    assert _err(got[:4], a @ x) < 1e-3
    w = np.zeros(slots)
    w[:4] = [0.5, 0.25, -0.5, 1.0]
    d = hegwas.dot_prod(eng, hegwas.encrypt_values(xv, 45, pk, params, rng),
                        hegwas.encrypt_values(w, 45, pk, params, rng), 4)
    assert abs(hegwas.decrypt_values(d, sk).real[0] - float(x @ w[:4])) < 1e-4

"""Error behaviour of the drop-in API: the same exception classes the reference raises for the
same misuse (hegwas/ckks.py:60-279, keys.py:45-54, matrix.py:79-218, logreg.py:54-80; the
reference's own tests test_ckks.py / test_matrix.py check these classes).  Checks run on
metadata before any launch, so a failing call leaves no GPU work behind."""
import random
from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import paper_1902_04303_b200 as hg

    params = hg.CkksParams(log_n=8, log_l=350, log_p=45, log_p_small=30, h=16)
    sk, pk, evk, rot = hg.keygen(params, seed=9)
    return hg, params, sk, pk, evk, rot, hg.HeEngine(params, evk, rot)


def _enc(env, vals, seed):
    hg, params, sk, pk, *_ = env
    return hg.encrypt_values(vals, params.log_p, pk, params, random.Random(seed))


def test_alignment_errors(env):
    hg, params, *_ = env
    a = _enc(env, [0.1], 1)
    b = hg.mod_down(_enc(env, [0.2], 2), 200)
    with pytest.raises(hg.AlignmentError):
        hg.add(a, b)
    with pytest.raises(hg.AlignmentError):
        hg.sub(a, b)
    with pytest.raises(hg.AlignmentError):      # same level, different scale
        hg.add(a, replace(_enc(env, [0.3], 3), scale_bits=40))
    with pytest.raises(hg.AlignmentError):
        hg.mod_down(b, 300)                     # mod_down cannot raise the level
    out = hg.add(hg.mod_down(a, 200), b)        # aligned: fine
    assert out.level_bits == 200


def test_budget_errors(env):
    hg, params, sk, pk, evk, rot, eng = env
    ct = _enc(env, [0.5], 4)
    with pytest.raises(hg.BudgetDepletedError):
        hg.mod_down(ct, 44)                     # below the scale floor
    low = hg.mod_down(ct, 45)
    assert abs(hg.decrypt_values(low, sk)[0] - 0.5) < 1e-6   # level == scale still decrypts
    with pytest.raises(hg.BudgetDepletedError):
        hg.decrypt_values(replace(low, scale_bits=46), sk)  # exhausted
    with pytest.raises(hg.BudgetDepletedError):
        hg.rescale(ct, 400)                     # more than the level
    with pytest.raises(hg.BudgetDepletedError):
        hg.rescale(ct, 45)                      # would destroy the scale
    with pytest.raises(hg.ParameterError):
        hg.rescale(ct, -1)
    with pytest.raises(hg.BudgetDepletedError):
        eng.mult(hg.mod_down(ct, 60), hg.mod_down(ct, 60))
    chain = ct
    steps = (params.log_l - params.log_p) // params.log_p
    for _ in range(steps):
        chain = eng.mult(chain, chain)
    with pytest.raises(hg.BudgetDepletedError):
        eng.mult(chain, chain)


def test_missing_rotation_key(env):
    from paper_1902_04303_b200.keys import RotationKeySet

    hg, params, sk, pk, evk, rot, eng = env
    ct = _enc(env, [1.0], 5)
    bare = hg.HeEngine(params, evk, RotationKeySet(keys={}, conj=None))
    with pytest.raises(hg.MissingKeyError):
        bare.rotate(ct, 1)
    with pytest.raises(hg.MissingKeyError):
        bare.conjugate(ct)


def test_matrix_dimension_errors(env):
    from paper_1902_04303_b200 import matrix as mx

    hg, params, sk, pk, evk, rot, eng = env
    rng = random.Random(6)
    a = mx.pack_cp(np.ones((4, 3)), pk, params, rng)
    b = mx.pack_cp(np.ones((2, 2)), pk, params, rng)
    with pytest.raises(hg.DimensionError):
        mx.cp_matmul(eng, a, b)                 # inner dimensions differ
    with pytest.raises(hg.DimensionError):
        mx.replicate(eng, a.cols[0], params.slot_count + 1)
    with pytest.raises(hg.DimensionError):
        mx.CPMatrix(cols=a.cols[:2], rows=4, cols_logical=3)
    rep = mx.pack_rep(np.ones((3, 2)), 2, pk, params, rng)
    with pytest.raises(hg.DimensionError):
        mx.cp_rep_matmul(eng, a, rep)           # repeat != padded column height


def test_logreg_and_config_errors(env):
    from paper_1902_04303_b200.gwas import GwasConfig
    from paper_1902_04303_b200.logreg import hom_logreg

    hg, params, *_ = env
    with pytest.raises(hg.InputError):
        hom_logreg(env[-1], None, 0)
    with pytest.raises(hg.ParameterError):      # projector needs next_pow2(n) * n slots
        GwasConfig(n=20, d=2, k=4).resolve(params)

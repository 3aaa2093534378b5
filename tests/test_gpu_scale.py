"""BASELINE config 4 (paper_1902_04303_b200/gwas_scale.py): the projector-free encrypted GWAS
on the GPU at a small shape (n=200, d=4, k=100, N=2^12, block 32).  No reference execution
exists for config 4: the decrypted numerators / denominators are checked against
the float64 replay of the reference's approximate circuit (oracle/replay.replay_gwas), which
the reformulation equals algebraically (tests/test_host.py::test_scale_gwas_layout_and_identity)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fused", [True, False])
def test_scale_gwas_matches_replay(fused):
    import paper_1902_04303_b200 as hg
    from oracle.replay import replay_gwas
    from paper_1902_04303_b200.data import synth_gwas_dataset
    from paper_1902_04303_b200.gwas_scale import (ScaleConfig, compute_scale_gwas, decrypt_scale_statistics,
                                                  encrypt_scale_inputs)

    params = hg.CkksParams(log_n=12, log_l=1700, log_p=40, log_p_small=30, h=64)
    sk, pk, evk, rot = hg.keygen(params, seed=21)
    eng = hg.HeEngine(params, evk, rot)
    ds = synth_gwas_dataset(200, 4, 100, seed=4)
    cfg = ScaleConfig(n=200, d=4, k=100, block=32)
    inputs = encrypt_scale_inputs(ds.X, ds.y, ds.S, cfg, params, pk, random.Random(5))
    setup, outs = compute_scale_gwas(eng, inputs, fused=fused)
    assert len(outs) == 2
    num, den, res = decrypt_scale_statistics(outs, cfg, params, sk)
    ref = replay_gwas(ds.X, ds.y, ds.S)
    assert np.max(np.abs(num - ref["numerator"])) < 1e-3
    assert np.max(np.abs(den - ref["denominator"]) / np.abs(ref["denominator"])) < 1e-4
    assert min(o.num_ct.level_bits for o in outs) > 0
    # intermediates decrypt to the replay's
    beta = hg.decrypt_values(setup.beta, sk).real[:5]
    assert np.max(np.abs(beta - ref["beta"])) < 1e-4
    zp = hg.decrypt_values(setup.z_prime, sk).real[:200]
    assert np.max(np.abs(zp - ref["z_prime"])) < 1e-3


def test_encode_device_matches_host_encode():
    """The GPU encoder (config-4 client simulation) agrees with the reference-exact host
    encoder to within one unit per coefficient (cuFFT vs pocketfft rounding) and decrypts
    to the input."""
    import torch

    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.encoding import encode, encode_device

    params = hg.CkksParams(log_n=12, log_l=600, log_p=40, log_p_small=30, h=64)
    vals = np.random.default_rng(0).standard_normal(params.slot_count) * 3
    a = encode_device(vals, params.log_p, params).m.coeffs
    b = encode(vals, params.log_p, params).m.coeffs
    half, full = 1 << (params.log_l - 1), 1 << params.log_l
    diff = [((x - y + half) % full) - half for x, y in zip(a, b)]
    assert max(abs(d) for d in diff) <= 1
    sk, pk, evk, rot = hg.keygen(params, seed=2)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1)
    ct = hg.encrypt(encode_device(vals, params.log_p, params), pk, params, gen)
    assert np.max(np.abs(hg.decrypt_values(ct, sk).real - vals)) < 1e-6

"""Decrypted GWAS statistics of the GPU pipeline at larger scale vs the float64 replay of the
approximate circuit (oracle/replay.py, pinned to the reference by test_oracle_golden.py).
Target from BASELINE.json: <= 1e-3 absolute agreement of the decrypted outputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(n, k, log_n, seed=0):
    import torch

    import paper_1902_04303_b200 as hg
    from oracle.replay import finalize, replay_gwas
    from paper_1902_04303_b200.data import synth_gwas_dataset
    from paper_1902_04303_b200.gwas import (
        GwasConfig,
        assemble_result,
        compute_gwas_encrypted,
        decrypt_statistics,
        encrypt_gwas_inputs,
    )

    params = hg.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 11, device_rng=True)
    ds = synth_gwas_dataset(n, 4, k, seed=seed)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed + 5)
    config = GwasConfig(n=n, d=4, k=k).resolve(params)
    enc = encrypt_gwas_inputs(ds, config, params, pk, gen)
    with hg.track_ops() as ops:
        out = compute_gwas_encrypted(hg.HeEngine(params, evk, rot), enc)
    _run.last_ops = ops.snapshot()
    num, den = decrypt_statistics(out.batch_outputs, config, params, sk)
    res = assemble_result(num, den)
    rep = replay_gwas(ds.X, ds.y, ds.S)
    eff, se, pv = finalize(rep["numerator"], rep["denominator"])
    return num, den, res, rep, eff, se, pv


def test_replay_agreement_n64_k256():
    num, den, res, rep, eff, se, pv = _run(64, 256, 13)
    assert np.max(np.abs(num - rep["numerator"])) < 1e-3
    assert np.max(np.abs(den - rep["denominator"])) < 1e-3
    ok = np.isfinite(eff)
    assert np.max(np.abs(res.effects[ok] - eff[ok])) < 1e-3
    assert np.max(np.abs(res.std_err[ok] - se[ok])) < 1e-3
    assert np.max(np.abs(res.p_values[ok] - pv[ok])) < 1e-3


@pytest.mark.slow
def test_replay_agreement_config0_p17():
    """Config 0 at the parity preset P17: n=245, d=4, 256 SNPs, N=2^17, log_l=1700."""
    num, den, res, rep, eff, se, pv = _run(245, 256, 17)
    # exact op-count contract of the reference at config-0 shape (dry run)
    assert _run.last_ops == {"ct_mults": 596, "pt_mults": 577, "rotations": 8191,
                             "conjugations": 1, "keyswitches": 8788, "rescales_ct": 596,
                             "rescales_pt": 577}
    assert np.max(np.abs(num - rep["numerator"])) < 1e-3
    assert np.max(np.abs(den - rep["denominator"])) < 1e-3
    ok = np.isfinite(eff)
    assert np.max(np.abs(res.effects[ok] - eff[ok])) < 1e-3
    assert np.max(np.abs(res.p_values[ok] - pv[ok])) < 1e-3

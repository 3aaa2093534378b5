"""End-to-end parity of the encrypted GWAS pipeline (logistic regression, projector,
per-batch statistics) against the reference run captured in tests/golden/gwas_toy.npz
(n=8, d=4, k=16, log_n=7, log_l=1700, log_p_small=30; SURVEY §4 item iii)."""
import random

import numpy as np
import pytest

from tests.gpu_helpers import assert_ct_equal, ct_from, params_from, ring_hash

pytestmark = pytest.mark.gpu


def _complex(g) -> bool:
    return bool(int(g.arr("complex_packing"))) if "complex_packing" in g else True


# gwas_toy: k=16 = one full batch; gwas_toy_ragged: k=21 = 16 + 5 SNPs (a partial batch whose
# last complex column carries one SNP); gwas_toy_real: real packing, k=11 = 8 + 3
@pytest.fixture(scope="module", params=["gwas_toy", "gwas_toy_ragged", "gwas_toy_real"])
def toy(request, golden):
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.data import CleartextDataset
    from paper_1902_04303_b200.gwas import GwasConfig

    g = golden(request.param)
    params = params_from(g)
    n, d, k, seed, key_seed = (int(x) for x in g.arr("shape"))
    sk, pk, evk, rot = hg.keygen(params, key_seed)
    ds = CleartextDataset(X=g.arr("X"), S=g.arr("S"), y=g.arr("y"))
    tau = int(g.arr("tau")) if "tau" in g and int(g.arr("tau")) else None
    config = GwasConfig(n=n, d=d, k=k, complex_packing=_complex(g), tau=tau).resolve(params)
    return g, params, (sk, pk, evk, rot), ds, config, seed


def _golden_inputs(g, params, config):
    from paper_1902_04303_b200.gwas import EncryptedGwasInputs, SnpBatch
    from paper_1902_04303_b200.logreg import LogRegInputs
    from paper_1902_04303_b200.matrix import CPMatrix, REPMatrix, next_pow2

    n, d = config.n, config.d
    cs = next_pow2(n)
    X = CPMatrix(cols=[ct_from(g, f"in.X{j}", params) for j in range(d + 1)], rows=n,
                 cols_logical=d + 1)
    Xt = REPMatrix(rows_ct=[ct_from(g, f"in.Xt{j}", params) for j in range(d + 1)], repeat=cs,
                   rows=d + 1, cols_logical=n)
    XtXinv = CPMatrix(cols=[ct_from(g, f"in.XtXinv{j}", params) for j in range(d + 1)],
                      rows=d + 1, cols_logical=d + 1)
    y = ct_from(g, "in.y", params)
    batches = []
    for bi in range(int(g.arr("n_batches"))):
        offset = bi * config.tau
        count = min(config.tau, config.k - offset)
        ncols = (count + 1) // 2 if config.complex_packing else count
        rows = [ct_from(g, f"in.b{bi}.S{j}", params) for j in range(n)]
        batches.append(SnpBatch(index=bi, S_packed=REPMatrix(rows_ct=rows, repeat=cs, rows=n,
                                                            cols_logical=ncols),
                                snp_offset=offset, snp_count=count, complex_packing=config.complex_packing))
    return EncryptedGwasInputs(logreg=LogRegInputs(X=X, Xt_rep=Xt, XtX_inv=XtXinv, y=y),
                               batches=batches, config=config)


def test_toy_keys_match_reference(toy):
    g, params, (sk, pk, evk, rot), *_ = toy
    want = g.key_hashes()
    got = {"sk.s": ring_hash(sk.s), "pk.b": ring_hash(pk.b), "pk.a": ring_hash(pk.a),
           "evk.b": ring_hash(evk.b), "evk.a": ring_hash(evk.a)}
    assert got == want


def test_toy_encryption_matches_reference(toy):
    from paper_1902_04303_b200.gwas import encrypt_gwas_inputs

    g, params, (sk, pk, evk, rot), ds, config, seed = toy
    enc = encrypt_gwas_inputs(ds, config, params, pk, random.Random(seed))
    for j, c in enumerate(enc.logreg.X.cols):
        assert_ct_equal(c, g, f"in.X{j}")
    for j, c in enumerate(enc.logreg.Xt_rep.rows_ct):
        assert_ct_equal(c, g, f"in.Xt{j}")
    assert_ct_equal(enc.logreg.y, g, "in.y")
    for bi, batch in enumerate(enc.batches):
        for j, c in enumerate(batch.S_packed.rows_ct):
            assert_ct_equal(c, g, f"in.b{bi}.S{j}")


def test_toy_pipeline_bit_exact(toy):
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.gwas import assemble_result, compute_gwas_encrypted, decrypt_statistics

    g, params, (sk, pk, evk, rot), ds, config, seed = toy
    enc = _golden_inputs(g, params, config)
    engine = hg.HeEngine(params, evk, rot)
    with hg.track_ops() as ops:
        out = compute_gwas_encrypted(engine, enc)
    names = [str(s) for s in g.arr("op_count_names")]
    assert ops.snapshot() == dict(zip(names, [int(x) for x in g.arr("op_counts")]))
    assert ops.rotation_amounts == [int(x) for x in g.arr("rotation_amounts")]
    assert_ct_equal(out.beta, g, "out.beta")
    assert_ct_equal(out.p_prev, g, "out.p_prev")
    inter = out.intermediates
    for name in ("w", "w_inv", "z", "z_prime"):
        assert_ct_equal(getattr(inter, name), g, f"out.{name}")
    for j, c in enumerate(inter.M.cols):
        assert_ct_equal(c, g, f"out.M{j}")
    for bo in out.batch_outputs:
        assert_ct_equal(bo.num_ct, g, f"out.b{bo.index}.num")
        assert_ct_equal(bo.den_even_ct, g, f"out.b{bo.index}.den_even")
        if config.complex_packing:
            assert_ct_equal(bo.den_odd_ct, g, f"out.b{bo.index}.den_odd")
        else:
            assert bo.den_odd_ct is None
    num, den = decrypt_statistics(out.batch_outputs, config, params, sk)
    assert np.array_equal(num, g.arr("num"))
    assert np.array_equal(den, g.arr("den"))
    res = assemble_result(num, den)
    assert np.all(np.isfinite(res.effects[den > 0]))


def test_toy_pipeline_streamed_batches_bit_exact(toy):
    """The same pipeline with the SNP batches uploaded from pinned host memory by
    SnpBatchStream (side-stream copies, per-row ready events, two device slots reused across
    batches) reproduces the reference's per-batch outputs."""
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.gwas import HostSnpBatch, SnpBatchStream, compute_gwas_encrypted

    g, params, (sk, pk, evk, rot), ds, config, seed = toy
    enc = _golden_inputs(g, params, config)
    host = [HostSnpBatch.from_device(b) for b in enc.batches]
    # three passes over the batches so both device slots are reused while the next one loads;
    # then the rows streamed only at the projector's level (mod_down on upload)
    m_level = g.meta("out.M0")["level_bits"]
    # ... and a ring of three slots whose first uploads are issued before the setup runs
    # (early="manual"), or by compute_gwas_encrypted before the setup's M_dup stage (early=True)
    for level, slots, early in ((None, 2, False), (m_level, 2, False), (m_level, 3, "manual"),
                                (m_level, 4, True)):
        stream = SnpBatchStream(host * 3, params, level=level, slots=slots, early=early is True)
        if early == "manual":
            stream.start()
        out = compute_gwas_encrypted(hg.HeEngine(params, evk, rot), enc, cache=stream)
        assert len(out.batch_outputs) == 3 * len(host)
        for bo in out.batch_outputs:
            assert_ct_equal(bo.num_ct, g, f"out.b{bo.index}.num")
            assert_ct_equal(bo.den_even_ct, g, f"out.b{bo.index}.den_even")
            if config.complex_packing:
                assert_ct_equal(bo.den_odd_ct, g, f"out.b{bo.index}.den_odd")


def test_batch_keys_prepared_by_the_setup(toy):
    """gwas.batch_key_plan names every (switching key, level) the batch loop uses: after the
    setup (which prepares them) a batch makes no further key preparation."""
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200.ckks import KEY_CACHE
    from paper_1902_04303_b200.gwas import compute_batch, compute_setup

    g, params, (sk, pk, evk, rot), ds, config, seed = toy
    enc = _golden_inputs(g, params, config)
    engine = hg.HeEngine(params, evk, rot)
    beta, p_prev, inter, m_dup = compute_setup(engine, enc)
    misses = KEY_CACHE.misses
    for batch in enc.batches:
        bo = compute_batch(engine, enc, inter, m_dup, batch)
        assert_ct_equal(bo.num_ct, g, f"out.b{bo.index}.num")
    assert KEY_CACHE.misses == misses


def test_projector_duplicated_in_column_groups(toy, monkeypatch):
    """compute_setup runs the M_dup ladders and prepares column group by column group
    (gwas.DUP_GROUP); groups of 3 over the toy's 8 columns (3 + 3 + 2) give the reference's op
    counts, rotation order and batch outputs, and HostSnpBatch.to_device round-trips a batch."""
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200 import gwas
    from paper_1902_04303_b200.gwas import HostSnpBatch, compute_gwas_encrypted

    g, params, (sk, pk, evk, rot), ds, config, seed = toy
    enc = _golden_inputs(g, params, config)
    enc.batches = [HostSnpBatch.from_device(b).to_device(params) for b in enc.batches]
    monkeypatch.setattr(gwas, "DUP_GROUP", 3)
    with hg.track_ops() as ops:
        out = compute_gwas_encrypted(hg.HeEngine(params, evk, rot), enc)
    names = [str(s) for s in g.arr("op_count_names")]
    assert ops.snapshot() == dict(zip(names, [int(x) for x in g.arr("op_counts")]))
    assert ops.rotation_amounts == [int(x) for x in g.arr("rotation_amounts")]
    for bo in out.batch_outputs:
        assert_ct_equal(bo.num_ct, g, f"out.b{bo.index}.num")
        assert_ct_equal(bo.den_even_ct, g, f"out.b{bo.index}.den_even")
        if config.complex_packing:
            assert_ct_equal(bo.den_odd_ct, g, f"out.b{bo.index}.den_odd")

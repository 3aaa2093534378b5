"""CPU-only tests: the native library's exported surface, host logic (params, counters,
GWAS configuration), and host-side algorithms that must be bit-identical to the
reference (encoding, samplers) checked against the golden fixtures."""
import math
import os
import random
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    import ctypes

    from paper_1902_04303_b200 import _lib

    header = open(os.path.join(ROOT, "include", "hegwas_b200.h")).read()
    declared = set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", header))
    assert len(declared) >= 25
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(_lib.SIGNATURES) == declared
    assert _lib.load_library().hg_version() == 1


def test_params_validation_and_json():
    from paper_1902_04303_b200 import CkksParams, ParameterError, P17, security_status

    with pytest.raises(ParameterError):
        CkksParams(log_n=4, log_l=120, log_p=45, log_p_small=10, h=99)
    with pytest.raises(ParameterError):
        CkksParams(log_n=21, log_l=120)
    with pytest.raises(ParameterError):
        CkksParams(log_n=8, log_l=40, log_p=45)
    assert CkksParams.from_json(P17.to_json()) == P17
    with pytest.raises(ParameterError):
        CkksParams.from_json('{"log_n": 8, "log_l": 100, "bogus": 1}')
    assert security_status(P17)[0] == "accepted"
    assert security_status(CkksParams(log_n=17, log_l=2440))[0] == "warn"


def test_op_counter_nesting():
    from paper_1902_04303_b200 import instrument

    with instrument.track_ops() as outer:
        instrument.record(ct_mults=1, keyswitches=1)
        with instrument.track_ops() as inner:
            instrument.record(rotations=1, keyswitches=1, rotation_amounts=[4])
    assert outer.snapshot()["keyswitches"] == 2 and inner.snapshot()["keyswitches"] == 1
    assert outer.rotation_amounts == [4] and outer.all_rotations_power_of_two()
    c = instrument.OpCounter()
    c.merge(outer)
    assert c.snapshot() == outer.snapshot()


def test_gwas_config_capacity_rules():
    from paper_1902_04303_b200 import CkksParams, ParameterError
    from paper_1902_04303_b200.gwas import GwasConfig, default_tau

    # n=245 does not fit at log_n=16 (256 x 245 > 32768 slots)
    with pytest.raises(ParameterError):
        GwasConfig(n=245, d=4, k=256).resolve(CkksParams(log_n=16, log_l=1700, log_p_small=30))
    p17 = CkksParams(log_n=17, log_l=1700, log_p_small=30)
    cfg = GwasConfig(n=245, d=4, k=10643).resolve(p17)
    assert cfg.tau == default_tau(p17, 245) == 512
    assert cfg.num_batches == 21 and cfg.cols_per_batch == 256
    # n=6000 is beyond any supported ring
    with pytest.raises(ParameterError):
        GwasConfig(n=6000, d=4, k=100000).resolve(CkksParams(log_n=20, log_l=1700, log_p_small=30))


def test_fuse_snp_pairs_and_assemble():
    from paper_1902_04303_b200.gwas import assemble_result, fuse_snp_pairs

    s = np.arange(15, dtype=float).reshape(3, 5)
    f = fuse_snp_pairs(s)
    assert f.shape == (3, 3)
    assert np.array_equal(f.real, s[:, 0::2]) and np.array_equal(f.imag[:, :2], s[:, 1::2])
    assert np.all(f.imag[:, 2] == 0)
    res = assemble_result(np.array([1.0, 2.0, 3.0]), np.array([4.0, 0.0, -1.0]))
    assert res.effects[0] == 0.25 and math.isnan(res.effects[1]) and math.isnan(res.p_values[2])
    assert res.p_values[0] == pytest.approx(math.erfc(0.25 * 2 / math.sqrt(2)))


def test_words_roundtrip():
    from paper_1902_04303_b200.ring import ints_to_words, words_to_ints

    rng = random.Random(3)
    for bits in (1, 31, 32, 33, 350, 1700):
        vals = [rng.getrandbits(bits) for _ in range(17)] + [0, (1 << bits) - 1]
        w = ints_to_words(vals, bits)
        assert w.shape == ((bits + 31) // 32, 19)
        assert words_to_ints(w) == vals
    assert words_to_ints(ints_to_words([-1, -5], 40)) == [(1 << 40) - 1, (1 << 40) - 5]


@pytest.mark.parametrize("name", ["unit_ops", "deep_ops"])
def test_encoding_bit_identical_to_reference(golden, name):
    from paper_1902_04303_b200 import CkksParams
    from paper_1902_04303_b200.encoding import decode_coefficients, encode_coefficients
    from paper_1902_04303_b200.ring import ints_to_words

    g = golden(name)
    log_n, log_l, log_p, log_p_small, h = g.params_tuple()
    params = CkksParams(log_n=log_n, log_l=log_l, log_p=log_p, log_p_small=log_p_small, h=h)
    want, bits = g.words("encode_a")
    got = ints_to_words(encode_coefficients(g.arr("vec_a"), log_p, params), bits)
    assert np.array_equal(got, want)
    vec = np.zeros(params.slot_count)
    vec[3] = 1.0
    want, bits = g.words("mask_slot3")
    assert np.array_equal(ints_to_words(encode_coefficients(vec, log_p_small, params), bits), want)
    # decode of the reference's decrypted product
    m, mbits = g.ints("decrypt_eng_mult")
    half, full = 1 << (mbits - 1), 1 << mbits
    cen = [c - full if c > half else c for c in m]
    scale = int(g.meta("eng_mult")["scale_bits"])
    assert np.array_equal(decode_coefficients(cen, scale, params.n), g.arr("decoded_eng_mult"))


def test_samplers_reproduce_reference_keys(golden):
    """Secret and uniform key parts involve no products: check the host RNG restatement."""
    from paper_1902_04303_b200.ring import derive_rng, ints_to_words, sample_hamming, sample_uniform

    g = golden("unit_ops")
    log_n, log_l, log_p, log_p_small, h = g.params_tuple()
    n = 1 << log_n
    seed = int(g.arr("key_seed"))
    s = sample_hamming(n, h, derive_rng(seed, "secret"))
    want, bits = g.words("sk.s")
    assert np.array_equal(ints_to_words(s, bits), want)
    a_pk = sample_uniform(n, log_l, derive_rng(seed, "public"))
    want, bits = g.words("pk.a")
    assert np.array_equal(ints_to_words(a_pk, bits), want)
    a_rot = sample_uniform(n, 2 * log_l, derive_rng(seed, "switch", "rot2"))
    want, bits = g.words("rot2.a")
    assert np.array_equal(ints_to_words(a_rot, bits), want)


def test_synthetic_dataset_shapes():
    from paper_1902_04303_b200.data import synth_gwas_dataset

    ds = synth_gwas_dataset(245, 4, 256, seed=0)
    assert ds.X.shape == (245, 5) and ds.S.shape == (245, 256) and ds.y.shape == (245,)
    assert np.allclose(ds.X[:, 0], 1.0)
    assert np.allclose(ds.X[:, 1:].mean(axis=0), 0.0, atol=1e-12)
    assert set(np.unique(ds.y)) <= {0.0, 1.0}
    assert 0.2 < ds.y.mean() < 0.8


def test_mask_multi_scale_encode_is_bit_identical():
    """One FFT per mask serves every scale (encoding.encode_mask_scales): the rounded
    coefficients equal encode_float's at each scale, for every mask kind, at the ring sizes
    the pipeline uses (N=2^17 is P17)."""
    from paper_1902_04303_b200 import CkksParams
    from paper_1902_04303_b200.encoding import encode_float, encode_mask_scales, mask_vector

    for log_n, specs in [(7, [("slot", 0), ("slot", 63), ("range", 16, 32), ("range_value", 0, 8, 0.5)]),
                         (13, [("slot", 5), ("range", 0, 245), ("range", 256, 512)]),
                         (17, [("slot", 244), ("range", 2048, 2304), ("range_value", 0, 245, 0.5)])]:
        params = CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30)
        for spec in specs:
            scales = (30, 45, 10)
            got = encode_mask_scales(spec, scales, params)
            for s, host in zip(scales, got):
                want = encode_float(mask_vector(spec, params.slot_count), s, params).astype(np.int64)
                if host[0] == "compact":
                    from paper_1902_04303_b200.ring import int64_to_words
                    assert np.array_equal(host[2], int64_to_words(want, host[1])), (log_n, spec, s)
                else:
                    assert np.array_equal(host[1], want), (log_n, spec, s)


def test_mask_batch_encode_is_bit_identical():
    """Masks encoded in one 2-D FFT (encode_masks_batch) equal the per-mask encodes."""
    from paper_1902_04303_b200 import CkksParams
    from paper_1902_04303_b200.encoding import encode_mask_scales, encode_masks_batch

    params = CkksParams(log_n=14, log_l=1700, log_p=45, log_p_small=30)
    specs = [("slot", 0), ("slot", 200), ("range", 256, 512), ("range_value", 0, 245, 0.5), ("slot", 8191)]
    batch = encode_masks_batch(specs, (30, 45), params)
    for spec, got in zip(specs, batch):
        want = encode_mask_scales(spec, (30, 45), params)
        for g, w in zip(got, want):
            assert g[0] == w[0] and g[1] == w[1] and np.array_equal(g[2], w[2])


def test_setup_mask_plan_covers_pipeline_masks():
    from paper_1902_04303_b200 import P17
    from paper_1902_04303_b200.gwas import GwasConfig, setup_masks

    plan = setup_masks(GwasConfig(n=245, d=4, k=10643), P17)
    specs = [s for s, _ in plan]
    assert len(specs) == len(set(specs)) == 2 * 245 + 2
    assert all(("slot", i) in specs and ("range", 256 * i, 256 * (i + 1)) in specs for i in range(245))


def test_matrix_ext_host_algebra():
    """Host halves of the config-2 extras: generalized diagonals reproduce A v under right
    rotations (np.roll), LS sigmoid fits, and the Newton replay converges."""
    from paper_1902_04303_b200.matrix_ext import (generalized_diagonals, newton_alpha,
                                                  newton_inverse_replay, periodic_vector,
                                                  sigmoid_ls_coeffs, sigmoid_poly_eval)

    rs = np.random.default_rng(0)
    for shape in [(5, 5), (245, 5), (8, 8), (16, 4)]:
        a = rs.standard_normal(shape)
        v0 = rs.standard_normal(shape[1])
        diags, big_r, big_c = generalized_diagonals(a, 512)
        v = periodic_vector(v0, big_c, 512).real
        y = sum(d * np.roll(v, i) for i, d in enumerate(diags))
        assert np.allclose(y[:shape[0]], a @ v0)
        assert np.allclose(y[big_r:big_r + shape[0]], a @ v0)
    xs = np.linspace(-8, 8, 1001)
    errs = [np.max(np.abs(sigmoid_poly_eval(xs, sigmoid_ls_coeffs(d)) - 1 / (1 + np.exp(-xs))))
            for d in (3, 5, 7)]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.05
    # the degree-7 least-squares fit is the reference's published sigma7, reflected
    # (reference oracle.py:18-22 evaluates it at -x)
    from paper_1902_04303_b200.logreg import SIGMA7_C1, SIGMA7_C3, SIGMA7_C5, SIGMA7_C7

    assert np.allclose(sigmoid_ls_coeffs(7), [-SIGMA7_C1, -SIGMA7_C3, -SIGMA7_C5, -SIGMA7_C7], atol=2e-3)
    x = rs.standard_normal((245, 5))
    x[:, 0] = 1
    a = x.T @ np.diag(rs.uniform(0, 0.25, 245)) @ x
    e = [np.linalg.norm(newton_inverse_replay(a, newton_alpha(245, 5), k) @ a - np.eye(5)) for k in (1, 3, 6)]
    assert e[0] > e[1] > e[2]


def test_scale_gwas_layout_and_identity():
    """Config-4 reformulation (gwas_scale): the group/block slot layout makes sum_b V_b * ct_b
    plus a within-block sum equal X^T S, and the projector-free num/den identities equal the
    reference's M-based statistics (oracle/replay.replay_gwas) in float64."""
    from oracle.replay import replay_gwas
    from paper_1902_04303_b200.data import synth_gwas_dataset
    from paper_1902_04303_b200.gwas_scale import ScaleConfig, group_slots

    ds = synth_gwas_dataset(200, 4, 100, seed=3)
    cfg = ScaleConfig(n=200, d=4, k=100, block=32)
    slots = 2048
    per = slots // cfg.block
    for g in range(2):
        for a in range(5):
            acc = np.zeros(slots)
            for b in range(cfg.num_blocks()):
                v = np.zeros(cfg.block)
                seg = ds.X[b * 32:(b + 1) * 32, a]
                v[:seg.size] = seg
                acc += np.tile(v, per) * group_slots(ds.S, g, b, cfg, slots)
            got = acc.reshape(per, cfg.block).sum(axis=1)
            want = ds.X[:, a] @ ds.S[:, g * per:(g + 1) * per]
            assert np.allclose(got[:want.size], want)
    ref = replay_gwas(ds.X, ds.y, ds.S)
    x, w, zp, s = ds.X, ref["w"], ref["z_prime"], ds.S
    g_inv = np.linalg.inv(x.T @ x)
    a = w * zp
    t = x.T @ s
    c = g_inv @ t
    num = a @ s - (x @ g_inv).T @ a @ t
    den = (w @ (s * s)) - 2 * np.einsum("aj,aj->j", x.T @ (w[:, None] * s), c) \
        + np.einsum("aj,ab,bj->j", c, x.T @ (w[:, None] * x), c)
    assert np.allclose(num, ref["numerator"]) and np.allclose(den, ref["denominator"])


def test_cli_io_audit_and_manifest(tmp_path):
    """CLI host plumbing: audited atomic file access, the reference encrypt manifest read into
    a GwasConfig, and the argument parser (no GPU work)."""
    import json

    from paper_1902_04303_b200 import P17, cli
    from paper_1902_04303_b200 import io as hio

    with hio.audit_file_access() as audit:
        hio.write_json(tmp_path / "a" / "x.json", {"b": 1, "a": [1.5]})
        assert hio.read_json(tmp_path / "a" / "x.json") == {"a": [1.5], "b": 1}
        hio.write_tsv(tmp_path / "t.tsv", ["k", "v"], [("s0", 0.25)])
    assert [m for m, _ in audit] == ["write", "read", "write"]
    assert hio.read_tsv(tmp_path / "t.tsv") == (["k", "v"], [["s0", "0.25"]])
    assert not list(tmp_path.glob("**/*.tmp"))
    gold = os.path.join(ROOT, "tests", "golden", "cli_toy")
    m = json.load(open(os.path.join(gold, "encrypted", "manifest.json")))
    params = cli._load_params(os.path.join(gold, "keys"))
    cfg = cli._config_from_manifest(m, params)
    assert (cfg.n, cfg.d, cfg.k, cfg.num_batches) == (8, 4, 16, 1)
    assert len(m["files"]["batches"][0]) == 8
    args = cli.build_parser().parse_args(["keygen", "--log-n", "17", "--log-l", "1700", "--outdir", "x"])
    assert cli._params(args).log_n == P17.log_n


def test_native_samplers_replay_cpython_random():
    """The native CPython-random replay (hg_rng_ternary / hg_rng_gaussian) produces exactly the
    Python samplers' draws and leaves the generator in exactly the same state (incl. the
    cached Box-Muller spare), across the MT19937 624-word refill boundary."""
    import random as pyrandom

    from paper_1902_04303_b200 import ring

    assert ring._native_samplers()
    for seed, n in [(1, 64), (7, 1000), (123456789, 4097), (2 ** 63 + 5, 3333)]:
        a, b = pyrandom.Random(seed), pyrandom.Random(seed)
        b.random()                                   # start mid-block
        a.random()
        got = ring.sample_ternary(n, a) + ring.sample_gaussian(n, 3.2, a) + ring.sample_gaussian(n + 1, 3.2, a)
        os.environ["HG_PY_SAMPLERS"] = "1"
        try:
            want = ring.sample_ternary(n, b) + ring.sample_gaussian(n, 3.2, b) + ring.sample_gaussian(n + 1, 3.2, b)
        finally:
            del os.environ["HG_PY_SAMPLERS"]
        assert got == want, seed
        assert a.getstate() == b.getstate()
        assert a.getrandbits(64) == b.getrandbits(64) and a.gauss(0, 1) == b.gauss(0, 1)


def test_row_events_hand_out_only_issued_rows():
    """gwas._RowEvents (the ready list of a streamed batch): indexing blocks until the uploader
    thread has marked the row, and an uploader failure surfaces in the consumer."""
    import threading
    import time

    from paper_1902_04303_b200.gwas import _RowEvents

    ev = _RowEvents(["e0", "e1", "e2"])
    assert len(ev) == 3
    got = []
    t = threading.Thread(target=lambda: got.append(ev[1]))
    t.start()
    time.sleep(0.05)
    assert not got            # row 1 not issued yet
    ev.mark(0)
    time.sleep(0.05)
    assert not got
    ev.mark(1)
    t.join(timeout=5)
    assert got == ["e1"] and ev[0] == "e0"
    bad = _RowEvents(["e0"])
    bad.fail(RuntimeError("upload failed"))
    with pytest.raises(RuntimeError, match="upload failed"):
        bad[0]

"""The cluster NTT variants against the two-pass kernels of csrc/hg_ntt.cu, word for word (same
butterflies, same order, same lazy ranges): variant 1 (csrc/hg_ntt_cluster.cu, log_n 17: 8-CTA
clusters exchanging the transform once through distributed shared memory) and variant 2
(csrc/hg_ntt.cu ntt_c8l2 / intt_fused_c8l2, log_n 17 -- other sizes fall back to the two passes:
both passes in one cluster launch, the intermediate through L2) --
raw forward / inverse transforms over [B][P][N] rows with a prime offset, and every fused
NTT-domain product of the inverse (key switch x.kb / x.ka, tensor, plain product, shared factor;
batched and in place) through the scheme ops that use them at the parity preset P17 -- whose
outputs the oracle / reference-run goldens pin in test_gpu_ring.py and test_gpu_scale_parity.py
(reference: the exact product of ring.py:46-65 inside ckks.py:166-279)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _set(ctx, variant):
    from paper_1902_04303_b200 import _lib

    _lib.check(ctx.lib.hg_set_ntt_variant(ctx.handle, int(variant)))


@pytest.fixture(scope="module")
def ctx17():
    from paper_1902_04303_b200 import _lib

    ctx = _lib.get_context(17)
    yield ctx
    _set(ctx, 0)


@pytest.mark.parametrize("variant,log_n", [(1, 17), (2, 17), (2, 16)])
@pytest.mark.parametrize("from_end,rows", [(0, 5), (3, 9), (1, 4)])
def test_raw_transforms_identical(variant, log_n, from_end, rows):
    import torch

    from paper_1902_04303_b200 import _lib

    ctx = _lib.get_context(log_n)
    primes = ctx.primes()
    off = len(primes) - from_end if from_end else 0
    P = min(len(primes) - off, rows)
    n = 1 << log_n
    pr = torch.tensor([primes[off + i % P] for i in range(rows)], dtype=torch.int64, device="cuda")[:, None]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(rows)
    data = torch.randint(0, 1 << 62, (rows, n), dtype=torch.int64, device="cuda", generator=gen) % pr
    src = data.to(torch.int32).contiguous()
    outs = {}
    for cluster in (True, False):
        _set(ctx, variant if cluster else 0)
        buf = src.clone()
        _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), rows, off, ctx.stream()))
        fwd = buf.clone()
        red = ((buf.to(torch.int64) & 0xFFFFFFFF) % pr).to(torch.int32).contiguous()
        _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, red.data_ptr(), rows, off, ctx.stream()))
        outs[cluster] = (fwd, red)
    _set(ctx, 0)
    assert torch.equal(outs[True][0], outs[False][0]), "forward words differ"
    assert torch.equal(outs[True][1], outs[False][1]), "inverse words differ"
    got = (outs[True][1].to(torch.int64) & 0xFFFFFFFF) % pr
    assert torch.equal(got, (data * n) % pr), "inverse(forward(x)) != N x"


@pytest.fixture(scope="module")
def p17(ctx17):
    import torch

    import paper_1902_04303_b200 as hg

    params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 5, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    rng = np.random.default_rng(3)
    cts = [hg.mod_down(hg.encrypt_values(rng.uniform(-1, 1, params.slot_count), 45, pk, params, gen), lv)
           for lv in (1550, 1550, 1550, 230)]
    return hg, params, eng, cts


def _words(ct):
    return np.concatenate([ct.c0.numpy_words().ravel(), ct.c1.numpy_words().ravel()])


@pytest.mark.parametrize("variant", [1, 2])
def test_fused_products_identical(ctx17, p17, variant):
    hg, params, eng, (a, b, c, z) = p17
    mask = eng.mask(("range", 0, 4096))
    ops = {
        "mult": lambda: [eng.mult(a, b)],                                   # tensor + key switch
        "mult_low": lambda: [eng.mult(z, z)],
        "mult_many": lambda: eng.mult_many([a, b, c], [c, a, b]),
        "prepared_many": lambda: eng.mult_prepared_many([eng.prepare(a), eng.prepare(b)], [c, c]),
        "rotate_many": lambda: eng.rotate_many([a, b, c], 4),              # batched key switch
        "rotate_add": lambda: eng.rotate_add_many([a, z], 1),
        "conjugate": lambda: [eng.conjugate(b)],
        "mult_plain": lambda: [eng.mult_plain(a, mask)],                   # plain product
        "mult_plain_each": lambda: eng.mult_plain_each(b, [mask, eng.mask(("slot", 9))]),
    }
    for name, fn in ops.items():
        got = {}
        for cluster in (True, False):
            _set(ctx17, variant if cluster else 0)
            got[cluster] = [_words(ct) for ct in fn()]
        _set(ctx17, 0)
        assert len(got[True]) == len(got[False])
        for g, w in zip(got[True], got[False]):
            assert np.array_equal(g, w), f"{name}: cluster NTT output differs from the two-pass NTT"

"""Ring-level parity of the native kernels against the CPU oracle (oracle/ring_oracle.py,
itself pinned to the reference by tests/test_oracle_golden.py).  Mirrors the reference's
test_ring.py properties on the device, plus edge cases of the RNS/CRT engine."""
import random

import numpy as np
import pytest

from oracle import ckks_oracle as C
from oracle import ring_oracle as R

pytestmark = pytest.mark.gpu


def rnd(n, bits, seed):
    rng = random.Random(seed)
    return [rng.getrandbits(bits) for _ in range(n)]


def dev(n, bits, coeffs):
    from paper_1902_04303_b200.ring import RingElement

    return RingElement(n, bits, coeffs)


SIZES = [(4, 20), (8, 64), (16, 1), (32, 77), (64, 200), (128, 2400), (256, 350),
         (512, 1700), (512, 3400), (1024, 1700), (4096, 1440), (8192, 240), (16384, 960)]


@pytest.mark.parametrize("n,bits", SIZES)
def test_mul_matches_oracle(n, bits):
    a, b = rnd(n, bits, 1), rnd(n, bits, 2)
    assert dev(n, bits, a).mul(dev(n, bits, b)).coeffs == R.mul(a, b, bits, n)


@pytest.mark.parametrize("n,bits", SIZES[:8])
def test_elementwise_matches_oracle(n, bits):
    a, b = rnd(n, bits, 3), rnd(n, bits, 4)
    A, B = dev(n, bits, a), dev(n, bits, b)
    assert A.add(B).coeffs == R.add(a, b, bits)
    assert A.sub(B).coeffs == R.sub(a, b, bits)
    assert A.neg().coeffs == R.neg(a, bits)
    for k in (3, -1, 4, 1 << 45, -(1 << 70) + 12345):
        assert A.scalar_mul(k).coeffs == R.scalar_mul(a, k, bits)
    for k in (5, 2 * n - 1, 25, 3):
        assert A.automorphism(k).coeffs == R.automorphism(a, k, bits)
    if bits > 8:
        assert A.reduce_to(bits - 7).coeffs == R.reduce_to(a, bits - 7)
    assert A.lift_centered_to(bits + 77).coeffs == R.lift_centered_to(a, bits, bits + 77)
    for sh in (s for s in (0, 1, 31, 32, 33, 45, 64) if s < bits):
        assert A.divide_round(sh, bits - sh).coeffs == R.divide_round(a, sh, bits - sh)


def test_extreme_coefficients():
    # zero polynomial, all-ones coefficients, top-bit patterns (wrap and sign handling)
    for n, bits in ((64, 350), (2048, 1700)):
        full = (1 << bits) - 1
        half = 1 << (bits - 1)
        patterns = [[0] * n, [full] * n, [half] * n, [half + 1] * n,
                    [full if i % 2 else 0 for i in range(n)]]
        for pa in patterns:
            for pb in patterns[1:]:
                got = dev(n, bits, pa).mul(dev(n, bits, pb)).coeffs
                assert got == R.mul(pa, pb, bits, n)


def test_mul_mod_wider_output_and_small_operand():
    n, bits = 512, 600
    a = rnd(n, bits, 5)
    kb = rnd(n, 2 * bits, 6)
    out_bits = bits + 333
    got = dev(n, bits, a).mul_mod(dev(n, 2 * bits, kb).reduce_to(out_bits), out_bits).coeffs
    assert got == R.mul_mod(a, bits, R.reduce_to(kb, out_bits), out_bits, out_bits, n)
    from paper_1902_04303_b200.ring import RingElement

    srng = random.Random(7)
    s = [srng.choice((-1, 0, 0, 1)) for _ in range(n)]
    S = RingElement.from_signed(n, bits, s)
    assert S.compact_bits == 2
    assert dev(n, bits, a).mul(S).coeffs == R.mul(a, R.reduce(s, bits), bits, n)


def test_keyswitch_carry_window_rescan():
    """Drive the CRT's truncated carry window into its ambiguous band: x = 1 and key
    coefficients placed so that c + 2^(L-1) lands exactly on / just below 2^L."""
    import ctypes

    from paper_1902_04303_b200 import _lib
    from paper_1902_04303_b200.ring import RingElement, empty_words

    n, level, big_l = 256, 400, 500
    x = [0] * n
    x[0] = 1
    kb = [0] * n
    half = 1 << (big_l - 1)
    kb[0] = half - 1          # c0 + 2^(L-1) = 2^L - 1  -> rounds to 0
    kb[1] = half              # c1 + 2^(L-1) = 2^L      -> rounds to 1
    kb[2] = (1 << (2 * big_l)) - half - 1   # negative side: -(2^(L-1)+1) -> -1
    kb[3] = (1 << big_l) + half - 1
    ka = rnd(n, 2 * big_l, 9)
    KB, KA = dev(n, 2 * big_l, kb), dev(n, 2 * big_l, ka)
    X = dev(n, level, x)
    ctx = _lib.get_context(8)
    h = ctypes.c_void_p()
    _lib.check(ctx.lib.hg_key_prepare(ctx.handle, KB.words.data_ptr(), KA.words.data_ptr(),
                                      2 * big_l, level, big_l, ctx.stream(), ctypes.byref(h)))
    o0, o1 = empty_words(level, n), empty_words(level, n)
    _lib.check(ctx.lib.hg_keyswitch(ctx.handle, h, X.words.data_ptr(), 1, o0.data_ptr(),
                                    o1.data_ptr(), ctx.stream()))
    got0 = RingElement(n, level, words=o0).coeffs
    got1 = RingElement(n, level, words=o1).coeffs
    ctx.lib.hg_key_destroy(h)
    w0, w1 = C.keyswitch(x, kb, ka, level, big_l, n)
    assert got0 == w0 and got1 == w1
    assert got0[0] == 0 and got0[1] == 1 and got0[2] == (1 << level) - 1


def test_raw_ntt_roundtrip():
    import ctypes

    import torch

    from paper_1902_04303_b200 import _lib

    for log_n in (3, 7, 11, 12, 14, 15, 17):
        ctx = _lib.get_context(log_n)
        primes = ctx.primes()
        rows = 6
        n = 1 << log_n
        data = torch.randint(0, 1 << 20, (rows, n), dtype=torch.int64, device="cuda")
        pr = torch.tensor(primes[:rows], dtype=torch.int64, device="cuda")[:, None]
        data = data % pr
        buf = data.to(torch.int32).contiguous()
        _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), rows, 0, ctx.stream()))
        # forward output is lazily reduced ([0, 4p)); the inverse takes inputs below 2p
        fwd = (buf.to(torch.int64) & 0xFFFFFFFF) % pr
        buf = fwd.to(torch.int32).contiguous()
        _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, buf.data_ptr(), rows, 0, ctx.stream()))
        got = (buf.to(torch.int64) & 0xFFFFFFFF) % pr
        want = (data * n) % pr   # the inverse leaves out 1/N (folded into the CRT)
        assert torch.equal(got, want), f"log_n={log_n}"


@pytest.mark.slow
def test_p17_keyswitch_and_mult_full_size():
    """One P17-size HeEngine.mult (N=2^17, level 1550) against the gmp-backed oracle."""
    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200 import ckks
    from paper_1902_04303_b200.ring import RingElement

    n, log_n, level, big_l = 1 << 17, 17, 1550, 1700
    params = hg.CkksParams(log_n=17, log_l=1700, log_p=45, log_p_small=30)
    a0, a1, b0, b1 = (rnd(n, level, s) for s in (11, 12, 13, 14))
    kb, ka = rnd(n, 2 * big_l, 15), rnd(n, 2 * big_l, 16)
    evk = hg.EvaluationKey(b=dev(n, 2 * big_l, kb), a=dev(n, 2 * big_l, ka))
    ct_a = hg.Ciphertext(c0=dev(n, level, a0), c1=dev(n, level, a1), level_bits=level,
                         scale_bits=45, slots=n // 2, params=params)
    ct_b = hg.Ciphertext(c0=dev(n, level, b0), c1=dev(n, level, b1), level_bits=level,
                         scale_bits=45, slots=n // 2, params=params)
    eng = hg.HeEngine(params, evk, None)
    out = eng.mult(ct_a, ct_b)
    w0, w1 = C.engine_mult(a0, a1, b0, b1, level, kb, ka, big_l, 45, n)
    assert out.c0.coeffs == w0
    assert out.c1.coeffs == w1
    assert isinstance(out.c0, RingElement) and ckks.KEY_CACHE.bytes > 0

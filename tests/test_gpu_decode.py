"""Decode on the GPU: the centered big-integer -> float64 conversion of
encoding.py:93-105 runs in `hg_poly_to_double`; it must equal Python's float(int) of the
floor-shifted centered coefficients bit for bit (round to nearest, ties to even), including
the >960-bit shift, negative values whose shifted quotient rounds up, exact halves and the
c == 2^(bits-1) representative.  The host restatement `encoding.coeffs_to_float` is the
reference's own algorithm (pinned through tests/test_gpu_ckks.py::test_decrypt_and_decode)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(n, bits, coeffs):
    from paper_1902_04303_b200.ring import RingElement

    return RingElement(n, bits, coeffs)


def _expect(n, bits, coeffs):
    from paper_1902_04303_b200.encoding import coeffs_to_float

    half, full = 1 << (bits - 1), 1 << bits
    centered = [c - full if c > half else c for c in coeffs]
    return coeffs_to_float(centered)


def _check(n, bits, coeffs):
    arr, mult = _dev(n, bits, coeffs).to_float64()
    want, wmult = _expect(n, bits, coeffs)
    assert mult == wmult
    bad = np.nonzero(arr.view(np.uint64) != want.view(np.uint64))[0]
    assert bad.size == 0, (bits, bad[:5], arr[bad[:5]], want[bad[:5]])


def _ties(bits, rng, count):
    """Values whose magnitude sits exactly on / next to a float64 rounding boundary."""
    out = []
    for _ in range(count):
        top = rng.randrange(54, min(bits - 1, 900))
        mant = rng.getrandbits(53) | (1 << 52)
        m = mant << (top - 52)
        half = 1 << (top - 53)
        v = m + rng.choice([half, half - 1, half + 1, 0, 1, (1 << (top - 52)) - 1])
        out.append(v if rng.random() < 0.5 else -v)
    return out


@pytest.mark.parametrize("n,bits", [(16, 1), (32, 31), (32, 32), (64, 33), (256, 63), (256, 64),
                                    (256, 65), (512, 230), (1024, 1700), (4096, 1440)])
def test_to_float64_random(n, bits):
    rng = random.Random(bits * 7 + n)
    coeffs = [rng.getrandbits(bits) for _ in range(n)]
    # small centered values of both signs, the exact half, zero and all-ones
    special = [0, (1 << bits) - 1, 1 << (bits - 1), 1, ((1 << bits) - 1) & ~1]
    for k, v in enumerate(special):
        coeffs[k % n] = v
    _check(n, bits, coeffs)


@pytest.mark.parametrize("bits", [700, 1700])
def test_to_float64_small_values_and_ties(bits):
    n = 2048
    rng = random.Random(bits)
    vals = _ties(bits, rng, n // 2) + [rng.randrange(-(1 << 60), 1 << 60) for _ in range(n // 2)]
    _check(n, bits, [v % (1 << bits) for v in vals])


@pytest.mark.parametrize("top_bits", [961, 1000, 1500, 1699])
def test_to_float64_shifted(top_bits):
    """bitlen > 960: every coefficient is floor-shifted by bitlen - 500 first (negative
    quotients round toward -inf, i.e. the magnitude rounds up), multiplier 2^min(s, 300)."""
    bits, n = 1700, 1024
    rng = random.Random(top_bits)
    vals = [rng.getrandbits(rng.randrange(1, top_bits)) * rng.choice([1, -1]) for _ in range(n)]
    vals[3] = (1 << (top_bits - 1)) + rng.getrandbits(top_bits - 1)
    vals[4] = -((1 << (top_bits - 1)))
    s = top_bits - 500
    # quotient boundary cases: exact multiples of 2^s (no round-up) and one past them
    vals[5] = -(rng.getrandbits(400) << s)
    vals[6] = -((rng.getrandbits(400) << s) + 1)
    vals[7] = -(((1 << 400) - 1) << s) - 1  # quotient all ones: the round-up carries through it
    _check(n, bits, [v % (1 << bits) for v in vals])


def test_decode_device_matches_host_restatement():
    """decode() through the GPU conversion equals the reference's algorithm on the host."""
    from paper_1902_04303_b200 import encoding as E
    from paper_1902_04303_b200.encoding import Plaintext

    n, bits = 4096, 1440
    rng = random.Random(5)
    coeffs = [rng.randrange(-(1 << 70), 1 << 70) % (1 << bits) for _ in range(n)]
    pt = Plaintext(m=_dev(n, bits, coeffs), scale_bits=45, slots=n // 2)
    got = E.decode(pt)
    want = E.decode_coefficients(pt.m.centered(), 45, n)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))

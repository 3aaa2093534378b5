"""The opt-in prime-range NTT launches (HG_NTT_L2_MB: both passes of a transform run prime range
by prime range so the intermediate stays in L2; csrc/hg_ntt.cu prime_chunk) give the oracle's
products.  The budget is read once per process, so the check runs in a child process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import random, sys
sys.path.insert(0, %r)
from oracle import ring_oracle as R
from paper_1902_04303_b200.ring import RingElement
for n, bits in ((1 << 15, 240), (1 << 16, 480)):
    rng = random.Random(n)
    a = [rng.getrandbits(bits) for _ in range(n)]
    b = [rng.getrandbits(bits) for _ in range(n)]
    assert RingElement(n, bits, a).mul(RingElement(n, bits, b)).coeffs == R.mul(a, b, bits, n), n
print("chunked ok")
"""


@pytest.mark.parametrize("mb", ["1", "3"])
def test_products_with_prime_range_ntt_launches(mb):
    env = dict(os.environ, HG_NTT_L2_MB=mb)
    r = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "chunked ok" in r.stdout

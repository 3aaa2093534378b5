"""A minimal ``gmpy2`` stand-in for running the REFERENCE package fast (golden generation and
CPU timing only; never imported by the product).

The reference's ring.py uses exactly one gmpy2 feature: ``int(mpz(a) * mpz(b))`` for the
Kronecker big multiply (hegwas/ring.py:15-23, 55).  gmpy2 is not installed in this image and
there is no network, but libgmp.so.10 is; this module forwards that one product to libgmp's
mpz_mul through oracle/ring_oracle.big_multiply (ctypes).  Big-integer multiplication is exact
either way, so the reference's results are unchanged -- only its speed is.
Put this directory first on sys.path before importing hegwas.
"""
from __future__ import annotations

import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

from oracle.ring_oracle import big_multiply  # noqa: E402

SHIM = True   # lets callers record that the shim (not real gmpy2) was in use


class mpz:  # noqa: N801 - gmpy2's spelling
    __slots__ = ("v",)

    def __init__(self, v=0):
        self.v = int(v)

    def __mul__(self, other):
        a = self.v
        b = other.v if isinstance(other, mpz) else int(other)
        if a < 0 or b < 0 or a.bit_length() < 4096 or b.bit_length() < 4096:
            return mpz(a * b)
        xa = a.to_bytes((a.bit_length() + 7) // 8, "little")
        xb = b.to_bytes((b.bit_length() + 7) // 8, "little")
        return mpz(int.from_bytes(big_multiply(xa, xb), "little"))

    __rmul__ = __mul__

    def __int__(self):
        return self.v

    __index__ = __int__

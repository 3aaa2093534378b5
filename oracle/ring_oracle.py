"""CPU restatement of the reference ring arithmetic -- TEST INFRASTRUCTURE ONLY.

Follows hegwas/ring.py (file:line cited per function).  Polynomials are plain lists of
Python ints.  The exact negacyclic product uses Kronecker substitution (ring.py:46-58):
coefficients are packed into one integer with a slot wide enough for the sum of n cross
products, multiplied once, and unpacked with the x^n = -1 wrap.  The single big multiply
goes through libgmp (ctypes) when libgmp.so.10 is present, else CPython ints; both are
exact, so results are identical -- gmp only makes N >= 2^12 parity cases finish in
seconds.
"""
from __future__ import annotations

import ctypes
import ctypes.util

_GMP = None


class _Mpz(ctypes.Structure):
    _fields_ = [("alloc", ctypes.c_int), ("size", ctypes.c_int), ("d", ctypes.c_void_p)]


def _gmp():
    global _GMP
    if _GMP is None:
        lib = None
        for name in ("libgmp.so.10", ctypes.util.find_library("gmp")):
            if not name:
                continue
            try:
                lib = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if lib is not None:
            lib.__gmpz_init.argtypes = [ctypes.POINTER(_Mpz)]
            lib.__gmpz_clear.argtypes = [ctypes.POINTER(_Mpz)]
            lib.__gmpz_import.argtypes = [ctypes.POINTER(_Mpz), ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t,
                                          ctypes.c_void_p]
            lib.__gmpz_export.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t),
                                          ctypes.c_int, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_size_t, ctypes.POINTER(_Mpz)]
            lib.__gmpz_export.restype = ctypes.c_void_p
            lib.__gmpz_mul.argtypes = [ctypes.POINTER(_Mpz)] * 3
        _GMP = lib or False
    return _GMP or None


def big_multiply(x: bytes, y: bytes) -> bytes:
    """Product of two little-endian byte strings (nonnegative), little-endian bytes."""
    lib = _gmp()
    if lib is None:
        prod = int.from_bytes(x, "little") * int.from_bytes(y, "little")
        return prod.to_bytes(len(x) + len(y), "little")
    a, b, c = _Mpz(), _Mpz(), _Mpz()
    for z in (a, b, c):
        lib.__gmpz_init(ctypes.byref(z))
    try:
        bx = ctypes.create_string_buffer(x, len(x))
        by = ctypes.create_string_buffer(y, len(y))
        lib.__gmpz_import(ctypes.byref(a), len(x), -1, 1, 0, 0, bx)
        lib.__gmpz_import(ctypes.byref(b), len(y), -1, 1, 0, 0, by)
        lib.__gmpz_mul(ctypes.byref(c), ctypes.byref(a), ctypes.byref(b))
        out = ctypes.create_string_buffer(len(x) + len(y) + 16)
        cnt = ctypes.c_size_t(0)
        lib.__gmpz_export(out, ctypes.byref(cnt), -1, 1, 0, 0, ctypes.byref(c))
        return out.raw[: len(x) + len(y)]
    finally:
        for z in (a, b, c):
            lib.__gmpz_clear(ctypes.byref(z))


def schoolbook_negacyclic(a: list[int], b: list[int], n: int) -> list[int]:
    """O(n^2) exact negacyclic convolution (ring.py:29-43)."""
    out = [0] * n
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                if i + j < n:
                    out[i + j] += x * y
                else:
                    out[i + j - n] -= x * y
    return out


def negacyclic_mul(a: list[int], b: list[int], n: int, a_bits: int, b_bits: int) -> list[int]:
    """Exact negacyclic convolution of nonnegative vectors (ring.py:46-65), unreduced."""
    if n <= 8:
        return schoolbook_negacyclic(a, b, n)
    width = a_bits + b_bits + max(1, n - 1).bit_length() + 2
    wb = (width + 7) // 8
    xa = b"".join(c.to_bytes(wb, "little") for c in a)
    xb = b"".join(c.to_bytes(wb, "little") for c in b)
    prod = big_multiply(xa, xb)
    prod = prod + bytes(max(0, 2 * n * wb - len(prod)))
    c = [int.from_bytes(prod[k * wb:(k + 1) * wb], "little") for k in range(2 * n)]
    return [c[k] - c[k + n] for k in range(n)]


def reduce(coeffs: list[int], bits: int) -> list[int]:
    mask = (1 << bits) - 1
    return [c & mask for c in coeffs]


def add(a, b, bits):            # ring.py:114
    return reduce([x + y for x, y in zip(a, b)], bits)


def sub(a, b, bits):            # ring.py:123
    return reduce([x - y for x, y in zip(a, b)], bits)


def neg(a, bits):               # ring.py:132
    return reduce([-x for x in a], bits)


def scalar_mul(a, k, bits):     # ring.py:136
    return reduce([x * k for x in a], bits)


def mul(a, b, bits, n):         # ring.py:140 (same modulus)
    return reduce(negacyclic_mul(a, b, n, bits, bits), bits)


def mul_mod(a, a_bits, b, b_bits, out_bits, n):   # ring.py:145
    return reduce(negacyclic_mul(a, b, n, a_bits, b_bits), out_bits)


def automorphism(a, k, bits):   # ring.py:152
    n = len(a)
    n2 = 2 * n
    k %= n2
    mask = (1 << bits) - 1
    out = [0] * n
    for j, c in enumerate(a):
        e = (j * k) % n2
        if e < n:
            out[e] = c
        else:
            out[e - n] = (-c) & mask
    return out


def reduce_to(a, bits):          # ring.py:168
    return reduce(a, bits)


def centered(a, bits):           # ring.py:106
    half = 1 << (bits - 1)
    full = 1 << bits
    return [c - full if c > half else c for c in a]


def lift_centered_to(a, in_bits, out_bits):   # ring.py:177
    return reduce(centered(a, in_bits), out_bits)


def divide_round(a, shift, out_bits):          # ring.py:184
    half = 1 << (shift - 1) if shift > 0 else 0
    mask = (1 << out_bits) - 1
    return [((c + half) >> shift) & mask for c in a]

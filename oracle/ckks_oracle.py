"""CPU restatement of the scheme operations -- TEST INFRASTRUCTURE ONLY.

Ciphertexts are (c0, c1) pairs of coefficient lists at an explicit level; every function
cites the reference routine (hegwas/ckks.py) it follows.
"""
from __future__ import annotations

from . import ring_oracle as R


def keyswitch(x, kb, ka, level, big_l, n):
    """ckks._keyswitch (ckks.py:187-194)."""
    kb_r = R.reduce_to(kb, level + big_l)
    ka_r = R.reduce_to(ka, level + big_l)
    t0 = R.mul_mod(x, level, kb_r, level + big_l, level + big_l, n)
    t1 = R.mul_mod(x, level, ka_r, level + big_l, level + big_l, n)
    return R.divide_round(t0, big_l, level), R.divide_round(t1, big_l, level)


def mult(a0, a1, b0, b1, level, evk_b, evk_a, big_l, n):
    """ckks.mult without rescale (ckks.py:166-184)."""
    d0 = R.mul(a0, b0, level, n)
    d1 = R.add(R.mul(a0, b1, level, n), R.mul(a1, b0, level, n), level)
    d2 = R.mul(a1, b1, level, n)
    e0, e1 = keyswitch(d2, evk_b, evk_a, level, big_l, n)
    return R.add(d0, e0, level), R.add(d1, e1, level)


def rescale(c0, c1, bits, level):
    """ckks.rescale ring part (ckks.py:215-219)."""
    return R.divide_round(c0, bits, level - bits), R.divide_round(c1, bits, level - bits)


def engine_mult(a0, a1, b0, b1, level, evk_b, evk_a, big_l, log_p, n):
    """HeEngine.mult on aligned inputs (ckks.py:310-313)."""
    c0, c1 = mult(a0, a1, b0, b1, level, evk_b, evk_a, big_l, n)
    return rescale(c0, c1, log_p, level)


def apply_automorphism(c0, c1, k, kb, ka, level, big_l, n):
    """ckks._apply_automorphism (ckks.py:247-253)."""
    a0 = R.automorphism(c0, k, level)
    a1 = R.automorphism(c1, k, level)
    e0, e1 = keyswitch(a1, kb, ka, level, big_l, n)
    return R.add(a0, e0, level), e1


def rotation_exponent(log_n: int, amount: int) -> int:
    """keys.rotation_exponent (keys.py:57-60)."""
    n = 1 << log_n
    slots = n // 2
    return pow(5, (slots - amount) % slots, 2 * n)


def mult_plain(c0, c1, m, m_bits, level, n):
    """ckks.mult_plain ring part (ckks.py:154-161)."""
    mm = R.reduce_to(m, level) if m_bits >= level else R.lift_centered_to(m, m_bits, level)
    return R.mul(c0, mm, level, n), R.mul(c1, mm, level, n)


def engine_inner(a_list, b_list, level, evk_b, evk_a, big_l, log_p, n):
    """sum_b a_b (x) b_b relinearised and rescaled ONCE (HeEngine.inner_product; no reference
    counterpart -- composed from the reference's own mul / _keyswitch / divide_round,
    ckks.py:166-194, 215-219): the three tensor parts are summed mod 2^level first."""
    d0 = d1 = d2 = [0] * n
    for (a0, a1), (b0, b1) in zip(a_list, b_list):
        d0 = R.add(d0, R.mul(a0, b0, level, n), level)
        d1 = R.add(d1, R.add(R.mul(a0, b1, level, n), R.mul(a1, b0, level, n), level), level)
        d2 = R.add(d2, R.mul(a1, b1, level, n), level)
    e0, e1 = keyswitch(d2, evk_b, evk_a, level, big_l, n)
    return rescale(R.add(d0, e0, level), R.add(d1, e1, level), log_p, level)

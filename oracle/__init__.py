"""CPU oracle for parity tests -- TEST INFRASTRUCTURE ONLY.

Restates the reference's ring / scheme arithmetic (hegwas/ring.py, hegwas/ckks.py) with
Python integers (optionally multiplied through libgmp via ctypes for speed; results are
identical).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or the timed CPU
baseline -- never as the product path.

Parity pinning: the oracle is checked bit-for-bit against golden vectors produced by
running the reference package itself (tests/golden/*.npz, made by tools/make_golden.py).
"""

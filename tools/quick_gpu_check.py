"""Quick GPU-vs-oracle check of the ring kernels (development aid; pytest -m gpu is the
real suite).  Usage: python tools/quick_gpu_check.py"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import ring_oracle as R  # noqa: E402
from paper_1902_04303_b200.ring import RingElement  # noqa: E402


def rnd(n, bits, seed):
    rng = random.Random(seed)
    return [rng.getrandbits(bits) for _ in range(n)]


def check(name, got, want):
    ok = got == want
    print(f"{'OK  ' if ok else 'FAIL'} {name}")
    if not ok:
        bad = [i for i in range(len(want)) if got[i] != want[i]]
        print("   first mismatches:", bad[:5], len(bad))
        i = bad[0]
        print("   got ", hex(got[i])[:80])
        print("   want", hex(want[i])[:80])
    return ok


def main():
    allok = True
    for log_n, bits in [(4, 40), (7, 300), (8, 350), (10, 1700), (12, 1440), (13, 240)]:
        n = 1 << log_n
        a = rnd(n, bits, 1)
        b = rnd(n, bits, 2)
        A = RingElement(n, bits, a)
        B = RingElement(n, bits, b)
        allok &= check(f"add n={n} bits={bits}", A.add(B).coeffs, R.add(a, b, bits))
        allok &= check(f"sub n={n} bits={bits}", A.sub(B).coeffs, R.sub(a, b, bits))
        allok &= check(f"neg n={n} bits={bits}", A.neg().coeffs, R.neg(a, bits))
        for k in (3, -1, 4, 1 << 45, -(1 << 70) + 12345):
            allok &= check(f"scalar_mul k={k} n={n}", A.scalar_mul(k).coeffs, R.scalar_mul(a, k, bits))
        for k in (5, 2 * n - 1, 25, 3):
            allok &= check(f"automorphism k={k} n={n}", A.automorphism(k).coeffs, R.automorphism(a, k, bits))
        allok &= check(f"reduce_to n={n}", A.reduce_to(bits - 37).coeffs, R.reduce_to(a, bits - 37))
        allok &= check(f"lift n={n}", A.lift_centered_to(bits + 77).coeffs, R.lift_centered_to(a, bits, bits + 77))
        for sh in [s for s in (0, 1, 45, 64, 30) if s < bits]:
            allok &= check(f"divide_round sh={sh} n={n}", A.divide_round(sh, bits - sh).coeffs,
                           R.divide_round(a, sh, bits - sh))
        t = time.time()
        want = R.mul(a, b, bits, n)
        t_cpu = time.time() - t
        t = time.time()
        got = A.mul(B).coeffs
        t_gpu = time.time() - t
        allok &= check(f"mul n={n} bits={bits} (cpu {t_cpu:.2f}s gpu {t_gpu:.3f}s)", got, want)
        # mul_mod with wider output (keyswitch-like)
        kb = rnd(n, 2 * bits, 3)
        K = RingElement(n, 2 * bits, kb)
        out_bits = bits + bits // 2
        Kr = K.reduce_to(out_bits)
        want = R.mul_mod(a, bits, R.reduce_to(kb, out_bits), out_bits, out_bits, n)
        allok &= check(f"mul_mod n={n}", A.mul_mod(Kr, out_bits).coeffs, want)
        # small signed operand
        s = [rng_v for rng_v in (random.Random(5).choice((-1, 0, 0, 1)) for _ in range(n))]
        S = RingElement.from_signed(n, bits, s)
        want = R.mul(a, R.reduce(s, bits), bits, n)
        allok &= check(f"mul small n={n}", A.mul(S).coeffs, want)
    torch.cuda.synchronize()
    print("ALL OK" if allok else "SOME FAILED")
    return 0 if allok else 1


if __name__ == "__main__":
    sys.exit(main())

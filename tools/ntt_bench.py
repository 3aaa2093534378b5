"""Device-timed raw NTTs at N=2^17: forward / inverse over [B][P][N] rows, two-pass vs cluster
kernels (hg_set_ntt_variant), same buffers.  --ncu: one launch of each inside a profiler window.

    python tools/ntt_bench.py [--rows-per-prime 4] [--primes 164] [--ncu]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1902_04303_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows-per-prime", type=int, default=4)
    ap.add_argument("--primes", type=int, default=164)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--variants", type=int, nargs="+", default=[0, 2, 0, 2])
    a = ap.parse_args()
    ctx = _lib.get_context(17)
    primes = ctx.primes()
    P = a.primes
    off = len(primes) - P
    rows = P * a.rows_per_prime
    n = 1 << 17
    pr = torch.tensor([primes[off + i % P] for i in range(rows)], dtype=torch.int64, device="cuda")[:, None]
    buf = (torch.randint(0, 1 << 62, (rows, n), dtype=torch.int64, device="cuda") % pr).to(torch.int32)
    st = ctx.stream()
    if a.ncu:
        for v in sorted(set(a.variants)):
            _lib.check(ctx.lib.hg_set_ntt_variant(ctx.handle, v))
            _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), rows, off, st))
            _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, buf.data_ptr(), rows, off, st))
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        for v in sorted(set(a.variants)):
            _lib.check(ctx.lib.hg_set_ntt_variant(ctx.handle, v))
            _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), rows, off, st))
            _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, buf.data_ptr(), rows, off, st))
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return
    s = torch.cuda.current_stream()
    for v in a.variants:
        _lib.check(ctx.lib.hg_set_ntt_variant(ctx.handle, v))
        res = {}
        for name, fn in (("fwd", ctx.lib.hg_ntt_forward), ("inv", ctx.lib.hg_ntt_inverse)):
            for _ in range(3):
                _lib.check(fn(ctx.handle, buf.data_ptr(), rows, off, st))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(a.reps):
                _lib.check(fn(ctx.handle, buf.data_ptr(), rows, off, st))
            e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.reps
            res[name] = (us, us / rows, 2 * rows * n * 4 / us / 1e3)
        print(f"cluster={v} rows={rows}: " + "  ".join(
            f"{k} {t:8.1f} us ({per:.3f} us/row, {gbs:6.0f} GB/s algorithmic)" for k, (t, per, gbs) in res.items()),
            flush=True)


if __name__ == "__main__":
    main()

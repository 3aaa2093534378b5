"""Per-op device timings (CUDA events) for the scheme ops at P17 and config-1 points.

    python tools/op_bench.py [--log-n 17] [--log-l 1700] [--reps 5] [--only mult,rot,...]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-n", type=int, default=17)
    ap.add_argument("--log-l", type=int, default=1700)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(args.only.split(",")) if args.only else None
    params = hg.CkksParams(log_n=args.log_n, log_l=args.log_l, log_p=45, log_p_small=30)
    t = time.time()
    sk, pk, evk, rot = hg.keygen(params, 1, device_rng=True)
    torch.cuda.synchronize()
    print(json.dumps({"op": "keygen_device_rng", "s": round(time.time() - t, 3)}), flush=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    vals = np.random.default_rng(0).uniform(-1, 1, params.slot_count)
    t = time.time()
    a = hg.encrypt_values(vals, 45, pk, params, gen)
    b = hg.encrypt_values(vals[::-1], 45, pk, params, gen)
    torch.cuda.synchronize()
    print(json.dumps({"op": "encrypt_x2", "s": round(time.time() - t, 3)}), flush=True)
    ctx = _lib.get_context(args.log_n)
    levels = [args.log_l, args.log_l - 150, 230]
    for lv in levels:
        if lv > args.log_l or lv < 100:
            continue
        al, bl = hg.mod_down(a, lv), hg.mod_down(b, lv)
        rec = {"level": lv, "N": params.n}
        if only is None or "mult" in only:
            eng.mult(al, bl)  # prepare evk at this level
            rec["mult_ms"] = round(timed(lambda: eng.mult(al, bl), args.reps), 3)
        if only is None or "rot" in only:
            eng.rotate(al, 1)
            rec["rotate1_ms"] = round(timed(lambda: eng.rotate(al, 1), args.reps), 3)
        if only is None or "rotb" in only:
            cts = [al, bl, hg.negate(al), hg.negate(bl)]
            eng.rotate_many(cts, 1)
            rec["rotate1_x4_ms"] = round(timed(lambda: [eng.rotate(c, 1) for c in cts], args.reps), 3)
            rec["rotate1_batch4_ms"] = round(timed(lambda: eng.rotate_many(cts, 1), args.reps), 3)
        if only is None or "pmul" in only:
            m = eng.mask(("slot", 3))
            rec["mult_plain_ms"] = round(timed(lambda: eng.mult_plain(al, m), args.reps), 3)
        if only is None or "rescale" in only:
            rec["rescale30_ms"] = round(timed(lambda: hg.rescale(al, 30), args.reps), 3)
        if only is None or "add" in only:
            rec["add_ms"] = round(timed(lambda: hg.add(al, bl), args.reps), 3)
        print(json.dumps(rec), flush=True)
    # raw NTT throughput: P rows of length N
    P = 64
    buf = torch.randint(0, 1 << 20, (P, params.n), dtype=torch.int32, device="cuda")
    ms = timed(lambda: _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), P, 0, ctx.stream())), 10)
    print(json.dumps({"op": "ntt_forward", "rows": P, "N": params.n, "ms": round(ms, 4),
                      "ntt_per_s": round(P / ms * 1e3), "GBps": round(P * params.n * 8 / ms / 1e6, 1)}), flush=True)
    ms = timed(lambda: _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, buf.data_ptr(), P, 0, ctx.stream())), 10)
    print(json.dumps({"op": "ntt_inverse", "rows": P, "N": params.n, "ms": round(ms, 4),
                      "ntt_per_s": round(P / ms * 1e3)}), flush=True)
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    ops = ctypes.c_double()
    iters = 4096
    fn = lambda: _lib.check(ctx.lib.hg_bench_modmul(ctx.handle, iters, sink.data_ptr(), ctypes.byref(ops), ctx.stream()))  # noqa: E731
    ms = timed(fn, 5)
    print(json.dumps({"op": "modmul_probe", "butterflies_per_s": ops.value / ms * 1e3}), flush=True)


if __name__ == "__main__":
    main()

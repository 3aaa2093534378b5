"""BASELINE config 1: CKKS primitive sweep on random ciphertexts.

N in {2^13..2^16} x log_l in {240, 480, 960, 1440} x batch in {1, 4, 16, 64, 256}; dnum = 1
(the only key-switch form with reference semantics).  Ops, each timed on the device over a
batch of independent ciphertexts with inputs resident:
  ntt / intt      one length-N negacyclic transform over one 30-bit prime (batch x P rows, P =
                  the prime count of a top-level tensor product)
  mult            HeEngine.mult (tensor + relinearise + rescale by log_p) at the top level
  rotate          rotate by +2^k (one key switch), k = 1
  rotate_left     rotate_left by 2^k (popcount(slots - 2^k) key switches), k = 1
  rescale         rescale(log_p)
  mult_plain      HeEngine.mult_plain with a random mask plaintext at scale 30
Random ciphertexts: c0, c1 uniform mod 2^l (ckks.sample_uniform semantics, device RNG).

    python tools/config1_sweep.py [--batches 1,4,16,64,256] [--out profiles/r1_config1_sweep.json]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1902_04303_b200 as hg  # noqa: E402
from paper_1902_04303_b200 import _lib, ckks  # noqa: E402
from paper_1902_04303_b200.ring import RingElement, words_for  # noqa: E402


def device_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def random_ct(params, gen, scale_bits):
    """c0, c1 uniform mod 2^log_l (a valid Ciphertext object; decryption is noise)."""
    n, lvl = params.n, params.log_l
    w = words_for(lvl)

    def poly():
        x = torch.randint(-(1 << 31), 1 << 31, (w, n), dtype=torch.int64, device="cuda", generator=gen)
        x = x.to(torch.int32)
        if lvl & 31:
            x[w - 1] &= (1 << (lvl & 31)) - 1
        return RingElement(n, lvl, words=x)

    return ckks.Ciphertext(c0=poly(), c1=poly(), level_bits=lvl, scale_bits=scale_bits,
                           slots=params.slot_count, params=params)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log-ns", default="13,14,15,16")
    ap.add_argument("--log-ls", default="240,480,960,1440")
    ap.add_argument("--batches", default="1,4,16,64,256")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    batches = [int(b) for b in args.batches.split(",")]
    rows = []
    for log_n in [int(x) for x in args.log_ns.split(",")]:
        for log_l in [int(x) for x in args.log_ls.split(",")]:
            params = hg.CkksParams(log_n=log_n, log_l=log_l, log_p=45, log_p_small=30)
            t0 = time.time()
            sk, pk, evk, rot = hg.keygen(params, 7, device_rng=True)
            eng = hg.HeEngine(params, evk, rot)
            gen = torch.Generator(device="cuda")
            gen.manual_seed(log_n * 10000 + log_l)
            mask = hg.encode(np.random.default_rng(1).uniform(-1, 1, params.slot_count), 30, params)
            ctx = _lib.get_context(log_n)
            # primes of a top-level tensor product (centered operands, d1 is a sum of two)
            P = ctx.primes_for_bits(2 * (log_l - 1) + 1 + log_n + 3) if hasattr(ctx, "primes_for_bits") else \
                math.ceil((2 * log_l + log_n + 4) / 29.9)
            for b in batches:
                cts = [random_ct(params, gen, 45) for _ in range(b)]
                reps = max(1, args.reps)
                rec = {"log_n": log_n, "N": params.n, "log_l": log_l, "batch": b}
                # warm the key cache at this level
                eng.mult(cts[0], cts[0])
                eng.rotate(cts[0], 2)
                eng.rotate_left(cts[0], 2)
                # batches of independent ciphertexts go through the batched engine calls
                # (mult_many: two products per group of launches; rotate_many: four per group);
                # batch 1 is the single-op latency
                rec["mult_per_s"] = b / device_time(
                    (lambda: eng.mult_many(cts, cts)) if b > 1 else (lambda: eng.mult(cts[0], cts[0])), reps)
                rec["rotate_per_s"] = b / device_time(lambda: eng.rotate_many(cts, 2), reps)
                rec["rotate_left_per_s"] = b / device_time(
                    lambda: eng.rotate_many(cts, params.slot_count - 2), reps)
                rec["rotate_left_keyswitches"] = bin(params.slot_count - 2).count("1")
                hi = [ckks.Ciphertext(c0=c.c0, c1=c.c1, level_bits=c.level_bits, scale_bits=90,
                                      slots=c.slots, params=params) for c in cts]   # post-mult scale
                # rescale / mult_plain batches through the array-of-handles entry points
                # (hg_ct_rescale_batch, hg_ct_mult_plain_batch: one launch group per 8 / per batch)
                rec["rescale_per_s"] = b / device_time(
                    (lambda: eng.rescale_many(hi, 45)) if b > 1 else (lambda: hg.rescale(hi[0], 45)), reps)
                rec["mult_plain_per_s"] = b / device_time(
                    (lambda: eng.mult_plain_many(cts, mask)) if b > 1 else (lambda: eng.mult_plain(cts[0], mask)), reps)
                # hg_ntt_forward cycles rows over min(count, 320) primes: keep the batched fast
                # path by using whole multiples of the 320-prime table past it
                nrows = b * P if b * P <= 320 else 320 * (min(b * P, 4096) // 320)
                buf = torch.randint(0, 1 << 20, (nrows, params.n), dtype=torch.int32, device="cuda")
                rec["ntt_rows"] = nrows
                rec["ntt_per_s"] = nrows / device_time(lambda: _lib.check(ctx.lib.hg_ntt_forward(
                    ctx.handle, buf.data_ptr(), nrows, 0, ctx.stream())), reps)
                rec["intt_per_s"] = nrows / device_time(lambda: _lib.check(ctx.lib.hg_ntt_inverse(
                    ctx.handle, buf.data_ptr(), nrows, 0, ctx.stream())), reps)
                for k, v in list(rec.items()):
                    if k.endswith("_per_s"):
                        rec[k] = round(v, 1)
                print(json.dumps(rec), flush=True)
                rows.append(rec)
                del cts, buf
            torch.cuda.empty_cache()
            print(json.dumps({"log_n": log_n, "log_l": log_l, "wall_s": round(time.time() - t0, 1)}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"config": "BASELINE config 1 (primitive sweep), dnum=1, device-timed, resident inputs; "
                                 "batches > 1 through HeEngine.mult_many / rotate_many / rescale_many / "
                                 "mult_plain_many",
                       "device": torch.cuda.get_device_name(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()

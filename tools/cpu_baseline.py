"""CPU baseline of the REFERENCE evaluator itself (hegwas, imported read-only from
/root/reference): medians of >= 3 runs per op, single thread.

  * per op: HeEngine.mult (+ rescale), rotate(2^k) (one key switch), rotate_left(2^k)
    (popcount(slots - 2^k) key switches), rescale, mult_plain (+ rescale) with a slot mask,
    and one key-switch-sized negacyclic_mul, at every config-1 point (log_n 13..16 x
    log_l 240 / 480 / 960 / 1440, top level) and at P17 levels {1700, 1550, 230};
  * two arithmetic back ends, labelled: "gmp" (tools/gmpy2_shim: libgmp's mpz_mul for the one
    big multiply, hegwas/ring.py:55) everywhere, and "cpython" (the reference as installed
    here: CPython ints) where a point finishes in minutes;
  * the toy encrypted GWAS (compute_gwas_encrypted, cache=None) at n=8 / log_n=7 and
    n=16 / log_n=9 (log_l 1700, log_p_small 30), both back ends.

This measures the reference on THIS container's CPU (not the GPU box); bench.py's
--impl reference arm is the box-side baseline.  Output: profiles/r2_cpu_baseline.json.

    python tools/cpu_baseline.py [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from multiprocessing import Pool

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "profiles", "r2_cpu_baseline.json")


def _setup(backend: str):
    if backend == "gmp":
        sys.path.insert(0, os.path.join(REPO, "tools", "gmpy2_shim"))
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(0, REPO)


def op_point(args):
    """Median seconds of each op at one (log_n, log_l, level) point."""
    backend, log_n, log_l, level, reps, ops = args
    _setup(backend)
    import random

    import hegwas
    from hegwas import ring as rring

    assert rring.HAVE_GMPY2 == (backend == "gmp")
    params = hegwas.CkksParams(log_n=log_n, log_l=log_l, log_p=45, log_p_small=30, h=64)
    t0 = time.perf_counter()
    sk, pk, evk, rot = hegwas.keygen(params, 1)
    t_key = time.perf_counter() - t0
    eng = hegwas.HeEngine(params, evk, rot)
    rng = random.Random(2)
    slots = params.slot_count
    a = hegwas.encrypt_values([complex(rng.uniform(-1, 1), 0) for _ in range(slots)], params.log_p, pk, params, rng)
    b = hegwas.encrypt_values([complex(rng.uniform(-1, 1), 0) for _ in range(slots)], params.log_p, pk, params, rng)
    if level < log_l:
        a, b = hegwas.mod_down(a, level), hegwas.mod_down(b, level)
    mask = eng.mask(("slot", 3))
    fns = {
        "mult": lambda: eng.mult(a, b),
        "rotate_2k": lambda: eng.rotate(a, 16),
        "rotate_left_2k": lambda: eng.rotate_left(a, slots // 2),
        "rescale": lambda: hegwas.rescale(a, 30),
        "mult_plain": lambda: eng.mult_plain(a, mask),
        "negacyclic_mul_ks": lambda: rring.negacyclic_mul(a.c1.coeffs, evk.b.coeffs, params.n, level, 2 * log_l),
    }
    res = {}
    for name in ops:
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            fns[name]()
            ts.append(time.perf_counter() - t)
        res[name] = round(statistics.median(ts), 4)
    return {"backend": backend, "log_n": log_n, "log_l": log_l, "level": level, "keygen_s": round(t_key, 2),
            "median_s": res, "reps": reps}


def toy_pipeline(args):
    backend, n, log_n, k = args
    _setup(backend)
    import random

    import hegwas
    from hegwas.gwas import GwasConfig, compute_gwas_encrypted, encrypt_gwas_inputs
    from hegwas.oracle import CleartextDataset

    from paper_1902_04303_b200.data import synth_gwas_dataset

    params = hegwas.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30, h=64)
    ds = synth_gwas_dataset(n, 4, k, seed=0)
    sk, pk, evk, rot = hegwas.keygen(params, 5)
    config = GwasConfig(n=n, d=4, k=k).resolve(params)
    enc = encrypt_gwas_inputs(CleartextDataset(X=ds.X, S=ds.S, y=ds.y), config, params, pk, random.Random(0))
    eng = hegwas.HeEngine(params, evk, rot)
    t = time.perf_counter()
    with hegwas.track_ops() as ops:
        compute_gwas_encrypted(eng, enc, cache=None)
    dt = time.perf_counter() - t
    return {"backend": backend, "n": n, "log_n": log_n, "k": k, "compute_s": round(dt, 2),
            "snp_per_s": round(k / dt, 5), "op_counts": ops.snapshot()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    ops_all = ["mult", "rotate_2k", "rotate_left_2k", "rescale", "mult_plain", "negacyclic_mul_ks"]
    jobs = []
    for ln in (13, 14, 15, 16):
        for ll in (240, 480, 960, 1440):
            jobs.append(("gmp", ln, ll, ll, 3, ops_all))
    # the reference as installed (CPython ints): the points it finishes in minutes
    jobs += [("cpython", 13, 240, 240, 3, ops_all), ("cpython", 13, 480, 480, 3, ops_all)]
    p17 = [l for l in (1700, 1550, 230)]
    jobs += [("gmp", 17, 1700, lv, 3, ["mult", "rotate_2k", "rescale", "mult_plain", "negacyclic_mul_ks"])
             for lv in p17]
    toys = [("gmp", 8, 7, 16), ("gmp", 16, 9, 32), ("cpython", 8, 7, 16)]
    if args.quick:
        jobs = [j for j in jobs if j[1] <= 14]
        toys = toys[:1]
    jobs.sort(key=lambda j: -(j[1] * 10000 + j[2]))
    cpu = subprocess.run(["sh", "-c", "grep -m1 'model name' /proc/cpuinfo"], capture_output=True,
                         text=True).stdout.strip()
    out = {"host": {"cpu": cpu, "cores": os.cpu_count(), "threads_per_op": 1},
           "note": "the reference package itself (hegwas) timed on this container's CPU; 'gmp' = with "
                   "tools/gmpy2_shim (libgmp mpz_mul for ring.py:55), 'cpython' = as installed (no gmpy2)",
           "ops": [], "toy_pipeline": []}
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        for r in pool.imap_unordered(op_point, jobs):
            out["ops"].append(r)
            print(json.dumps(r), flush=True)
            json.dump(out, open(OUT, "w"), indent=1)
        for r in pool.imap_unordered(toy_pipeline, toys):
            out["toy_pipeline"].append(r)
            print(json.dumps(r), flush=True)
            json.dump(out, open(OUT, "w"), indent=1)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()

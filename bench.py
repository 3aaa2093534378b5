"""Benchmark of the encrypted semi-parallel GWAS hot path on B200.

Workload (config.workload): the paper-scale job (BASELINE.json config 3: n=245 samples,
d=4 covariates, 10643 SNPs, complex-packed 512 SNPs per batch) at the parity preset P17
(N=2^17, log_l=1700, log_p=45, log_p_small=30).  A *step* is one SNP batch
of the per-batch hot loop (gwas.py:314-331): the CP x REP projection M S_i (245 fused
ciphertext multiplies at level 1550) plus the batch statistics (5 ct-mults, 1 pt-mult,
67 rotations, 1 conjugation).  The setup (logistic regression, w^-1, z, M, z', M_dup) runs
once before the timed region and is timed separately; `whole_job` combines both into the
config-3 end-to-end rate.  Inputs are seeded synthetic data with the paper's shapes
(the iDASH dataset is not distributed); ciphertexts are encrypted with device RNG.

  value : SNPs/s over K timed steps with the batch ciphertexts resident in HBM
  e2e   : the same steps through the public API with the batch's 245 input ciphertexts
          copied from pinned host memory every step and the 3 result ciphertexts read back

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
N_SAMPLES, N_COV, K_PAPER = 245, 4, 10643


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log-n", type=int, default=17)
    ap.add_argument("--log-l", type=int, default=1700)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-primitives", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
def dist_setup():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks() -> dict:
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


# ---------------------------------------------------------------------------------------------
def probe_integer_peaks(ctx, torch):
    """Register-resident probes of the exact instruction mixes the kernels execute."""
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    out = {}
    for name, fn, iters in (("butterflies_per_s", ctx.lib.hg_bench_modmul, 8192),
                            ("macs_per_s", ctx.lib.hg_bench_mac, 4096)):
        ops = ctypes.c_double()
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn(ctx.handle, iters, ctypes.c_void_p(sink.data_ptr()), ctypes.byref(ops), ctx.stream())
            e.record()
            torch.cuda.synchronize()
            best = max(best, ops.value / (s.elapsed_time(e) / 1e3))
        out[name] = best
    return out


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    import paper_1902_04303_b200 as hg
    from paper_1902_04303_b200 import _lib
    from paper_1902_04303_b200.data import synth_gwas_dataset
    from paper_1902_04303_b200.gwas import (
        GwasConfig,
        HostSnpBatch,
        SnpBatchStream,
        build_snp_batch,
        compute_batch,
        compute_setup,
        encrypt_gwas_inputs,
        plan_setup,
    )

    from paper_1902_04303_b200.parallel import compute_setup_sharded, shard_batches

    if os.environ.get("HG_BENCH_NOGC") == "1":   # diagnostic: are host stalls the cyclic collector?
        import gc

        gc.disable()
    # a process that has just exited (e.g. the test run before this bench) can still be releasing
    # its device memory: wait, bounded, until the GPU is (nearly) empty before sizing the pools
    t_wait = time.time()
    while time.time() - t_wait < 60:
        free, total = torch.cuda.mem_get_info()
        if free > 0.95 * total:
            break
        time.sleep(0.5)
    params = hg.CkksParams(log_n=args.log_n, log_l=args.log_l, log_p=45, log_p_small=30)
    t_wall0 = time.time()
    # every rank holds the same keys and setup inputs: the column-split setup combines their
    # ciphertexts (parallel.compute_setup_sharded)
    sk, pk, evk, rot = hg.keygen(params, 1000, device_rng=True)
    engine = hg.HeEngine(params, evk, rot)
    ctx = _lib.get_context(params.log_n)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    tau = 2 * params.slot_count // 256
    ds = synth_gwas_dataset(N_SAMPLES, N_COV, tau, seed=0)
    config = GwasConfig(n=N_SAMPLES, d=N_COV, k=K_PAPER).resolve(params)
    inputs = encrypt_gwas_inputs(ds, GwasConfig(n=N_SAMPLES, d=N_COV, k=tau), params, pk, gen,
                                 lazy_batches=True)
    torch.cuda.synchronize()
    t_keys_inputs = time.time() - t_wall0

    # -- one batch of SNP ciphertexts, resident + a pinned host copy --------------------------------
    batch = build_snp_batch(ds.S, 0, inputs.config, params, pk, gen)
    hbatch = HostSnpBatch.from_device(batch) if not args.no_e2e else None
    torch.cuda.synchronize()
    if hbatch is not None:
        batch = None   # the whole job streams from the host copy; resident again for the timed steps

    def mem_note(tag):
        if os.environ.get("HG_BENCH_DEBUG"):
            free, total = torch.cuda.mem_get_info()
            print(f"[bench] {tag}: free {free / 1e9:.1f} of {total / 1e9:.1f} GB, torch reserved "
                  f"{torch.cuda.memory_reserved() / 1e9:.1f} / allocated {torch.cuda.memory_allocated() / 1e9:.1f} GB, "
                  f"library pool {ctx.pool_bytes() / 1e9:.1f} / in use {ctx.pool_bytes(True) / 1e9:.1f} GB",
                  file=sys.stderr, flush=True)

    mem_note("before the whole job")

    def read_back(out, keep):
        """the step's 3 result ciphertexts -> pinned host memory, stream-ordered (no host stall)"""
        host = []
        for c in (out.num_ct, out.den_even_ct, out.den_odd_ct):
            for w in (c.c0.words, c.c1.words):
                h = torch.empty(w.shape, dtype=w.dtype, pin_memory=True)
                h.copy_(w, non_blocking=True)
                host.append(h)
        keep.append((out, host))
        return sum(int(h.numel()) * 4 for h in host)

    # -- the whole config-3 job, cold, end to end: setup once, then all 21 batches streamed from
    #    pinned host memory (SnpBatchStream: side-stream uploads, per-row ready events) with every
    #    batch's results read back -- device-timed; the setup is bracketed on its own as well ------
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_setup = torch.cuda.Event(enable_timing=True)
    nb = math.ceil(K_PAPER / tau)
    my_batches = len(shard_batches(nb, rank, world))   # round-robin SNP batches of this rank
    barrier(world)
    torch.cuda.synchronize()
    s.record()
    # rows stream at the projector's level (the M S_i products read only those words).  The ring
    # (3 slots) starts before the setup's last stage, as compute_gwas_encrypted(cache=stream) does
    # for an early stream: its uploads are issued by the stream's own thread (issuing a batch's
    # copies blocks for as long as the copy queue is full), so the setup keeps its time and the
    # first ~12 batches find their rows in HBM (same-box A/B: whole job 8.36 -> 7.91 s,
    # profiles/r2_stream_early_v4_ab.txt).  HG_STREAM_EARLY=0: ring started after the setup
    m_level = params.log_l - 150
    stream = None
    early = os.environ.get("HG_STREAM_EARLY", "1") == "1" and world == 1
    n_slots = int(os.environ.get("HG_STREAM_SLOTS", "3" if early else "2"))
    when = os.environ.get("HG_STREAM_WHEN", "dup")   # "dup": before the M_dup ladders; "start": with the setup
    if hbatch is not None and early:
        # the first uploads run while the setup's kernels leave the PCIe link idle
        stream = SnpBatchStream([hbatch] * my_batches, params, level=m_level, slots=n_slots, early=True)
        if when == "start":
            plan_setup(engine, config)   # the ring's slots come out of the planned reservation
            stream.start()
    if hbatch is not None and stream is None:
        # as compute_gwas_encrypted(cache=stream) does: the ring's slots and events are allocated
        # behind the setup's last, device-bound stage; the uploads start after the setup
        stream = SnpBatchStream([hbatch] * my_batches, params, level=m_level, slots=n_slots)
    if world > 1:   # column-split setup + NCCL all-gathers of z' partials and M_dup
        beta, p_prev, inter, m_dup = compute_setup_sharded(engine, inputs, rank, world, gather_m=False)
    else:
        hook = None
        if stream is not None:
            hook = (stream.start if when == "dup" else None) if early else stream.allocate
        beta, p_prev, inter, m_dup = compute_setup(engine, inputs, before_dup=hook)
        del hook   # a bound method of the stream: the ring's slots go back when `stream` is deleted
    e_setup.record()
    if os.environ.get("HG_BENCH_DEBUG"):
        from paper_1902_04303_b200.ckks import KEY_CACHE

        free, total = torch.cuda.mem_get_info()
        print(f"[bench] after setup: free {free / 1e9:.1f} GB, torch reserved "
              f"{torch.cuda.memory_reserved() / 1e9:.1f} / allocated {torch.cuda.memory_allocated() / 1e9:.1f} GB, "
              f"library pool {ctx.pool_bytes() / 1e9:.1f} / in use {ctx.pool_bytes(True) / 1e9:.1f} GB, "
              f"key cache {KEY_CACHE.bytes / 1e9:.1f} GB, torch peak allocated "
              f"{torch.cuda.max_memory_allocated() / 1e9:.1f} GB", file=sys.stderr, flush=True)
    job_keep = []
    marks = []
    if inter.M.cols[0].level_bits != m_level:
        raise RuntimeError(f"projector level {inter.M.cols[0].level_bits} != the streamed level {m_level}")
    if stream is not None:
        for b in stream:
            read_back(compute_batch(engine, inputs, inter, m_dup, b), job_keep)
            if os.environ.get("HG_BENCH_DEBUG"):
                marks.append(torch.cuda.Event(enable_timing=True))
                marks[-1].record()
    e.record()
    torch.cuda.synchronize()
    t_setup = max_over_ranks(s.elapsed_time(e_setup) / 1e3, world)
    if marks:
        prev, per = e_setup, []
        for m in marks:
            per.append(round(prev.elapsed_time(m), 1))
            prev = m
        print(f"[bench] whole-job batch ms: {per}; library OOM retries {_lib.OOM_RETRIES}", file=sys.stderr,
              flush=True)
    t_whole = max_over_ranks(s.elapsed_time(e) / 1e3, world) if hbatch is not None else None
    b = None
    del job_keep, stream   # the ring's slots (k x 12.6 GB) go back before the resident steps
    if batch is None:
        batch = hbatch.to_device(params)
        torch.cuda.synchronize()

    def step_resident():
        return compute_batch(engine, inputs, inter, m_dup, batch)

    mem_note("before the resident steps")
    for _ in range(args.warmup):
        step_resident()
    torch.cuda.synchronize()

    # -- timed: K resident steps ----------------------------------------------------------------------
    launches0 = _lib.total_launches()
    # events bracket only the dominant kernel class inside the timed region (its roofline is
    # the one reported); the per-class breakdown comes from one extra, separately run step
    live_events = os.environ.get("HG_BENCH_NTT_EVENTS", "1") != "0"
    if live_events:
        ctx.set_kernel_timing(True, kinds=("ntt",))
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        s.record()
        outs = [step_resident() for _ in range(args.steps)]
        e.record()
        torch.cuda.synchronize()
    t_steps = s.elapsed_time(e) / 1e3
    barrier(world)
    launches = _lib.total_launches() - launches0
    ntt_live = ctx.kernel_stats("ntt")
    ctx.set_kernel_timing(False)
    t_steps = max_over_ranks(t_steps, world)
    del outs
    ctx.set_kernel_timing(True)
    step_resident()
    kstats = {k: ctx.kernel_stats(k) for k in ("crt", "modup", "ntt", "pointwise", "elementwise")}
    ctx.set_kernel_timing(False)
    for k in kstats:   # per-step figures from the breakdown step, scaled to K steps
        kstats[k] = {kk: v * args.steps for kk, v in kstats[k].items()}
    if live_events:
        kstats["ntt"] = ntt_live
    if os.environ.get("HG_PROFILE_STEP"):
        # one more step inside a profiler window: `ncu --profile-from-start off` sees exactly it
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        step_resident()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()

    # -- e2e: host -> device inputs, device -> host results, through the public API ------------------
    # The batch's 245 ciphertexts sit in pinned host memory; SnpBatchStream copies batch i+1 on a
    # side stream while batch i computes; every step's 3 result ciphertexts are read back.
    e2e = None
    mem_note("before e2e")
    if not args.no_e2e:
        def run_e2e(nsteps):
            # every step's 3 result ciphertexts are copied to pinned host memory asynchronously
            # (stream-ordered after the step's kernels); the caller's synchronize() closes the
            # timed region, so all reads complete inside it without a host stall per step
            d2h, keep = 0, []
            for b in SnpBatchStream([hbatch] * nsteps, params, level=m_level):
                d2h = read_back(compute_batch(engine, inputs, inter, m_dup, b), keep)
            return d2h

        run_e2e(1)
        torch.cuda.synchronize()
        barrier(world)
        s.record()
        d2h = run_e2e(args.steps)
        e.record()
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(s.elapsed_time(e) / 1e3, world)
        h2d = hbatch.nbytes_at(m_level)
        e2e = {"value": round(tau * args.steps * world / t_e2e, 3), "unit": "SNP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(1e3 * t_e2e / args.steps, 2)}

    peaks = probe_integer_peaks(ctx, torch)
    prims = None if args.no_primitives else measure_primitives(torch, hg, _lib)
    return {
        "params": params, "tau": tau, "t_setup": t_setup, "t_steps": t_steps, "t_whole": t_whole,
        "launches": launches, "kstats": kstats, "clocks": clocks.summary(), "e2e": e2e,
        "peaks": peaks, "t_keys_inputs": t_keys_inputs, "primitives": prims,
        "key_cache_gb": round(__import__("paper_1902_04303_b200.ckks", fromlist=["KEY_CACHE"]).KEY_CACHE.bytes / 1e9, 2),
    }


def measure_primitives(torch, hg, _lib, log_n: int = 16, level: int = 1550, reps: int = 20):
    """BASELINE's secondary metric: key switches / NTTs per second at N=2^16 (device-timed,
    inputs resident).  Key switch = the relinearisation switch of a level-1550 ciphertext
    (ModUp to the key basis, NTT, x.key fused into the inverse NTT, CRT window [L, L+l));
    NTT = one length-2^16 negacyclic transform over one 30-bit prime (batches of 163 rows)."""
    import ctypes  # noqa: F401
    import numpy as np

    from paper_1902_04303_b200 import ckks

    params = hg.CkksParams(log_n=log_n, log_l=1700, log_p=45, log_p_small=30)
    sk, pk, evk, rot = hg.keygen(params, 5, device_rng=True)
    eng = hg.HeEngine(params, evk, rot)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    v = np.random.default_rng(2).uniform(-1, 1, params.slot_count)
    a = hg.mod_down(hg.encrypt_values(v, 45, pk, params, gen), level)
    b = hg.mod_down(hg.encrypt_values(v[::-1], 45, pk, params, gen), level)
    key = (evk.b, evk.a)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 1e3 / reps

    t_ks = timed(lambda: ckks._keyswitch(a.c1, key, level, params.log_l))
    t_mult = timed(lambda: eng.mult(a, b))
    t_rot = timed(lambda: eng.rotate(a, 1))
    ctx = _lib.get_context(log_n)
    rows = 163
    buf = torch.randint(0, 1 << 20, (rows, params.n), dtype=torch.int32, device="cuda")
    t_ntt = timed(lambda: _lib.check(ctx.lib.hg_ntt_forward(ctx.handle, buf.data_ptr(), rows, 0, ctx.stream())))
    t_intt = timed(lambda: _lib.check(ctx.lib.hg_ntt_inverse(ctx.handle, buf.data_ptr(), rows, 0, ctx.stream())))
    # automorphism x -> x^5 of a level-1550 polynomial: a pure permutation-with-sign (HBM-bound)
    # HBM-bound ops over 10 distinct level-1550 polys (10 x 25.7 MB > the 126 MB L2), cycled
    polys = [hg.mod_down(hg.encrypt_values(v * (1 + 0.01 * i), 45, pk, params, gen), level).c0
             for i in range(10)]
    cyc = {"i": 0}

    def nxt():
        cyc["i"] = (cyc["i"] + 1) % len(polys)
        return polys[cyc["i"]]
    def kernel_time(fn):
        """device time of the elementwise kernel itself (CUDA events around each launch):
        one Python-level op costs more host time than its kernel takes"""
        fn()
        torch.cuda.synchronize()
        ctx.set_kernel_timing(True, kinds=("elementwise",))
        for _ in range(reps):
            fn()
        st = ctx.kernel_stats("elementwise")
        ctx.set_kernel_timing(False)
        return st["ms"] / 1e3 / max(1, st["launches"])
    t_aut = kernel_time(lambda: nxt().automorphism(5))
    t_add = kernel_time(lambda: nxt().add(nxt()))
    peak = (load_peaks().get("hbm_gbs") or 6550.4) * 1e9
    w64 = lambda bits: -(-bits // 64)  # noqa: E731  (SURVEY §8(d) counts radix-2^64 limbs)
    ks_bytes = 8 * params.n * (w64(level) + 2 * w64(level + params.log_l) + 2 * w64(level))
    aut_bytes = 2 * params.n * 4 * -(-level // 32)
    return {"N": params.n, "level_bits": level, "keyswitch_per_s": round(1 / t_ks, 1),
            "keyswitch_hbm": {"algorithmic_bytes": ks_bytes, "GBps": round(ks_bytes / t_ks / 1e9, 1),
                              "frac_of_hbm_peak": round(ks_bytes / t_ks / peak, 4),
                              "note": "SURVEY §8(d) bytes (x, key pair, output pair); the key switch is "
                                      "integer-pipe / tensor bound (NTT + base conversions), so its HBM "
                                      "fraction is low by construction"},
            "automorphism": {"kernel_us": round(t_aut * 1e6, 2), "GBps": round(aut_bytes / t_aut / 1e9, 1),
                             "frac_of_hbm_peak": round(aut_bytes / t_aut / peak, 4),
                             "bytes": aut_bytes},
            "add": {"kernel_us": round(t_add * 1e6, 2), "GBps": round(1.5 * aut_bytes / t_add / 1e9, 1),
                    "frac_of_hbm_peak": round(1.5 * aut_bytes / t_add / peak, 4), "bytes": 3 * aut_bytes // 2},
            "ct_mult_rescale_per_s": round(1 / t_mult, 1), "rotation_per_s": round(1 / t_rot, 1),
            "ntt_per_s": round(rows / t_ntt), "intt_per_s": round(rows / t_intt),
            "ntt_butterflies_per_s": round(rows / t_ntt * (params.n // 2) * log_n / 1e9, 1),
            "note": "device-timed, resident inputs; NTT = one length-N transform over one prime"}


def ncu_traffic(dom: str):
    """DRAM bytes per unit of the dominant kernel from the committed `ncu --set full` capture
    (profiles/r2_ncu_traffic.json): per row-pass of the contiguous NTT pass (the largest NTT
    launch), against its algorithmic read+write of 2^17 words."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.json")) as f:
            cap = json.load(f)
    except OSError:
        return None
    if dom != "ntt":
        return None
    for ln in cap["launches"]:
        if ln["kernel"].startswith("void ntt_lo8_kernel<1, 11, 2>"):
            rows = int(ln["grid_size"]) // 32   # 64 chunks per row, 2 rows per block: 32 blocks/row
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3}.get(ln["unit"], 1.0)
            per_row = (ln["dram_read"] + ln["dram_write"]) * scale / rows
            return {"bytes_per_row_pass": round(per_row), "algorithmic_bytes_per_row_pass": 2 * (1 << 17) * 4,
                    "ratio": round(per_row / (2 * (1 << 17) * 4), 3),
                    "source": "profiles/r2_ncu_traffic.json (ncu --set full, ntt_lo8_kernel<1,11,2>, "
                              f"{rows} rows); the excess over 1.0 is the twiddle table"}
    return None


# ---------------------------------------------------------------------------------------------
# CPU baseline: the reference evaluator's time is >= 99.7% big Kronecker products (hegwas
# ring.py:46-58, the multiply at :55), so one batch step's CPU cost is the sum over its
# products, each timed at its exact operand widths through oracle/ (the reference algorithm
# restated, libgmp's mpz_mul for the big multiply).

def batch_step_products(big_l: int = 1700, log_p: int = 45, log_p_small: int = 30) -> dict:
    """{(a_bits, b_bits): count} of the big products in one config-3 batch step at P17, from the
    reference's own op sequence (gwas.py:197-229, 325-331; ckks.py:166-194, 256-279):
    a ct-mult at level l = 4 tensor products l x l + 2 key-switch products l x (l + L); a rotation
    or conjugation = 2 key-switch products; a plaintext mult = 2 products l x l (the mask is held
    mod 2^l).  Levels: M at 1700-150, S' = M S at 1505, w 545, z' 185 (SURVEY §8 level table)."""
    lm = big_l - 150
    s1 = lm - log_p                                  # S' = M S_i
    lw, lz = 545, 185
    wz = min(lw, lz) - log_p                         # w z' (aligned at z')
    num = wz - log_p                                 # dup(w z') S'
    wm = lw - log_p_small                            # w (.) 0.5-mask
    ws = wm - log_p                                  # dup(w_m) S'
    den = ws - log_p                                 # ws S', ws conj(S')
    prods: dict = {}

    def add(a, b, k):
        prods[(a, b)] = prods.get((a, b), 0) + k

    def mult(level, k=1):
        add(level, level, 4 * k)
        add(level, level + big_l, 2 * k)

    def rot(level, k=1):
        add(level, level + big_l, 2 * k)

    mult(lm, 245)                                    # orthogonalize_snps: 245 ct-mults
    mult(lz)                                         # w z'
    rot(wz, 8)                                       # duplicate(w z', 256)
    mult(wz)                                         # num terms
    rot(num, 8 + 9)                                  # col_sum: 8 ladder steps + rotate_left(255)
    add(lw, lw, 2)                                   # mult_plain(w, range-value mask)
    rot(wm, 8)                                       # duplicate(w_m)
    mult(wm)                                         # ws
    mult(ws, 2)                                      # wss, wsc
    rot(s1)                                          # conjugate(S')
    rot(den, 2 * 17)                                 # two col_sums
    return prods


def cpu_product_sample(log_n: int, a_bits: int, b_bits: int, seed: int = 0) -> float:
    """Seconds for one exact negacyclic product of uniform a_bits x b_bits operands through
    oracle/ (ring.py:46-58 restated; gmp multiply), single thread."""
    import random

    from oracle import ring_oracle as R

    n = 1 << log_n
    rng = random.Random(seed)
    a = [rng.getrandbits(a_bits) for _ in range(n)]
    b = [rng.getrandbits(b_bits) for _ in range(n)]
    t = time.perf_counter()
    R.negacyclic_mul(a, b, n, a_bits, b_bits)
    return time.perf_counter() - t


def cpu_step_seconds(prods: dict, times: dict) -> float:
    """CPU-seconds of one batch step: every product class at its timed cost; a class without its
    own sample takes the nearest timed class's cost scaled by operand width (a + b)."""
    total = 0.0
    for (a, b), k in prods.items():
        if (a, b) in times:
            t = times[(a, b)]
        else:
            ref = min(times, key=lambda c: abs(c[0] + c[1] - a - b))
            t = times[ref] * (a + b) / (ref[0] + ref[1])
        total += k * t
    return total


def cpu_baseline_sample(log_n: int, big_l: int) -> dict:
    """Rank 0, N=1: the batch step's four costliest product classes timed once each on one core
    (~15-20 s at P17), the step's CPU time summed over its exact product list."""
    prods = batch_step_products(big_l)
    ranked = sorted(prods, key=lambda c: -prods[c] * (c[0] + c[1]))[:4]
    times = {c: cpu_product_sample(log_n, c[0], c[1], i) for i, c in enumerate(ranked)}
    sec = cpu_step_seconds(prods, times)
    return {"step_cpu_s": sec, "classes_timed": {f"{a}x{b}": round(t, 2) for (a, b), t in times.items()},
            "products": sum(prods.values())}


def run_reference(args, world, rank):
    """--impl reference: the reference algorithm (CPU oracle port; the reference is pure
    Python and cannot travel) on all host cores.  Each timed step runs `cores` concurrent exact
    products of the batch step's product classes (cycled, so every class is sampled); the step's
    CPU time is the exact product list x the per-class median; value = SNP/s with all cores."""
    if rank != 0:
        return None
    from concurrent.futures import ProcessPoolExecutor

    cores = os.cpu_count() or 1
    tau = 2 * (1 << (args.log_n - 1)) // 256
    prods = batch_step_products(args.log_l)
    classes = sorted(prods, key=lambda c: -prods[c] * (c[0] + c[1]))
    samples: dict = {c: [] for c in classes}
    walls = []
    with ProcessPoolExecutor(max_workers=cores) as ex:
        for i in range(args.warmup + args.steps):
            timed = i >= args.warmup
            # warm-up steps load gmp and fork the workers on a small ring; timed steps sample
            # the full-size classes
            log_n = args.log_n if timed else min(args.log_n, 12)
            k0 = (i - args.warmup) * cores if timed else 0
            picks = [classes[(k0 + c) % len(classes)] for c in range(cores)]
            t = time.perf_counter()
            res = list(ex.map(cpu_product_sample, [log_n] * cores, [c[0] for c in picks],
                              [c[1] for c in picks], range(cores)))
            dt = time.perf_counter() - t
            if timed:
                walls.append(dt)
                for c, r in zip(picks, res):
                    samples[c].append(r)
    times = {c: statistics.median(v) for c, v in samples.items() if v}
    step_cpu = cpu_step_seconds(prods, times)
    value = tau * cores / step_cpu
    line = {
        "impl": "reference", "metric": "encrypted semi-parallel GWAS SNPs/s", "value": value,
        "unit": "SNP/s", "higher_is_better": True, "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "dtype": "u32", "data": "synthetic",
        "ms_per_step": round(1e3 * statistics.median(walls), 1),
        "config": {"workload": f"config3 per-batch step, P17 (N=2^{args.log_n}, log_l={args.log_l}), "
                               f"{tau} SNPs/batch, n=245", "scaling": "n/a"},
        "cpu_baseline": {"value": value, "unit": "SNP/s", "cores": cores, "kind": "port",
                         "sample": f"each step: {cores} concurrent exact negacyclic products (oracle/, gmp) "
                                   f"cycling over the batch step's {len(classes)} product classes; step CPU "
                                   f"time = its {sum(prods.values())} products (245 ct-mults at 1550 + the "
                                   f"statistics' 5 ct-mults, 1 pt-mult, 67 rotations, 1 conjugation) x the "
                                   f"per-class medians = {step_cpu:.0f} core-s",
                         "classes_s": {f"{a}x{b}": round(t, 2) for (a, b), t in times.items()}},
        "e2e": {"value": value, "unit": "SNP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    return line


# ---------------------------------------------------------------------------------------------
def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) started as a plain process: re-run it under torchrun with one
    rank per GPU (127.0.0.1 rendezvous, a free port); returns torchrun's exit code."""
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if env_world is not None and int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}; launch one rank per GPU")
    world, rank, local = dist_setup() if args.impl == "ours" else (
        int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        line = run_reference(args, world, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return
    r = run_ours(args, world, rank, local)
    if rank != 0:
        return
    peaks_file = load_peaks()
    tau, steps, params = r["tau"], args.steps, r["params"]
    value = tau * steps * world / r["t_steps"]
    ms_step = 1e3 * r["t_steps"] / steps
    nb = math.ceil(K_PAPER / tau)
    whole = K_PAPER / (r["t_setup"] + math.ceil(nb / world) * r["t_steps"] / steps)
    whole_e2e = K_PAPER / r["t_whole"] if r.get("t_whole") else None
    ks = r["kstats"]
    # roofline of the dominant kernel class (integer pipe: CRT reconstruction MACs)
    dom = max(("crt", "modup", "ntt"), key=lambda k: ks[k]["ms"])
    step_ms_total = 1e3 * r["t_steps"]
    peak_key = "butterflies_per_s" if dom == "ntt" else "macs_per_s"
    achieved = ks[dom]["work"] / (ks[dom]["ms"] / 1e3) if ks[dom]["ms"] else 0.0
    roofline = {
        "bound": "int32", "kernel": {"crt": "crt_kernel", "modup": "modup_kernel",
                                     "ntt": "ntt_lo/hi_kernel"}[dom],
        "achieved": round(achieved / 1e9, 1), "peak": round(r["peaks"][peak_key] / 1e9, 1),
        "unit": "G" + ("butterflies" if dom == "ntt" else "MAC") + "/s",
        "frac": round(achieved / r["peaks"][peak_key], 4) if r["peaks"][peak_key] else None,
        "traffic": ncu_traffic(dom),
        "peak_source": "measured in-run: register-resident probe running the NTT kernels' own butterfly "
                       "(hgntt::fwd_bfly: IMAD.HI + 2 IMAD on the fma pipe, VIADDMNMX + 2 IADD3 on the alu pipe), "
                       "a burst at the unthrottled clock (MEASURED_PEAKS.json has no integer-pipe figure)",
        "share_of_step": round(ks[dom]["ms"] / step_ms_total, 3) if step_ms_total else None,
        "kernel_classes": {k: {"ms_per_step": round(v["ms"] / steps, 2), "launches": v["launches"],
                               "G_work_per_s": round(v["work"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] else 0}
                           for k, v in ks.items()},
        "hbm_peak_gbs": peaks_file.get("hbm_gbs"),
    }
    # the tensor-core classes against the i8 dense peak (2x the measured bf16 dense figure on
    # Blackwell): their work unit is a 32x32-bit MAC = 16 u8 MACs = 32 int8 ops
    i8_tops = 2 * float(peaks_file.get("bf16_tflops") or 2250.0)
    for k in ("crt", "modup"):
        v = ks[k]
        if v["ms"]:
            tops = v["work"] * 32 / (v["ms"] / 1e3) / 1e12
            roofline["kernel_classes"][k]["int8_tops"] = round(tops, 1)
            roofline["kernel_classes"][k]["frac_of_i8_peak"] = round(tops / i8_tops, 4)
    roofline["i8_peak_tops"] = round(i8_tops, 1)
    # the timed steps run power-capped below the clock the burst probe sees: the same pipe's
    # peak at the step's own median SM clock, next to the burst figure
    clk = r.get("clocks") or {}
    if dom == "ntt" and clk.get("sm_mhz") and clk.get("sm_max_mhz") and roofline["frac"]:
        scale = min(1.0, clk["sm_mhz"] / clk["sm_max_mhz"])
        roofline["peak_at_step_clock"] = round(roofline["peak"] * scale, 1)
        roofline["frac_at_step_clock"] = round(roofline["frac"] / scale, 4)
        roofline["note"] = ("the probe runs the kernels' own butterfly since round 2 (3.75-3.93 T/s); round 1's "
                            "probe carried one more ALU instruction per butterfly (3.0-3.1 T/s), against which "
                            "the same kernels read 0.68; ncu of the contiguous passes: fma-heavy pipe 70-72% of "
                            "elapsed cycles, first stall math_pipe_throttle (profiles/r2_v4_ncu_mult4_full.txt)")
    cpu = None
    if not args.no_cpu_baseline and world == 1:   # the contract: rank 0 at N=1 only
        cb = cpu_baseline_sample(params.log_n, params.log_l)
        cpu = {"value": round(tau / cb["step_cpu_s"], 6), "unit": "SNP/s", "cores": 1, "kind": "port",
               "sample": f"the batch step's {cb['products']} exact products (ring.py:55 Kronecker multiplies: "
                         f"250 ct-mults, 1 pt-mult, 67 rotations, 1 conjugation) costed from one timed product "
                         f"per dominant class via oracle/ (gmp) at N=2^{params.log_n}: {cb['classes_timed']} s; "
                         f"{cb['step_cpu_s']:.0f} core-s per step"}
    line = {
        "metric": "encrypted semi-parallel GWAS SNPs/s", "value": round(value, 3), "unit": "SNP/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded; config-3 shapes, device-RNG encryption)",
        "config": {"workload": f"config3 per-batch step: n=245, d=4, {tau} SNPs/batch, "
                               f"P17 (N=2^{params.log_n}, log_l={params.log_l}, log_p=45, log_p_small=30)",
                   "global_batch_snps": tau * world, "parallelism": f"snp-batch sharding x{world}",
                   "l2": "inputs > L2 (13 GB of batch ciphertexts per step)"},
        "config0_job": {"snps": 256, "s": round(r["t_setup"] + r["t_steps"] / steps, 2),
                        "value": round(256 / (r["t_setup"] + r["t_steps"] / steps), 2), "unit": "SNP/s",
                        "note": "config 0 (n=245, 256 SNPs = one batch): the cold setup + one resident "
                                "batch step of this run (the setup does not depend on k)"},
        "whole_job": {"snps": K_PAPER, "batches": nb, "setup_s": round(r["t_setup"], 2),
                      "value": round(whole_e2e, 3) if whole_e2e else round(whole, 3), "unit": "SNP/s",
                      "measured_s": round(r["t_whole"], 2) if r.get("t_whole") else None,
                      "from_resident_steps": round(whole, 3),
                      "note": "config-3 whole job, measured cold and end to end: setup once + 21 SNP "
                              "batches streamed from pinned host memory with every batch's results read "
                              "back (the batch data is one seeded batch replayed 21 times); "
                              "from_resident_steps = setup + 21 x the resident step"},
        "e2e": r["e2e"], "gpu_launches": r["launches"], "roofline": roofline, "cpu_baseline": cpu,
        "clocks": r["clocks"], "int_peaks": {k: round(v / 1e9, 1) for k, v in r["peaks"].items()},
        "primitives": r["primitives"],
        "key_cache_gb": r["key_cache_gb"], "prep_s": round(r["t_keys_inputs"], 1),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

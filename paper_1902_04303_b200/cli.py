"""Command-line phases on the B200 evaluator: keygen, compute, decrypt (reference
hegwas/cli.py:108-341).

The on-disk artifacts are the reference's: key files (sk.bin, pk.bin, evk.bin,
rotkeys.bin, params.json), the encrypt phase's manifest.json + one HEGW file per
ciphertext, the compute phase's result ciphertexts + compute_manifest.json, results.tsv,
and run_report.json for timings.  So the phases interoperate with the reference's: a
directory written by ``hegwas keygen`` / ``hegwas encrypt`` is computed here on the GPU and
decrypted by either package -- and because the evaluator is bit-exact, the result files are
byte-identical to ``hegwas compute``'s (tests/test_gpu_cli.py, fixtures written by the
reference itself, tools/make_cli_golden.py).

``compute`` replaces the reference's disk-spilling CiphertextCache (cache.py)
with the HBM pool: the logistic-regression inputs are uploaded once, and the SNP batches
are read from disk by a reader thread one batch ahead of the GPU (``--prefetch``) and
parsed straight into device memory.  It never opens the secret key and records its own
file-access audit to prove it.  ``encrypt`` (CSV preprocessing, client side) is the
reference's.

    python -m paper_1902_04303_b200 compute --encrypted DIR --keys DIR --outdir DIR
"""
from __future__ import annotations

import argparse
import sys
import contextvars
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

from . import io as hio
from . import serialize
from .ckks import HeEngine
from .errors import HegwasError, InputError, MissingKeyError
from .gwas import (BatchOutput, EncryptedGwasInputs, GwasConfig, SnpBatch, assemble_result,
                   compute_gwas_encrypted, decrypt_statistics)
from .instrument import track_ops
from .keys import keygen
from .logreg import LogRegInputs
from .matrix import CPMatrix, REPMatrix, next_pow2
from .params import CkksParams, security_status

SK_FILE, PK_FILE, EVK_FILE, ROTKEYS_FILE, PARAMS_FILE = (
    "sk.bin", "pk.bin", "evk.bin", "rotkeys.bin", "params.json")
PARAM_FLAGS = ("log_n", "log_l", "log_p", "log_p_small", "sigma", "h")


def _params(args) -> CkksParams:
    fields = {}
    if getattr(args, "params_file", None):
        fields.update(vars(CkksParams.from_json(hio.read_text(args.params_file))))
    fields.update({k: getattr(args, k) for k in PARAM_FLAGS if getattr(args, k, None) is not None})
    if "log_n" not in fields or "log_l" not in fields:
        raise InputError("provide --params-file or at least --log-n and --log-l")
    return CkksParams(**fields)


def _load_params(keys_dir) -> CkksParams:
    return CkksParams.from_json(hio.read_text(Path(keys_dir) / PARAMS_FILE))


def _report(outdir, phase: str, seconds: float, counter=None, extra=None) -> None:
    """Merge one phase's wall time (and op counts) into outdir/run_report.json."""
    path = Path(outdir) / "run_report.json"
    report = hio.read_json(path) if path.exists() else {}
    entry = {"seconds": round(seconds, 4)}
    if counter is not None:
        entry["op_counts"] = counter.snapshot()
    entry.update(extra or {})
    report.setdefault("phases", {})[phase] = entry
    hio.write_json(path, report)


def _config_from_manifest(m: dict, params: CkksParams) -> GwasConfig:
    return GwasConfig(n=m["n"], d=m["d"], k=m["k"], kappa=m["kappa"], tau=m["tau"],
                      inverse_iters=m["inverse_iters"], inverse_guess=m["inverse_guess"],
                      complex_packing=m["complex_packing"]).resolve(params)


# -- keygen -----------------------------------------------------------------------------------------

def cmd_keygen(args) -> int:
    t0 = time.time()
    params = _params(args)
    status, note = security_status(params)
    if status != "accepted":
        print(f"[security] {status}: {note}", file=sys.stderr)
    sk, pk, evk, rot = keygen(params, args.seed)
    out = Path(args.outdir)
    log_n = params.log_n
    hio.write_bytes(out / SK_FILE, serialize.secret_key_to_bytes(sk, log_n))
    hio.write_bytes(out / PK_FILE, serialize.public_key_to_bytes(pk, log_n))
    hio.write_bytes(out / EVK_FILE, serialize.evaluation_key_to_bytes(evk, log_n))
    hio.write_bytes(out / ROTKEYS_FILE, serialize.rotation_keys_to_bytes(rot, log_n))
    hio.write_text(out / PARAMS_FILE, params.to_json())
    _report(out, "context", time.time() - t0, extra={"security": [status, note]})
    print(f"keys written to {out}")
    return 0


# -- compute ----------------------------------------------------------------------------------------

class _BatchReader:
    """Reads SNP batch files from disk `depth` batches ahead of the GPU on a thread (file
    I/O releases the GIL); the consumer parses each batch into device memory."""

    def __init__(self, encdir: Path, names: list[list[str]], depth: int):
        self.encdir = encdir
        self.names = names
        self.depth = max(0, depth)
        self.pool = ThreadPoolExecutor(max_workers=1) if self.depth else None
        self.pending: dict[int, object] = {}
        self.lock = threading.Lock()

    def _read(self, b: int) -> list[bytes]:
        return [hio.read_bytes(self.encdir / name) for name in self.names[b]]

    def get(self, b: int) -> list[bytes]:
        if self.pool is None:
            return self._read(b)
        with self.lock:
            for nb in range(b, min(b + 1 + self.depth, len(self.names))):
                if nb not in self.pending:
                    # the io audit is a ContextVar: run the worker's read in the caller's
                    # context so every prefetched batch file lands in the audit log
                    ctx = contextvars.copy_context()
                    self.pending[nb] = self.pool.submit(ctx.run, self._read, nb)
            fut = self.pending.pop(b)
        return fut.result()

    def close(self):
        if self.pool is not None:
            self.pool.shutdown(wait=True, cancel_futures=True)


def load_encrypted_inputs(encdir, params: CkksParams, prefetch: int = 1):
    """The reference encrypt phase's directory (manifest.json + HEGW files) as
    EncryptedGwasInputs whose SNP batches are produced lazily from disk."""
    encdir = Path(encdir)
    manifest = hio.read_json(encdir / "manifest.json")
    config = _config_from_manifest(manifest, params)
    files = manifest["files"]

    def load(name):
        return serialize.ciphertext_from_bytes(hio.read_bytes(encdir / name), params)

    n, d1 = manifest["n"], manifest["d"] + 1
    cs = next_pow2(n)
    logreg = LogRegInputs(
        X=CPMatrix(cols=[load(f) for f in files["x_cols"]], rows=n, cols_logical=d1),
        Xt_rep=REPMatrix(rows_ct=[load(f) for f in files["xt_rows"]], repeat=cs, rows=d1, cols_logical=n),
        XtX_inv=CPMatrix(cols=[load(f) for f in files["xtx_inv_cols"]], rows=d1, cols_logical=d1),
        y=load(files["y"]),
    )
    reader = _BatchReader(encdir, files["batches"], prefetch)

    def batch(b: int) -> SnpBatch:
        offset = b * config.tau
        count = min(config.tau, config.k - offset)
        width = (count + 1) // 2 if config.complex_packing else count
        rows = [serialize.ciphertext_from_bytes(blob, params) for blob in reader.get(b)]
        return SnpBatch(index=b, S_packed=REPMatrix(rows_ct=rows, repeat=cs, rows=n, cols_logical=width),
                        snp_offset=offset, snp_count=count, complex_packing=config.complex_packing)

    inputs = EncryptedGwasInputs(logreg=logreg, batches=[], config=config, batch_source=batch)
    return inputs, manifest, reader


def cmd_compute(args) -> int:
    t0 = time.time()
    keys_dir = Path(args.keys)
    params = _load_params(keys_dir)
    try:
        evk = serialize.evaluation_key_from_bytes(hio.read_bytes(keys_dir / EVK_FILE))
    except FileNotFoundError:
        raise MissingKeyError(f"evaluation key file missing: {keys_dir / EVK_FILE}") from None
    try:
        rot = serialize.rotation_keys_from_bytes(hio.read_bytes(keys_dir / ROTKEYS_FILE))
    except FileNotFoundError:
        needed = [1 << j for j in range((params.n // 4).bit_length())]
        raise MissingKeyError(f"rotation keys missing: {keys_dir / ROTKEYS_FILE}; required key set is "
                              f"rotation amounts {needed} plus the conjugation key") from None
    out = Path(args.outdir)
    with hio.audit_file_access() as audit, track_ops() as counter:
        inputs, manifest, reader = load_encrypted_inputs(Path(args.encrypted), params, args.prefetch)
        try:
            outputs = compute_gwas_encrypted(HeEngine(params, evk, rot), inputs)
        finally:
            reader.close()
        results, cts = {"batches": []}, []
        for o in outputs.batch_outputs:
            entry = {"num": f"num_b{o.index:03d}.ct", "den_even": f"den_even_b{o.index:03d}.ct"}
            parts = [("num", o.num_ct), ("den_even", o.den_even_ct)]
            if o.den_odd_ct is not None:
                entry["den_odd"] = f"den_odd_b{o.index:03d}.ct"
                parts.append(("den_odd", o.den_odd_ct))
            for key, ct in parts:
                hio.write_bytes(out / entry[key], serialize.ciphertext_to_bytes(ct))
                cts.append(ct)
            results["batches"].append(entry)
    accessed = sorted({p for _, p in audit})
    sk_path = str((keys_dir / SK_FILE).resolve())
    depth = {"ct_rescales": max(c.depth_ct for c in cts), "pt_rescales": max(c.depth_pt for c in cts)}
    hio.write_json(out / "compute_manifest.json", {
        "results": results, "source_manifest": manifest, "op_counts": counter.snapshot(),
        "critical_path": depth, "rotations_power_of_two": counter.all_rotations_power_of_two(),
        "file_access_audit": accessed, "secret_key_accessed": sk_path in accessed,
    })
    _report(out, "compute", time.time() - t0, counter=counter, extra={"critical_path": depth})
    print("Homomorphic Operation         No. Operations")
    print(f"Plaintext Multiplication      {counter.pt_mults}")
    print(f"Ciphertext Multiplication     {counter.ct_mults}")
    print(f"Ciphertext Rotation           {counter.rotations}")
    print("Successive (critical path):")
    print(f"  Ciphertext-mult rescales    {depth['ct_rescales']}")
    print(f"  Plaintext-mult rescales     {depth['pt_rescales']}")
    if sk_path in accessed:
        raise HegwasError("privacy violation: compute phase read the secret key")
    print(f"encrypted statistics written to {out}")
    return 0


# -- decrypt ----------------------------------------------------------------------------------------

def cmd_decrypt(args) -> int:
    t0 = time.time()
    keys_dir = Path(args.keys)
    params = _load_params(keys_dir)
    sk = serialize.secret_key_from_bytes(hio.read_bytes(keys_dir / SK_FILE))
    resdir = Path(args.results)
    cm = hio.read_json(resdir / "compute_manifest.json")
    manifest = cm["source_manifest"]
    config = _config_from_manifest(manifest, params)

    def load(name):
        return serialize.ciphertext_from_bytes(hio.read_bytes(resdir / name), params)

    outputs = [BatchOutput(index=b, num_ct=load(e["num"]), den_even_ct=load(e["den_even"]),
                           den_odd_ct=load(e["den_odd"]) if "den_odd" in e else None)
               for b, e in enumerate(cm["results"]["batches"])]
    res = assemble_result(*decrypt_statistics(outputs, config, params, sk))
    out = Path(args.outdir)
    ids = manifest["snp_ids"]
    hio.write_tsv(out / "results.tsv", ["snp_id", "numerator", "denominator", "beta", "stderr", "pvalue"],
                  [(ids[i], res.numerator[i], res.denominator[i], res.effects[i], res.std_err[i],
                    res.p_values[i]) for i in range(config.k)])
    _report(out, "decrypt", time.time() - t0)
    print(f"results written to {out / 'results.tsv'}")
    return 0


# -- entry --------------------------------------------------------------------------------------------

def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1902_04303_b200",
                                 description="B200 evaluator phases (artifacts compatible with hegwas)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sp = sub.add_parser("keygen", help="generate key material (bit-identical to hegwas keygen)")
    sp.add_argument("--params-file")
    for flag in PARAM_FLAGS:
        sp.add_argument("--" + flag.replace("_", "-"), dest=flag, type=float if flag == "sigma" else int)
    sp.add_argument("--seed", type=int, default=0)
    sp.add_argument("--outdir", required=True)
    sp = sub.add_parser("compute", help="run the encrypted pipeline on the GPU (no secret key)")
    sp.add_argument("--encrypted", required=True)
    sp.add_argument("--keys", required=True)
    sp.add_argument("--outdir", required=True)
    sp.add_argument("--prefetch", type=int, default=1, help="SNP batches read ahead from disk")
    sp = sub.add_parser("decrypt", help="decrypt statistics and export results.tsv")
    sp.add_argument("--results", required=True)
    sp.add_argument("--keys", required=True)
    sp.add_argument("--outdir", required=True)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return {"keygen": cmd_keygen, "compute": cmd_compute, "decrypt": cmd_decrypt}[args.cmd](args)

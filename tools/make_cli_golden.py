"""Run the REFERENCE's own CLI phases (hegwas keygen / encrypt / compute / decrypt) on a toy
dataset and keep their on-disk artifacts as fixtures: tests/golden/cli_toy/{inputs,keys,
encrypted,computed,decrypted}.  tests/test_gpu_cli.py feeds the reference-written keys and
encrypted inputs to this repo's GPU `compute` phase and requires byte-identical result
ciphertexts.  Needs /root/reference (run in the build container, not on the GPU box).

    python tools/make_cli_golden.py [--out tests/golden/cli_toy]
"""
import argparse
import os
import shutil
import subprocess
import sys

import numpy as np

REF = "/root/reference/pkg/src"


def run(*args, cwd):
    env = dict(os.environ, PYTHONPATH=REF)
    print("$ hegwas", " ".join(args), flush=True)
    subprocess.run([sys.executable, "-m", "hegwas", *args], check=True, env=env, cwd=cwd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "cli_toy"))
    args = ap.parse_args()
    out = os.path.abspath(args.out)
    shutil.rmtree(out, ignore_errors=True)
    os.makedirs(out)
    sys.path.insert(0, REF)
    from hegwas.data import write_fixture_csvs   # the reference's own fixture writer

    rs = np.random.default_rng(11)
    n, d, k = 8, 4, 16
    covars = np.column_stack([rs.binomial(1, 0.5, n), rs.normal(50, 10, n), rs.normal(0, 1, (n, d - 2))])
    pheno = rs.binomial(1, 0.5, n)
    maf = rs.uniform(0.05, 0.5, k)
    dos = rs.binomial(2, maf, (n, k)).astype(float)
    dos[3, 5] = np.nan                      # one missing call: mean imputation path
    paths = write_fixture_csvs(os.path.join(out, "inputs"), covars, pheno, dos)
    run("keygen", "--log-n", "7", "--log-l", "1700", "--log-p", "45", "--log-p-small", "30",
        "--seed", "3", "--outdir", "keys", cwd=out)
    run("encrypt", "--covariates", paths["covariates"], "--pheno", paths["pheno"], "--snps", paths["snps"],
        "--keys", "keys", "--seed", "4", "--outdir", "encrypted", cwd=out)
    run("compute", "--encrypted", "encrypted", "--keys", "keys", "--outdir", "computed", cwd=out)
    run("decrypt", "--results", "computed", "--keys", "keys", "--outdir", "decrypted", cwd=out)
    # wall-clock reports vary run to run; keep only data artifacts
    for sub in ("keys", "encrypted", "computed", "decrypted"):
        rep = os.path.join(out, sub, "run_report.json")
        if os.path.exists(rep):
            os.remove(rep)


if __name__ == "__main__":
    main()

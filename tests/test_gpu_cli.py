"""The CLI phases against artifacts written by the REFERENCE's own CLI (tests/golden/cli_toy,
tools/make_cli_golden.py: hegwas keygen / encrypt / compute / decrypt on a toy dataset).

The reference-written keys and encrypted inputs go through this repo's GPU `compute`; every
result ciphertext file must be byte-identical to `hegwas compute`'s, the compute manifest
must carry the same op counts / critical path / result names, and `decrypt` must reproduce
the reference's results.tsv.  `keygen` with the same seed must write the same key files."""
import filecmp
import json
import os
import shutil

import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli_toy")


@pytest.fixture(scope="module")
def computed(tmp_path_factory):
    from paper_1902_04303_b200 import cli

    out = tmp_path_factory.mktemp("cli")
    enc, keys = out / "encrypted", out / "keys"
    shutil.copytree(os.path.join(GOLD, "encrypted"), enc)
    shutil.copytree(os.path.join(GOLD, "keys"), keys)
    assert cli.main(["compute", "--encrypted", str(enc), "--keys", str(keys), "--outdir",
                     str(out / "computed"), "--prefetch", "1"]) == 0
    return out


def test_compute_results_byte_identical_to_reference(computed):
    ref = json.load(open(os.path.join(GOLD, "computed", "compute_manifest.json")))
    ours = json.load(open(computed / "computed" / "compute_manifest.json"))
    for key in ("results", "op_counts", "critical_path", "rotations_power_of_two", "source_manifest"):
        assert ours[key] == ref[key], key
    assert ours["secret_key_accessed"] is False
    assert not any(p.endswith("sk.bin") for p in ours["file_access_audit"])

    # the audited file set (relative to the phase directories) is the reference's: every
    # prefetched SNP batch file read on the reader thread is logged too
    def rel(paths):
        return sorted("/".join(p.split("/")[-2:]) for p in paths)
    assert rel(ours["file_access_audit"]) == rel(ref["file_access_audit"])
    for entry in ref["results"]["batches"]:
        for name in entry.values():
            assert filecmp.cmp(computed / "computed" / name, os.path.join(GOLD, "computed", name),
                               shallow=False), name


def test_decrypt_matches_reference_tsv(computed):
    from paper_1902_04303_b200 import cli

    assert cli.main(["decrypt", "--results", str(computed / "computed"), "--keys", str(computed / "keys"),
                     "--outdir", str(computed / "decrypted")]) == 0
    assert open(computed / "decrypted" / "results.tsv").read() == \
        open(os.path.join(GOLD, "decrypted", "results.tsv")).read()


def test_keygen_writes_reference_key_files(tmp_path):
    from paper_1902_04303_b200 import cli

    params = json.load(open(os.path.join(GOLD, "keys", "params.json")))
    assert cli.main(["keygen", "--log-n", str(params["log_n"]), "--log-l", str(params["log_l"]),
                     "--log-p", str(params["log_p"]), "--log-p-small", str(params["log_p_small"]),
                     "--seed", "3", "--outdir", str(tmp_path)]) == 0
    for name in ("sk.bin", "pk.bin", "evk.bin", "rotkeys.bin", "params.json"):
        assert filecmp.cmp(tmp_path / name, os.path.join(GOLD, "keys", name), shallow=False), name

"""Top SASS instructions by warp-stall samples from `ncu -i X --page source --csv`."""
import csv
import io
import sys
from collections import Counter


def main(path, top=40):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    rows = [r for r in rows if r["Address"] != "Address"]
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    total = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
    agg = Counter()
    for r in rows:
        for c in stall_cols:
            agg[c] += int(r[c] or 0)
    print("total samples", total)
    print("stall mix:", ", ".join(f"{k[6:]}={100 * v / total:.1f}%" for k, v in agg.most_common(8)))
    hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]
    for r in hot:
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        reasons = sorted(((int(r[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"{100 * s / total:5.1f}% {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in reasons))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)


def opcode_mix(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))) if r["Address"] != "Address"]
    mix = Counter()
    samp = Counter()
    for r in rows:
        op = r["Source"].strip()
        if op.startswith("@"):
            op = op.split(None, 1)[1] if " " in op else op
        op = op.split()[0] if op else "?"
        mix[op] += int(r["Instructions Executed"] or 0)
        samp[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    tot = sum(mix.values())
    print("warp-instructions executed", tot)
    for op, v in mix.most_common(25):
        print(f"  {op:24s} {v:12d} {100 * v / tot:5.1f}%  samples {samp[op]}")

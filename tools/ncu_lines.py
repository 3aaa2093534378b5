"""Warp-stall samples per CUDA source line from `ncu -i X --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py report.csv [top]
"""
import csv
import sys
from collections import Counter


def _i(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    cols = rows[hdr]
    k_all = cols.index("Warp Stall Sampling (All Samples)")
    k_ex = cols.index("Instructions Executed")
    stall_cols = [(i, c) for i, c in enumerate(cols) if c.startswith("stall_") and "Not Issued" not in c]
    lines, total = [], 0
    fname = ""
    for r in rows[hdr + 1:]:
        if r and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        if r and r[0] not in ("", "Line No") and len(r) > k_ex and r[0].isdigit():
            s = _i(r[k_all])
            total += s
            reasons = Counter({c[6:]: _i(r[i]) for i, c in stall_cols if i < len(r)})
            lines.append((s, int(r[0]), (fname[:10] + ' ' + r[1].strip())[:70], _i(r[k_ex]), reasons))
    print("total samples", total)
    for s, ln, src, ex, reasons in sorted(lines, reverse=True)[:top]:
        rs = " ".join(f"{k}:{v}" for k, v in reasons.most_common(2) if v)
        print(f"{100 * s / max(total, 1):5.1f}% L{ln:<4d} {src:70s} ex={ex:<9d} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

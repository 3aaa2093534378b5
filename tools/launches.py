"""Summarise an ncu --csv launch list: per-launch time, DRAM bytes, share of total."""
import collections
import csv
import io
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        key = (int(r["ID"]), r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")[:48], r["Grid Size"], r["Block Size"])
        agg.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return agg


def main(path):
    agg = load(path)
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in agg.values())
    bykern = collections.Counter()
    for (i, k, g, b), d in agg.items():
        t = d.get("gpu__time_duration.sum", 0)
        bykern[k] += t
        print(f"{i:>4} {k:48s} grid{g:>14s} blk{b:>12s} {t / 1e3:9.1f}us {100 * t / tot:5.1f}%  "
              f"rd {d.get('dram__bytes_read.sum', 0) / 1e6:8.1f}MB wr {d.get('dram__bytes_write.sum', 0) / 1e6:8.1f}MB")
    print(f"total {tot / 1e3:.1f} us over {len(agg)} launches")
    for k, t in bykern.most_common():
        print(f"  {k:48s} {t / 1e3:9.1f}us {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])

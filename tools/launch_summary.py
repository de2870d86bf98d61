"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by
kernel: launches, total and mean time, share of the total."""
import csv
import sys
from collections import OrderedDict


def main(path, only_ours=True):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        if only_ours and ("at::" in name or "native" in name):
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + v)
    tot = sum(t for _, t in agg.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:8d} {t:10.1f} {t / n:9.2f} {t / tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1])

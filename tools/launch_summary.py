"""Per-kernel share of an ncu launch list (`--metrics gpu__time_duration.sum --csv`)."""
import collections
import csv
import sys


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:60]:60s} {n:8d} {t / 1e3:10.1f} {t / 1e3 / n:9.2f} {t / tot * 100:5.1f}%")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        print(summarise(p))

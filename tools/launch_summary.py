"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarise(path, top=25, by_grid=False):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[ui]]
        name = r[ki].split("(")[0][:52]
        if by_grid:
            name = f"{name} {r[h.index('Grid Size')]}"[:70]
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"{'kernel':70s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>8s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        lines.append(f"{k:70s} {cnt[k]:8d} {v / 1e3:9.3f} {100 * v / T:5.1f}% {v / cnt[k]:8.2f}")
    lines.append(f"total {T / 1e3:.3f} ms over {sum(cnt.values())} launches "
                 "(ncu-serialised, cold-cache: compare shares, not absolutes)")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarise(sys.argv[1], top=40 if "--by-grid" in sys.argv else 25,
                    by_grid="--by-grid" in sys.argv))

"""Critical-path share per kernel from a torch.profiler chrome trace of a
PDL-chained run: kernel i is charged end_i - max(start_i, end_{i-1}) (the
time the stream advanced because of it), so early-launched kernels waiting
in griddepcontrol.wait are not double counted.

    python tools/trace_exclusive.py gpurun_out/trace.json [--by-seq]
"""
import collections
import json
import sys


def main(path, by_seq=False):
    ev = json.load(open(path))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = [e for e in ev if e.get("cat") == "kernel" and e.get("ph") == "X"]
    ks.sort(key=lambda e: e["ts"])
    tot, cnt = collections.defaultdict(float), collections.Counter()
    prev_end = None
    seq = []
    for e in ks:
        s, d = e["ts"], e["dur"]
        end = s + d
        ex = end - (max(s, prev_end) if prev_end is not None else s)
        name = e["name"].split("(")[0][:58]
        g = e.get("args", {}).get("grid", "")
        key = f"{name} {g}" if by_seq else name
        tot[key] += max(ex, 0.0)
        cnt[key] += 1
        seq.append((name, g, round(ex, 2), round(d, 2)))
        prev_end = end if prev_end is None else max(prev_end, end)
    span = ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]
    T = sum(tot.values())
    print(f"span {span / 1e3:.3f} ms, charged {T / 1e3:.3f} ms over {len(ks)} kernels")
    print(f"{'kernel':72s} {'n':>6s} {'excl_us':>9s} {'share':>6s} {'avg_us':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:40]:
        print(f"{k:72s} {cnt[k]:6d} {v:9.1f} {100 * v / T:5.1f}% {v / cnt[k]:7.2f}")


if __name__ == "__main__":
    main(sys.argv[1], "--by-seq" in sys.argv)

"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel total device time, launches and share of the profiled window."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        out.append((r[ki], v * scale))
    return out


def summarize(path, top=40):
    data = load(path)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for name, us in data:
        key = name.split("(")[0].replace("void ", "")[:70]
        tot[key] += us
        cnt[key] += 1
    allt = sum(tot.values())
    print(f"{len(data)} launches, {allt:.1f} us total (ncu: serialized, cold-ish caches)")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{v:9.1f} us {100 * v / allt:5.1f}% {cnt[k]:4d}x  {k}")


if __name__ == "__main__":
    summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

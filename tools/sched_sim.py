"""Offline: makespan of the tensor-core conv's static work-item schedules on
the measured per-tile active-offset counts (gpurun_out/tile_costs.npz from
tools/tile_costs.py).  Cost model from tools/cta_probe.py: per CTA 2 us,
per item 1 us, per stage 0.45 us."""
import heapq
import sys

import numpy as np

d = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tile_costs.npz")


def stages(act, kd):
    return np.ceil(act / 2) if kd == 32 else act * (kd // 64)


def makespan(cost, order_of):
    G = 296
    n = len(cost)
    load = np.full(G, 2.0)
    for b in range(G):
        for w in order_of(b, G, n):
            load[b] += 1.0 + 0.45 * cost[w]
    return load.max()


def rr(b, G, n):
    return list(range(b, n, G))


def rev(b, G, n):
    return [n - 1 - w for w in range(b, n, G)]


def rev_snake(b, G, n):
    out, i = [], 0
    while True:
        w = i * G + (b if i % 2 == 0 else G - 1 - b)
        if i * G >= n:
            break
        if w < n:
            out.append(n - 1 - w)
        i += 1
    return out


def dyn(cost, desc):
    G = 296
    idx = np.argsort(-cost, kind="stable") if desc else np.arange(len(cost))
    h = [(2.0, b) for b in range(G)]
    for w in idx:
        t, b = heapq.heappop(h)
        heapq.heappush(h, (t + 1.0 + 0.45 * cost[w], b))
    return max(t for t, _ in h)


tot = {k: 0.0 for k in ("rr", "rev", "rev_snake", "dyn_asc", "dyn_lpt", "ideal")}
for k in d.files:
    if k.endswith(".kd"):
        continue
    kd = int(d[k + ".kd"][0])
    c = stages(d[k].astype(float), kd)
    if len(c) < 296:
        continue
    r = {"rr": makespan(c, rr), "rev": makespan(c, rev), "rev_snake": makespan(c, rev_snake),
         "dyn_asc": dyn(c, False), "dyn_lpt": dyn(c, True),
         "ideal": 2.0 + (len(c) + 0.45 * c.sum()) / 296}
    for kk in r:
        tot[kk] += r[kk]
    print(f"{k:16s} tiles {len(c):4d} " + " ".join(f"{kk} {v:5.1f}" for kk, v in r.items()))
print("total", " ".join(f"{kk} {v:6.1f}" for kk, v in tot.items()))

print("static schedules over tiles sorted by descending cost (the grouping's tile order):")
tot2 = {"rr": 0.0, "snake": 0.0, "dyn_lpt": 0.0}
for k in d.files:
    if k.endswith(".kd"):
        continue
    kd = int(d[k + ".kd"][0])
    c = stages(d[k].astype(float), kd)
    if len(c) < 296:
        continue
    cs = np.concatenate([np.sort(c[:-1])[::-1], c[-1:]])  # ragged last tile stays last

    def snake(b, G, n):
        out, i = [], 0
        while i * G < n:
            w = i * G + (b if i % 2 == 0 else G - 1 - b)
            if w < n:
                out.append(w)
            i += 1
        return out

    r = {"rr": makespan(cs, rr), "snake": makespan(cs, snake), "dyn_lpt": dyn(c, True)}
    for kk in r:
        tot2[kk] += r[kk]
    print(f"{k:16s} " + " ".join(f"{kk} {v:5.1f}" for kk, v in r.items()))
print("total", " ".join(f"{kk} {v:6.1f}" for kk, v in tot2.items()))

"""CPU stand-in for a SparseResNet stage engine (test helper for
tests/test_pipeline.py): same boundary buffers and entry points as
model.SparseResNetTrainer restricted to a unit range, with scalar-affine
units so the pipeline runtime's transport, schedule, weight stashing and
replica reduction can be exercised on CPU with the gloo backend.

Unit u: x <- w_u * x + 1 (every channel); the last stage's loss is
sum(x[:n]) / (n * C).  Coordinates pass through unchanged (one level), the
row count n is data dependent, labels ride along."""
import types

import torch

CAP, C, B = 40, 3, 4


class FakeParams:
    def __init__(self, n):
        self.p = torch.zeros(n, dtype=torch.float64)
        self.pb = torch.zeros(n, dtype=torch.float64)
        self.g = torch.zeros(n, dtype=torch.float64)
        self.size = n


class FakeEngine:
    def __init__(self, units, n_units, init_w, lr=0.05, momentum=0.9):
        u0, u1 = units
        self.u0, self.u1 = u0, u1
        self.first, self.last = u0 == 0, u1 == n_units - 1
        self.entry_level = self.exit_level = 0
        lv = types.SimpleNamespace(coords=torch.zeros((CAP, 4), dtype=torch.int32),
                                   n=torch.zeros(1, dtype=torch.int32), cap=CAP)
        self.levels = [lv]
        self.params = FakeParams(u1 - u0 + 1)
        self.params.p.copy_(torch.tensor(init_w[u0:u1 + 1], dtype=torch.float64))
        self.params.pb.copy_(self.params.p)
        self.x_in = torch.zeros((CAP, C), dtype=torch.float64)
        self.g_out_ext = torch.zeros((CAP, C), dtype=torch.float64)
        self.labels = torch.zeros(B, dtype=torch.int32)
        self.loss = torch.zeros(1, dtype=torch.float64)
        self.lr, self.momentum = lr, momentum
        self.grad_input = None
        self.out_act = torch.zeros((CAP, C), dtype=torch.float64)
        self._pts = None

    def set_batch(self, pts, lab):
        self._pts = pts
        self.labels.copy_(lab)

    def forward_body(self):
        lv = self.levels[0]
        if self.first:  # "voxelize": rows = points, n from the batch
            n = int(self._pts.shape[0])
            lv.n.fill_(n)
            lv.coords.zero_()
            lv.coords[:n, 0] = torch.arange(n, dtype=torch.int32) % B
            x = torch.zeros((CAP, C), dtype=torch.float64)
            x[:n] = self._pts
        else:
            x = self.x_in.clone()
        n = int(lv.n.item())
        self.acts = []
        for w in self.params.pb:
            self.acts.append(x.clone())
            x = w * x + 1.0
            x[n:] = 0.0
        self.out_act.copy_(x)
        if self.last:
            self.loss.fill_(float(x[:n].sum()) / (n * C))

    def backward_body(self):
        n = int(self.levels[0].n.item())
        if self.last:
            g = torch.zeros((CAP, C), dtype=torch.float64)
            g[:n] = 1.0 / (n * C)
        else:
            g = self.g_out_ext.clone()
        for i in reversed(range(len(self.acts))):
            self.params.g[i] = float((g[:n] * self.acts[i][:n]).sum())
            g = g * self.params.pb[i]
        self.grad_input = g

    def sgd_into(self, p, m, pb):
        m.mul_(self.momentum).add_(self.params.g)
        p.sub_(self.lr * m)
        pb.copy_(p)


def init_weights(n_units):
    return [1.0 + 0.1 * (u + 1) for u in range(n_units)]


def batch_of(mb):
    g = torch.Generator().manual_seed(1000 + mb)
    n = 20 + mb % 7
    pts = torch.randn((n, C), generator=g, dtype=torch.float64)
    lab = torch.arange(B, dtype=torch.int32) + mb
    return pts, lab


def make_factory(n_units):
    w = init_weights(n_units)
    return lambda units: FakeEngine(units, n_units, w)

"""Debug helper (GPU): per-layer relative errors of the trainer vs the
bf16-emulating oracle. Not collected by pytest (no test_ prefix)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np, torch
import voxpipe_oracle as O
from paper_2012_13846_b200 import model

def bf(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)

B, P, res = 4, 1500, 48
tr = model.SparseResNetTrainer(batch=B, points=P, resolution=res, seed=2)
pts, offs = O.synthetic_batch(B, P, res, seed=3, dtype=np.float32)
labels = (np.arange(B) * 7) % 40
p0 = tr.state_numpy()
loss = tr.train_step_from_host(pts, offs, labels)
c, f = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, res)
pr = {k: (bf(v) if k.endswith(".w") and not k.startswith("fc") else v) for k, v in p0.items()}
trace = {}
rloss, rg, _, _ = O.resnet_train_step(pr, c, f, labels, B, wdtype=bf, act_round=bf, trace=trace)
print("loss", loss, rloss)
def rel(a, b):
    return np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30)
g = tr.grads_numpy()
for L in tr.layers:
    n = int(L["dst"].n.item())
    nm = L["name"]
    y = L["y"][:n].float().cpu().numpy()
    gy = L["gy"][:n].float().cpu().numpy()
    print(f"{nm:12s} n={n:6d} y {rel(y, trace[nm+'.y']):.2e} mean {rel(L['mean'].cpu().numpy(), trace[nm+'.mean']):.2e} "
          f"rstd {rel(L['rstd'].cpu().numpy(), trace[nm+'.rstd']):.2e} gy {rel(gy, trace[nm+'.gy']):.2e} "
          f"gw {rel(g[nm+'.w'], rg[nm+'.w']):.2e} ggam {rel(g[nm+'.gamma'], rg[nm+'.gamma']):.2e}")

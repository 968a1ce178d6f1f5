"""Diagnostic: bf16 training-step error of the engine against the
bf16-emulating f64 oracle (loss, per-parameter gradient rel-L2 / cosine), as
the bench builds the trainer (prefetch + captured graphs), at a given config.
Prints one JSON line per config; used to set the tolerances written in
tests/test_gpu_bench_parity.py.  Test/diagnostic infrastructure only.

  python tools/parity_probe.py 64 2048 64      # C3
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import voxpipe_oracle as O  # noqa: E402
from paper_2012_13846_b200 import model  # noqa: E402


def bf16_round(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)


def engine_first_step(B, P, res, blocks, pts, labels):
    tr = model.SparseResNetTrainer(batch=B, points=P, resolution=res, blocks=blocks)
    p_init = tr.params.p.clone()
    tr.enable_prefetch()
    dp = torch.from_numpy(pts).cuda()
    dl = torch.from_numpy(labels.astype(np.int32)).cuda()
    tr.set_batch(dp, dl)
    tr.capture(warmup=1)
    tr.params.p.copy_(p_init)
    tr.params.m.zero_()
    tr.params.g.zero_()
    tr.params.pb[: tr.params.n_bf16].copy_(tr.params.p[: tr.params.n_bf16].to(torch.bfloat16))
    tr.prime(dp, dl)
    tr.set_batch(dp, dl)
    p0 = tr.state_numpy()
    tr.step()
    torch.cuda.synchronize()
    return tr, p0, float(tr.loss.item()), tr.grads_numpy()


def main():
    B, P, res = (int(v) for v in sys.argv[1:4])
    blocks = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    pts, offs = O.synthetic_batch(B, P, res, seed=0, dtype=np.float32)
    labels = (np.arange(B) * 7) % 40
    tr, p0, loss, g = engine_first_step(B, P, res, blocks, pts, labels)
    c, f = O.voxelize_batch(pts.astype(np.float64), offs, 1.0, res)
    pr = {k: (bf16_round(v) if k.endswith(".w") and not k.startswith("fc") else v) for k, v in p0.items()}
    t0 = time.time()
    rloss, rg, _, _ = O.resnet_train_step(pr, c, f, labels, B, blocks=blocks, wdtype=bf16_round,
                                          act_round=bf16_round)
    out = {"config": [B, P, res, blocks], "rows": len(c), "loss": loss, "ref_loss": rloss,
           "loss_rel": abs(loss - rloss) / abs(rloss), "oracle_s": round(time.time() - t0, 1), "grads": {}}
    for k, r in rg.items():
        e = np.linalg.norm(g[k] - r) / (np.linalg.norm(r) + 1e-30)
        cs = float((g[k] * r).sum() / (np.linalg.norm(g[k]) * np.linalg.norm(r) + 1e-30))
        out["grads"][k] = [round(float(e), 5), round(cs, 6)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

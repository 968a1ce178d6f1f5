"""SparsePipe pipeline on the GPU with the real stage engines (one process,
LocalPipeline driving the same per-rank 1F1B programs the multi-GPU runtime
runs): a pipelined run equals an emulation of PipeDream's stashed-weight
semantics on the single-GPU full-model engine — micro-batch i runs with stage
s's master weights at the version the schedule gives it, and each stage
applies its gradients in micro-batch order through the same SGD kernel.

fp32 engines (SIMT kernels, deterministic): losses and final weights agree to
1e-6 relative (the stage boundary moves tensors bit-exactly; only the
identity-branch gradient sum at a cut is re-associated).  bf16 engines
(tcgen05 path): loss rel 2e-3."""
import numpy as np
import pytest

import voxpipe_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

B, PTS, RES = 3, 1200, 32


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def batch_of_factory():
    cache = {}

    def batch_of(mb):
        if mb not in cache:
            pts, _ = O.synthetic_batch(B, PTS, RES, seed=50 + mb, dtype=np.float32)
            lab = torch.tensor([(mb * 5 + 3 * b) % 40 for b in range(B)], dtype=torch.int32)
            cache[mb] = (torch.from_numpy(pts).cuda(), lab.cuda())
        return cache[mb]

    return batch_of


def factory(dtype):
    from paper_2012_13846_b200 import model

    def make(units):
        return model.SparseResNetTrainer(batch=B, points=PTS, resolution=RES, seed=2, feature_dtype=dtype,
                                         units=units, lr=0.05)
    return make


def emulate(topo, M, dtype):
    """Reference semantics on the full-model engine (see module docstring)."""
    from paper_2012_13846_b200 import pipeline as PL

    make = factory(dtype)
    full = make(None)
    stages = [make((st.unit_start, st.unit_end)) for st in topo.stages]
    fpb = full.params
    ver = {(mb, s): fv for mb, s, fv, _ in PL.simulate_versions(topo, M)}
    hist = [[e.params.p.clone()] for e in stages]
    mom = [torch.zeros_like(e.params.p) for e in stages]
    shadow = [e.params.pb.clone() for e in stages]
    batch_of = batch_of_factory()
    losses = {}
    for i in range(M):
        for s, e in enumerate(stages):
            src = hist[s][ver[(i, s)]]
            for name in e.params.offsets:
                fpb.view(fpb.p, name).copy_(e.params.view(src, name))
        fpb.pb[: fpb.n_bf16].copy_(fpb.p[: fpb.n_bf16].to(torch.bfloat16))
        pts, lab = batch_of(i)
        full.set_batch(pts, lab)
        full.forward_body()
        full.backward_body()
        losses[i] = float(full.loss.item())
        for s, e in enumerate(stages):
            for name in e.params.offsets:
                e.params.view(e.params.g, name).copy_(fpb.view(fpb.g, name))
            p = hist[s][-1].clone()
            e.sgd_into(p, mom[s], shadow[s])
            hist[s].append(p)
    return losses, [h[-1] for h in hist]


@pytest.mark.parametrize("cuts", [[3], [1, 4, 6]])
def test_pipeline_equals_emulation_fp32(cuts):
    from paper_2012_13846_b200 import pipeline as PL

    M = 6
    n_units = len(factory(torch.float32)(None).units)
    topo = PL.Topology.even(n_units, cuts)
    pl = PL.LocalPipeline(topo, M, factory(torch.float32), batch_of_factory())
    stats = pl.run()
    ref_loss, ref_w = emulate(topo, M, torch.float32)
    last = topo.stages[-1].ranks[0]
    got = [float(stats[last].losses[i].item()) for i in range(M)]
    np.testing.assert_allclose(got, [ref_loss[i] for i in range(M)], rtol=1e-6)
    for s, st in enumerate(topo.stages):
        run = pl.runners[st.ranks[0]]
        assert all(fv == bv for _, _, fv, bv in run.stats.audit)
        np.testing.assert_allclose(run.master_p.cpu().numpy(), ref_w[s].cpu().numpy(), rtol=1e-5, atol=1e-6)


def test_pipeline_bf16_graphs_and_replicas():
    """bf16 tcgen05 engines under CUDA-graph replay: a 2-stage pipeline
    matches the emulation's losses; a replicated first stage ("2-1") keeps
    its replicas' weights identical."""
    from paper_2012_13846_b200 import pipeline as PL

    M = 4
    n_units = len(factory(torch.bfloat16)(None).units)
    topo = PL.Topology.even(n_units, [4])
    pl = PL.LocalPipeline(topo, M, factory(torch.bfloat16), batch_of_factory(), use_graphs=True)
    stats = pl.run()
    ref_loss, _ = emulate(topo, M, torch.bfloat16)
    got = [float(stats[1].losses[i].item()) for i in range(M)]
    np.testing.assert_allclose(got, [ref_loss[i] for i in range(M)], rtol=2e-3)
    topo2 = PL.Topology.even(n_units, [4], [2, 1])
    pl2 = PL.LocalPipeline(topo2, M, factory(torch.bfloat16), batch_of_factory())
    pl2.run()
    assert torch.equal(pl2.runners[0].master_p, pl2.runners[1].master_p)


@pytest.mark.parametrize("n,plan", [(2, "4"), (3, "2,5")])
def test_multiprocess_pipeline_bench_on_one_gpu(n, plan):
    """The multi-process SparsePipe runtime end to end (torchrun, one process
    per stage, StageRunner + DistTransport, bench.py's run_pipeline) with
    every rank on cuda:0 and gloo moving the stage tensors through host
    memory — NCCL cannot host two ranks on one device, so this is the
    functional check of the multi-GPU path available on one B200."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1", f"--nproc-per-node={n}",
           os.path.join(root, "bench.py"), "--gpus", str(n), "--plan", plan, "--pipeline-test", "--steps", "2",
           "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["value"] > 0
    assert len(d["config"]["stages"]) == n
    audit = d["weight_version_audit"]
    assert audit["checked"] == 2 * n * n and audit["violations"] == 0  # steps * world micro-batches x stages

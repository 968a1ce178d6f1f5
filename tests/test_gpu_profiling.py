"""The per-layer measurement harness: conv.benchmark_forward_backward
(reference conv.py:280-320) and profiling.run_benchmark_profile (reference
profiling.py:333-455) on the GPU.  The size fields of every record (kernel-map
pairs, activation bytes of the serialized output, parameter bytes) equal the
reference's own records on the same inputs; times are device µs > 0."""
import numpy as np
import pytest

import voxpipe_oracle as O
from parity_util import reference

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    mods = reference()
    if mods is None:
        pytest.skip("oracle/_ref not built")
    return mods


@pytest.mark.parametrize("stride", [1, 2])
def test_benchmark_forward_backward_record(ref, stride):
    R, RT = ref
    from paper_2012_13846_b200 import conv
    from paper_2012_13846_b200.tensor import SparseTensor
    pts, offs = O.synthetic_batch(2, 600, 24, seed=4, dtype=np.float64)
    coords, _ = O.voxelize_batch(pts, offs, 1.0, 24)
    rng = np.random.default_rng(0)
    x = rng.normal(size=(len(coords), 16))
    w = rng.normal(size=(27, 32, 16)) / np.sqrt(27 * 16)
    got = conv.benchmark_forward_backward(SparseTensor(coords, x, (1, 1, 1)), conv.ConvWeights(w),
                                          conv.KernelShape.hypercubic(3, 3), stride, 1, 3)
    exp = R.benchmark_forward_backward(R.SparseTensor(coords, x, (1, 1, 1)), R.ConvWeights(w),
                                       R.KernelShape.hypercubic(3, 3), stride, 0, 1)
    assert set(got) == set(exp)
    for k in ("kernel_map_pairs", "activation_bytes", "param_bytes"):
        assert got[k] == exp[k], k
    assert got["fwd_time_us"] > 0 and got["bwd_time_us"] > 0
    # the device path is orders of magnitude below the reference's CPU wall time
    assert got["fwd_time_us"] < exp["fwd_time_us"]


def test_run_benchmark_profile_matches_reference_sizes(ref):
    R, RT = ref
    import importlib
    import sys
    from paper_2012_13846_b200 import profiling
    RP = importlib.import_module("voxpipe.profiling")
    assert "voxpipe" in sys.modules
    desc = {"input": {"seed": 3, "dim": 3, "resolution": 20, "num_points": 3000, "feature_width": 1},
            "layers": [{"type": "sparse_conv", "out_channels": 32, "stride": 1},
                       {"type": "sparse_conv", "out_channels": 64, "stride": 2},
                       {"type": "synthetic", "fwd_time_us": 5.0, "bwd_time_us": 9.0, "activation_bytes": 10,
                        "param_bytes": 20},
                       {"type": "sparse_conv", "out_channels": 64, "stride": 1}]}
    got = profiling.run_benchmark_profile(desc, "B200", 1, 2)
    exp = RP.run_benchmark_profile(desc, "cpu", 0, 1)
    assert len(got) == len(exp) == 4
    for g, e in zip(got, exp):
        assert g.layer_id == e.layer_id
        assert g.activation_bytes == e.activation_bytes and g.param_bytes == e.param_bytes
        assert g.fwd_time_us > 0 and g.bwd_time_us > 0
    assert got[2].fwd_time_us == 5.0 and got[2].bwd_time_us == 9.0

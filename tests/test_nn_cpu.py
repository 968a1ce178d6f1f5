"""Host-side checks of the PyTorch drop-in (no GPU): module construction,
the reference weight layout (K, n_out, n_in) and its initialisation scale."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")


def test_module_layout_and_init():
    from paper_2012_13846_b200 import nn
    g = torch.Generator().manual_seed(0)
    m = nn.SparseConv3d(16, 32, kernel_size=3, stride=2, generator=g)
    assert tuple(m.weight.shape) == (27, 32, 16)  # conv.py:77-105 layout
    std = float(m.weight.detach().double().std())
    assert abs(std - 1 / np.sqrt(27 * 16)) < 0.1 / np.sqrt(27 * 16)
    assert "stride=2" in repr(m)
    t = nn.SparseConvTranspose3d(8, 4, kernel_size=(3, 1, 3))
    assert t.shape.num_offsets == 9 and tuple(t.weight.shape) == (9, 4, 8)
    bn = nn.SparseBatchNorm(32, relu=True)
    assert float(bn.weight.sum()) == 32 and float(bn.bias.abs().sum()) == 0


def test_ops_need_the_cuda_library_and_device():
    """No CPU fallback: without a device the op raises instead of computing."""
    from paper_2012_13846_b200 import errors, nn, tensor
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    with pytest.raises((errors.ConfigError, RuntimeError)):
        tensor.SparseTensor(np.zeros((1, 4), np.int64), np.zeros((1, 2)), (1, 1, 1))
    del nn

"""paper_2012_13846_b200 — B200-native (sm_100a) drop-in for the sparse
convolution hot path of voxpipe 0.1.0 / SparsePipe (arXiv 2012.13846).

Public API mirrors the reference modules:
  tensor  : SparseTensor, PointCloud, voxelize, voxelize_batch, dropout, batch,
            split_batches, to/from_json, to/from_binary     (voxpipe/tensor.py)
  kernels : build_table, lookup, pack_rows, CoordIndex, coord_index
            (the VOXPIPE_BACKEND seam, voxpipe/kernels.py)
  conv    : KernelShape, ConvWeights, KernelMap, generate_output_coords,
            build_kernel_map, sparse_conv_forward, sparse_conv_backward,
            sparse_conv_transposed, benchmark_forward_backward, weight I/O
            (voxpipe/conv.py)
  model   : SparseResNet trainer (graph-capturable training step)
All compute goes through libvoxpipe_b200.so (include/voxpipe_b200.h).
"""
from . import errors  # noqa: F401
from ._lib import LIB_PATH, load  # noqa: F401

__version__ = "0.1.0"

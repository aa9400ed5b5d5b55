"""B200-native (sm_100a) rotation-invariant scatter convolution (arXiv 2512.08888).

The hot path is the fused RI-conv layer forward behind the C-ABI in
include/rotconv_c.h (librotconv_b200.so); ``rotconv`` mirrors the reference's
operator names over it, ``distributed`` shards the batch across GPUs.
"""
from . import rotconv  # noqa: F401
from .rotconv import (  # noqa: F401
    AuxMemCounter, Desc, GroupSpec, MultCounter, RIConv, ScatterStrategy, SteerableBasis,
    TileConfig, bank_bases, bank_precompute, build_orientation_bank, clipped_writes,
    group_conv_scatter_reuse, orientation_pool_avg, orientation_pool_max, ri_conv,
    ri_conv_forward, scatter_conv_multi, scatter_conv_raw_multi, scatter_conv_single,
    shard_range, steer, subgroup_pool_max, tiled_scatter_conv, transform_kernel,
    gaussian_derivative_basis, loss_mag, loss_orth, total_loss, ri_conv_backward, RIConvFunction)

__all__ = [n for n in dir() if not n.startswith("_")]

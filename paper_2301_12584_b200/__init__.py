"""paper_2301_12584_b200 — B200-native exact KRP leverage-score sampler.

The hot path of arXiv 2301.12584 (segment-tree construction, batched
root-to-leaf descent, updates, exclude-one sampling, STS-CP gather) as
hand-written sm_100a CUDA behind the C ABI in include/krpg.h, with a Python
mirror of the reference's KrpSampler API for tests and benchmarks.
"""
from ._lib import (EXCLUDED, KrpgCudaError, KrpgError, KrpgInvalidArgument, build, lib)
from .sampler import ConditionalDistribution, KrpSampler, RowOrder, SampleBatch, device_count, product_lev_sample
from .segtree import SegmentTreeSampler
from .tensor import SparseTensor

__all__ = [
    "EXCLUDED", "KrpgCudaError", "KrpgError", "KrpgInvalidArgument", "build", "lib",
    "ConditionalDistribution", "KrpSampler", "RowOrder", "SampleBatch", "device_count",
    "SparseTensor", "SegmentTreeSampler", "product_lev_sample",
]

"""paper_1803_11385_b200 — B200-native H-CNN hash-conv hot path.

hash2col / col2hash / conv contraction / hash max-pool and unpool on batched
perfect-spatial-hash (super-PSH) tables, as hand-written sm_100a CUDA behind the
C ABI in include/hashconv_b200.h (libhcb200.so). See DESIGN.md.
"""
from ._lib import LIB_PATH, HashConvCudaError  # noqa: F401  (fails loudly if the library is missing)
from .psh import (PshLevel, SuperPsh, VoxelSet, build_pyramid, mix_seed, read_psh_file,  # noqa: F401
                  write_psh_file)

__all__ = ["LIB_PATH", "HashConvCudaError", "PshLevel", "SuperPsh", "VoxelSet", "build_pyramid", "mix_seed",
           "read_psh_file", "write_psh_file"]

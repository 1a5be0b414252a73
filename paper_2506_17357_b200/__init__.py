"""B200-native (sm_100a) full-neighbourhood VRP move evaluation (arXiv 2506.17357, TGA).

The hot path (attribute-rebuild scan, per-operator tile evaluation with fused
argmin, incremental update) is hand-written CUDA in ``csrc/`` behind the C ABI
``include/tga.h``; ``tga`` is its ctypes binding.
"""
from . import tga  # noqa: F401
from .tga import (Instance, Solution, Move, TgaError, OP_ALL, OP_INTER, OP_INTRA,  # noqa: F401
                  OP_FUSED_NS, OPERATORS, VARIANT_NAMES, N_VARIANTS, decode_key)

__all__ = ["tga", "Instance", "Solution", "Move", "TgaError", "OP_ALL", "OP_INTER", "OP_INTRA",
           "OP_FUSED_NS", "OPERATORS", "VARIANT_NAMES", "N_VARIANTS", "decode_key"]

"""B200-native TAPER hot path (arXiv 2605.06914): per-step branch admission and cascade
branch-decode attention as a C-ABI CUDA library (libtaper.so) with a thin binding.

``from paper_2605_06914_b200 import taper`` loads the library (and fails loudly if it is
not built -- there is no fallback)."""
__all__ = ["taper"]

"""paper_2405_19056_b200 -- B200-native GlassNet inference forward pass (arXiv 2405.19056).

The product is libglassnet.so (csrc/, C ABI in include/glassnet.h); this package is
its thin ctypes binding.  See DESIGN.md.
"""
from .glassnet import (BF16, FP32, Comm, Dims, GlassNet, GlassNetError, get_unique_id, lib, make_dims,  # noqa
                       tile_rows, weight_count)

__all__ = ["GlassNet", "Dims", "make_dims", "weight_count", "tile_rows", "get_unique_id", "Comm",
           "GlassNetError", "lib", "BF16", "FP32"]

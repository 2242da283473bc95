"""B200-native (sm_100a) hot path of the basic blocked polynomial codec of
arXiv 1805.01844 (Sec. 3.1 Eq. 1-2, Sec. 3.3) with 64-bit words.

The product is the C-ABI library libpolycomp.so (include/poly.h); this package
holds its CUDA sources (csrc/), the in-tree build (_build.py) and the ctypes
binding (polycomp.py).  It never imports oracle/.
"""
from .polycomp import (  # noqa: F401
    POLY_U16, POLY_U32, PolyError, compress, decompress, load_library, poly_compress,
    poly_compress_host, poly_decompress, poly_decompress_host, poly_init, poly_launches_per_call,
    poly_max_compressed_bytes, poly_read_header, poly_version, poly_workspace_bytes,
)

"""B200-native SCM engine for MC-PDIPM (arXiv 1310.6919): Python binding of libsdpc.

The compute path is the CUDA library libsdpc.so (csrc/, sm_100a).  This package is
argument marshalling only; it never imports the oracle and has no CPU fallback.
"""
from .sdpc import Handle, SdpcError, fp64_peak, lib, SYMBOLS, LIB_PATH  # noqa: F401

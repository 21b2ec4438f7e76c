"""B200 (sm_100a) hot path of the local character-based method for sparse linear
solves (Ye, An, Xu, arXiv 2001.01158).  The compute lives in liblc.so (C ABI,
include/lc.h); ``lc`` is the thin Python binding."""
from . import lc  # noqa: F401

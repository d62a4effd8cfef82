"""paper_2308_14258_b200 — B200-native distributed Mosaic Flow Predictor (arXiv 2308.14258).

The product is ``libmfp.so`` (C ABI in ``include/mfp.h``, sm_100a kernels + NCCL);
``mfp`` is its thin ctypes binding.  Importing fails loudly when the library is
not built — there is no CPU fallback.
"""
from .mfp import *  # noqa: F401,F403
from .mfp import EXPORTS, LIB_PATH, Mfp, MfpError  # noqa: F401

"""paper_2512_02278_b200 -- B200-native batched graph search (Fantasy hot path).

The product is libdvsg.so (CUDA kernels for sm_100a + C++ host layer behind
the C-ABI in include/dvsg.h).  This package only binds it; see api.py for the
reference-shaped interface.
"""
from ._lib import EXPORTED, LIB_PATH, FormatError, InternalError, InvalidArgument  # noqa: F401
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all

__all__ = list(_api_all) + ["EXPORTED", "LIB_PATH"]

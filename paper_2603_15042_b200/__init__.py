"""B200-native GPU-coroutine runtime (DetShare, arXiv 2603.15042).

The product is the native library ``libdetshare.so`` (csrc/: sm_100a executor,
arbiter and tenant bodies + C++ host runtime) behind the C ABI in
``include/detshare/ds.h``.  This package is the Python view over that ABI.
"""
from . import _abi  # noqa: F401
from ._abi import DsError  # noqa: F401

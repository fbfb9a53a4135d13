"""B200-native (sm_100a) SE(2) traversability hot path of SEB-Naver (arXiv 2503.02412).

The product is ``libse2map.so`` (C ABI, ``include/se2map.h``); ``se2map`` is its thin
Python binding.  Import raises if the CUDA library has not been built: there is no CPU path.
"""
from . import se2map  # noqa: F401
from .se2map import Se2Map, default_params  # noqa: F401

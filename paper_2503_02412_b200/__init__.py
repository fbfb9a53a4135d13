"""B200-native (sm_100a) SE(2) traversability hot path of SEB-Naver (arXiv 2503.02412).

The product is ``libse2map.so`` (C ABI, ``include/se2map.h``); ``se2map`` is its thin
Python binding.  Importing ``se2map`` raises if the CUDA library has not been built: there is
no CPU path.  (The package itself imports nothing eagerly so that ``_build`` can run first.)
"""


def __getattr__(name):
    if name in ("Se2Map", "default_params", "Se2mError"):
        from . import se2map
        return getattr(se2map, name)
    raise AttributeError(name)

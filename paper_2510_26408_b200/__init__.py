"""paper_2510_26408_b200 — B200-native Linear-Optical Feynman Path sum (arXiv 2510.26408).

The product is ``liblofp.so`` (C ABI in ``include/lofp.h``: sm_100a kernels + C++ host
runtime); ``lofp.Circuit`` is its thin Python binding.
"""
from .lofp import Circuit, LofpError, LIB_PATH, EXPORTS  # noqa: F401

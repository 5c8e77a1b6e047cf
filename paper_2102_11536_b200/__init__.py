"""B200-native explicit order-2k generalized-alpha + IGA mass PCG (arXiv 2102.11536).

The product is libgenalpha.so (C ABI in include/genalpha.h, CUDA for sm_100a);
this package holds its sources (csrc/), the build script and the ctypes
binding.  There is no CPU fallback: importing the binding without the built
library raises ImportError.
"""
from .genalpha import *  # noqa: F401,F403
from .genalpha import Context, GAError, ga_params, ga_query, make_desc  # noqa: F401

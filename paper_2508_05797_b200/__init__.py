"""B200-native hashless content-defined chunking (PAPER.md, arxiv 2508.05797).

The product is libcdc_b200.so (include/cdc_b200.h); this package is its thin
Python binding.  It never imports the test oracle and has no CPU fallback.
"""
from .api import *  # noqa: F401,F403
from .api import __all__  # noqa: F401

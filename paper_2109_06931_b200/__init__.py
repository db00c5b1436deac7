"""B200-native GPU PC-sample attribution (HPCToolkit GPU analysis hot path, arXiv 2109.06931).

`gpa` is the Python binding of the C-ABI library libgpa.so (include/gpa.h); `parallel`
shards record streams over ranks and reduces the histograms (NCCL).  See DESIGN.md.
"""
from . import gpa  # noqa: F401  (raises ImportError if libgpa.so is not built)
from . import parallel  # noqa: F401

__all__ = ["gpa", "parallel"]

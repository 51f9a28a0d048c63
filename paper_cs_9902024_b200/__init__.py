"""B200-native batched unsteady DSMC (Bogdanov et al., arxiv/paper_cs_9902024).

The hot path -- Generation, Motion, Enumeration/Indexing (LCR), Interaction
(NTC), Sampling -- lives in the CUDA kernels of libdsmc.so behind the C ABI of
include/dsmc.h; `dsmc` is the ctypes binding.  Build with `build.build()`.
"""
from . import build  # noqa: F401

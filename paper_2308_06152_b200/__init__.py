"""B200-native (sm_100a) two-level deflation + CSLP preconditioned FGMRES for the 2D
Helmholtz equation (arXiv:2308.06152).  The compute path is libhelm.so (csrc/, C ABI in
include/helm.h); `helm` is its thin ctypes binding.  Nothing here imports oracle/."""
from . import build  # noqa: F401

"""B200-native P-SWA entropy-model decode (arXiv 2605.20977).

Host C++ + sm_100a CUDA behind the C ABI in ``include/pswa/pswa_cuda.h``;
this package is the thin Python mirror used by tests and ``bench.py``.
"""
from ._lib import lib, check, PswaCfg, PswaError  # noqa: F401

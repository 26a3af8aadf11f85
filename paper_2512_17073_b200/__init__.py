"""B200-native router-guided low-rank-compensated MoE expert path (arXiv 2512.17073).

Drop-in for the hot path of the reference package ``moe-lrc`` 0.1.0: the
modules ``quant``, ``lowrank`` and ``moe`` keep the reference's names and
semantics; all numerics run in hand-written sm_100a CUDA kernels behind the
C-ABI in ``include/lrc.h`` (``_lib/liblrc.so``).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from . import _lib  # noqa: F401

"""B200-native (sm_100a) DMAS / CF beamforming hot path of arXiv 2511.09165.

The compute runs in ``libdmas.so`` (hand-written CUDA kernels behind the C ABI of
``include/dmas.h``); ``dmas`` is the thin ctypes binding, ``parallel`` the one-process-per-GPU
direction sharding over ``torch.distributed``.  Importing ``dmas`` fails loudly when the shared
library is missing: there is no CPU fallback.
"""

__all__ = ["dmas", "parallel"]

"""B200-native MAPLE hot path (arXiv 2412.13576): parallel extraction of approximate Graver-basis
directions and multi-start Graver-best augmentation, as a C-ABI library (libmaple.so, include/maple.h)
with hand-written sm_100a kernels. `maple` is the thin ctypes binding; `distributed` shards starts across
GPUs with one torch.distributed all-gather feeding the global merge."""
from . import maple  # noqa: F401

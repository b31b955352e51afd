"""B200-native CacheBlend (arXiv 2405.16444) KV-cache blending hot path.

libcacheblend.so (C-ABI, include/cacheblend.h) holds every step as sm_100a CUDA kernels; this
package is the thin ctypes binding (`api`). Build the library with
`python -m paper_2405_16444_b200.build`."""
from . import api  # noqa: F401
from .api import (CacheBlendError, Context, Group, ModelWeights, blend_forward, blend_layer,  # noqa: F401
                  kv_deviation_topk, nccl_unique_id, rope_realign, schedule)

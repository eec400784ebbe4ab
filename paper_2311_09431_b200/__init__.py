"""B200-native striped / ring causal attention (arXiv 2311.09431) behind the ringsim API.

Product code only: hand-written sm_100a CUDA (``csrc/``) behind a C ABI
(``include/striped_attn.h``), bound with ctypes (``_lib.py``), driven by a torch host
layer (``ring.py`` / ``api.py``).  There is no CPU fallback.
"""

from .api import (  # noqa: F401
    StripedAttnFunction,
    ring_attention,
    striped_attention,
    striped_attn_backward,
    striped_attn_forward,
    stripe_permute,
    stripe_unpermute,
)
from .layout import Layout, PermutedBatch, Scheme, Shard  # noqa: F401
from .masks import (  # noqa: F401
    CAUSAL_EXCLUSIVE,
    CAUSAL_INCLUSIVE,
    FULLY_MASKED,
    FULLY_UNMASKED,
    MaskKind,
    TileClass,
    block_mask,
    classify_bounds,
    get_mask_ring,
    get_mask_striped,
    kernel_tile_census,
)

__version__ = "0.1.0"

"""B200-native InfiniGen decode-time KV path (arXiv 2406.19707).

Drop-in for the reference ``speckv`` operators on the path
(speculation / pool / attention_head / decode engine); every hot op is a
hand-written sm_100a kernel in libinfinigen_b200.so (C ABI:
include/infinigen_b200.h).  There is no CPU fallback: operators raise if the
library or a CUDA device is missing.
"""

__version__ = "0.1.0"

from ._lib import ArtifactConsistencyError, LIB_PATH  # noqa: F401
from .speculation import (  # noqa: F401
    HeadArtifacts, PartialArtifacts, SpeculationConfig, build_partial, select_tokens,
    selection_bytes, speculate_scores,
)
from .pool import COUNTER_MAX, EvictionPolicy, KvPool  # noqa: F401
from .attention import attention_head  # noqa: F401
from .model import Model, ModelSpec, load_model  # noqa: F401
from .engine import DecodeEngine, RunConfig, run  # noqa: F401

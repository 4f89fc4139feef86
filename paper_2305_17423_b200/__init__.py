"""B200-native sparse edit step (FISEdit, arXiv 2305.17423) with the sparsedit 0.1.0 API.

Drop-in for the reference package's public surface (sparsedit/__init__.py:9-60);
all compute runs in hand-written sm_100a kernels (libfisedit.so, C ABI in
include/fisedit.h). See DESIGN.md.
"""

from .cache import BufferPool, CacheKey, CacheStats, CacheStore, CompactTensor, Role, compact_tensor, materialize_payload
from .errors import CacheMissError, ConfigError, ContractViolation
from .masks import (BinaryMask, DiffMap, MaskPyramid, OtsuResult, accumulate_diff, build_pyramid,
                    centered_square_mask, dilate, mask_from_tensor, mask_to_tensor, otsu_threshold, save_mask_pgm)
from .model import UNetConfig
from .sparse import GatherPlan, SparseLayerContext, select_gather_plan
from .tensors import ConvWeights, LayerMacs, MacsReport, load_tensor, macs_attention, macs_conv, save_tensor
from .unet import (EditResult, EditSession, PromptTokens, SharedTokenMap, UNet, detect_mask, edit, edit_batch,
                   embed_tokens, generate_dense, generate_dense_batch, get_precision, initial_latent, set_precision)

__version__ = "0.1.0"

_LAZY_OPS = ("gather_blocks", "sparse_conv", "sparse_cross_attention", "sparse_group_norm", "sparse_self_attention",
             "attention", "conv2d", "group_norm", "normalize_with_group_stats")


def __getattr__(name):
    if name in _LAZY_OPS:
        from . import ops
        return getattr(ops, name)
    raise AttributeError(name)

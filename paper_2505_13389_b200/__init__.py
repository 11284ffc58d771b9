# SPDX-License-Identifier: Apache-2.0
"""B200-native VSA (Video Sparse Attention, arXiv 2505.13389) hot path.

The six sm_100a kernels live in ``csrc/`` behind the C ABI ``include/vsa_b200.h``;
``api`` mirrors the reference C++ API (``/root/reference/proj/include/vsa``).
"""
from ._lib import LIB_PATH, VsaError, build, lib  # noqa: F401
from .api import (  # noqa: F401
    POOL_MAX, POOL_MEAN, CoarseArtifacts, FineResult, TileLayout, VsaHostPipeline, VsaOp, VsaParams, all_cubes,
    coarse_backward,
    coarse_forward_select, coarse_from_pooled, fine_backward, fine_forward, flatten_index, gate_backward,
    gates_from_hidden, pool_cubes, selection_transpose, tile, tile_pool, untile, validate_selection,
    aggregate_probs_to_cubes, selection_accuracy, selection_accuracy_qk, VsaOutput, VsaGrads, vsa_forward,
    vsa_backward, GATE_IDENTITY, GATE_SIGMOID, MacCounter,
)
from .ulysses import UlyssesExchange, UlyssesVsa, transpose_blocks_cuda  # noqa: F401,E402

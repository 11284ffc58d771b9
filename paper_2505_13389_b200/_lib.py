# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C ABI in include/vsa_b200.h (libvsa_b200.so).

The shared library is built in-tree (``paper_2505_13389_b200/_lib``) by
``__graft_entry__.build()`` / ``make -C paper_2505_13389_b200/csrc``. There is
no fallback: if the library is missing, importing the kernels raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VSA_LIB_PATH") or os.path.join(_PKG, "_lib", "libvsa_b200.so")  # override: A/B tools
CSRC = os.path.join(_PKG, "csrc")

VSA_F32, VSA_BF16 = 0, 1
POOL_MEAN, POOL_MAX = 0, 1
PAD_REJECT, PAD_ZERO, PAD_MASK = 0, 1, 2
FINE_COMBINE, FINE_UNTILE, FINE_ADAPTATION, FINE_FORCE_SIMT = 1, 2, 4, 8
IO_HEAD_MAJOR, IO_SEQ_MAJOR = 0, 1


class vsa_layout_t(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("t", "h", "w", "ct", "ch", "cw", "tp", "hp", "wp", "nt", "nh", "nw",
                                         "cube", "seq", "seq_padded", "nc")] + [
        ("pad_mode", C.c_int32), ("io_order", C.c_int32), ("io_batch", C.c_int64), ("io_heads", C.c_int64),
        ("io_chunk", C.c_int64)]


class vsa_op_desc_t(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("batch", "heads", "head_dim", "top_k", "max_sel_k", "model_dim")] + [
        (n, C.c_int32) for n in ("dtype", "pool_mode", "activation", "adaptation", "raster", "flags", "coarse",
                                 "reserved")] + [("task_begin", C.c_int64), ("task_end", C.c_int64)]


class vsa_op_buffers_t(C.Structure):
    _fields_ = [("base", C.c_void_p), ("bytes", C.c_size_t)] + [
        (n, C.c_void_p) for n in ("q_t", "k_t", "v_t", "qc", "kc", "vc", "ac", "oc_cube", "sel", "selT_offs",
                                  "selT_idx", "o_fine", "lse", "dof", "delta", "doc_cube", "dqc", "dkc", "dvc",
                                  "gc", "gf", "dgc", "dgf", "fine_sel")] + [
        ("fine_k", C.c_int64), ("bwd_used_workspace", C.c_int32)]


OP_FORCE_SIMT, OP_NO_DS_WORKSPACE = 1, 2
COARSE_F32, COARSE_BF16 = 0, 1
OP_STAGES = ["tile_pool", "coarse_fwd", "fine_fwd", "prologue", "coarse_bwd", "fine_bwd"]

EXPORTS = [
    "vsa_last_error", "vsa_version", "vsa_kernel_launches", "vsa_debug_trace", "vsa_debug_tile_counter", "vsa_layout_make", "vsa_flatten_index", "vsa_tile", "vsa_untile",
    "vsa_tile_pool", "vsa_pool_tiled", "vsa_coarse_forward", "vsa_coarse_bitmap_bytes", "vsa_selection_transpose",
    "vsa_validate_selection", "vsa_fine_forward", "vsa_backward_prologue", "vsa_coarse_backward",
    "vsa_fine_backward", "vsa_fine_backward_workspace_bytes", "vsa_unpool_max_add", "vsa_layout_set_io",
    "vsa_transpose_blocks", "vsa_gate_forward", "vsa_gate_backward", "vsa_gate_backward_workspace_bytes",
    "vsa_selection_accuracy_from_lse", "vsa_aggregate_probs_to_cubes", "vsa_selection_accuracy",
    "vsa_op_memory_bytes", "vsa_op_create", "vsa_op_destroy", "vsa_op_buffers", "vsa_op_set_workspace",
    "vsa_op_workspace_bytes", "vsa_op_forward", "vsa_op_forward_coarse", "vsa_op_forward_fine", "vsa_op_backward",
    "vsa_forward", "vsa_backward", "vsa_op_timing", "vsa_op_stage_ms", "vsa_coarse_backward_tokens",
    "vsa_coarse_workspace_bytes", "vsa_coarse_forward_ex", "vsa_coarse_backward_ex", "vsa_fine_forward_range",
    "vsa_fine_backward_range", "vsa_op_backward_prologue", "vsa_op_backward_finish",
]


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", CSRC], check=True)
    return LIB_PATH


class VsaError(RuntimeError):
    pass


_lib = None

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
LP = C.POINTER(vsa_layout_t)


def lib():
    """Load libvsa_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libvsa_b200.so not built at {LIB_PATH}; run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    L.vsa_last_error.restype = C.c_char_p
    L.vsa_version.restype = C.c_char_p
    L.vsa_kernel_launches.restype = C.c_uint64
    sig = {
        "vsa_layout_make": [I64] * 6 + [I32, LP],
        "vsa_debug_trace": [P, I32, I32, I32],
        "vsa_debug_tile_counter": [P],
        "vsa_layout_set_io": [LP, I32, I64, I64, I64],
        "vsa_transpose_blocks": [P, P, I64, I64, I64, P],
        "vsa_gate_forward": [LP, I64, I64, I64, I64, P, P, P, I32, I32, P, P, P],
        "vsa_gate_backward": [LP, I64, I64, I64, I64, P, P, P, P, P, P, I32, I32, P, P, P, P, P],
        "vsa_gate_backward_workspace_bytes": [LP, I64, I64, I64],
        "vsa_selection_accuracy_from_lse": [P, P, I64, I64, P, P],
        "vsa_aggregate_probs_to_cubes": [LP, I64, P, P, P],
        "vsa_selection_accuracy": [LP, I64, P, P, I64, P, P],
        "vsa_flatten_index": [LP, I64, I64, I64, C.POINTER(I64)],
        "vsa_tile": [LP, I64, I64, I32, P, P, P],
        "vsa_untile": [LP, I64, I64, I32, P, P, P],
        "vsa_tile_pool": [LP, I64, I64, I32, I32, C.POINTER(P), C.POINTER(P), C.POINTER(P), I32, P],
        "vsa_pool_tiled": [LP, I64, I64, I32, P, P, I32, P],
        "vsa_coarse_forward": [LP, I64, I64, P, P, P, I64, P, P, P, P, P, P, P],
        "vsa_selection_transpose": [LP, I64, P, I64, P, P, P, P],
        "vsa_validate_selection": [P, I64, I64, I64, P, P],
        "vsa_fine_forward": [LP, I64, I64, I32, P, P, P, P, I64, P, P, P, P, P, P, I32, P, P],
        "vsa_backward_prologue": [LP, I64, I64, I32, I32, P, P, P, P, P, I32, P, P, P, P, P, P],
        "vsa_coarse_backward": [LP, I64, I64, P, P, P, P, P, P, P, P, P, P],
        "vsa_fine_backward": [LP, I64, I64, I32, P, P, P, P, P, P, P, I64, P, P, P, P, P, I32, I32, P, P, P, P,
                              C.c_size_t, P],
        "vsa_unpool_max_add": [LP, I64, I64, I32, P, P, I32, P, P],
        "vsa_op_create": [LP, C.POINTER(vsa_op_desc_t), P, C.c_size_t, C.POINTER(P)],
        "vsa_op_destroy": [P],
        "vsa_op_buffers": [P, C.POINTER(vsa_op_buffers_t)],
        "vsa_op_set_workspace": [P, P, C.c_size_t],
        "vsa_op_forward": [P, P, P, P, P, P, P, I64, P, P],
        "vsa_op_forward_coarse": [P, P, P, P, P, I64, P],
        "vsa_op_forward_fine": [P, P, P, P, P],
        "vsa_op_backward": [P, P, P, P, P, P, P, P],
        "vsa_op_backward_prologue": [P, P, P, P, P],
        "vsa_op_backward_finish": [P, P, P, P, P],
        "vsa_fine_forward_range": [LP, I64, I64, I32, P, P, P, P, I64, P, P, P, P, P, P, I32, P, I64, I64, P],
        "vsa_fine_backward_range": [LP, I64, I64, I32, P, P, P, P, P, P, P, I64, P, P, P, P, P, I32, I32, P, P, P, P,
                                    C.c_size_t, I64, I64, P],
        "vsa_forward": [P, P, P, P, P, P, P, P, I64, P, P],
        "vsa_backward": [P, P, P, P, P, P, P, P, P, P, P],
        "vsa_op_timing": [P, I32],
        "vsa_op_stage_ms": [P, C.POINTER(C.c_float), C.POINTER(I32)],
        "vsa_coarse_forward_ex": [LP, I64, I64, P, P, P, I64, I32, P, P, P, P, P, P, P, P],
        "vsa_coarse_backward_ex": [LP, I64, I64, P, P, P, P, P, P, P, P, P, I32, P, P],
        "vsa_coarse_backward_tokens": [LP, I64, I64, I32, P, P, P, P, I32, P, P, P, P, P, P, P, P, P, P, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.vsa_coarse_bitmap_bytes.argtypes = [LP, I64]
    L.vsa_coarse_bitmap_bytes.restype = C.c_size_t
    L.vsa_fine_backward_workspace_bytes.argtypes = [LP, I64, I64]
    L.vsa_fine_backward_workspace_bytes.restype = C.c_size_t
    L.vsa_gate_backward_workspace_bytes.restype = C.c_size_t
    L.vsa_op_memory_bytes.argtypes = [LP, C.POINTER(vsa_op_desc_t)]
    L.vsa_op_memory_bytes.restype = C.c_size_t
    L.vsa_coarse_workspace_bytes.argtypes = [LP, I64, I64, I32]
    L.vsa_coarse_workspace_bytes.restype = C.c_size_t
    L.vsa_op_workspace_bytes.argtypes = [P, I64]
    L.vsa_op_workspace_bytes.restype = C.c_size_t
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's error behaviour (invalid_argument -> ValueError)."""
    if rc == 0:
        return
    msg = lib().vsa_last_error().decode()
    if rc < 0:
        raise ValueError(msg)
    raise VsaError(f"CUDA error {rc}: {msg}")

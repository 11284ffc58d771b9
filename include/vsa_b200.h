/* SPDX-License-Identifier: Apache-2.0
 *
 * vsa_b200.h — C ABI of the B200-native VSA (Video Sparse Attention) hot path.
 *
 * Drop-in boundary for the reference's C++ entry points in
 * /root/reference/proj/include/vsa/*.hpp. Every function takes plain device
 * pointers and sizes (no torch / Eigen types), is stream-ordered and
 * asynchronous, and returns an int status:
 *     0            success
 *     < 0          invalid argument (VSA_EINVAL) — the reference throws
 *                  std::invalid_argument for the same preconditions
 *                  (tensor.hpp:18-20); message via vsa_last_error()
 *     > 0          a cudaError_t from a launch
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *
 * Tensor conventions (AttnTensor, tensor.hpp:44-123): contiguous [B, H, S, d].
 *   raster  : S = t*h*w tokens in t-major raster order (the video grid)
 *   tiled   : S = nc*cube tokens in cube-contiguous order (layout.hpp:43-55),
 *             zero-padded to cube multiples when pad_mode = VSA_PAD_ZERO
 *   cube    : S = nc, one row per cube (pooled / coarse quantities), fp32
 * dtype VSA_BF16 = bf16 storage with fp32 accumulation (tcgen05 path);
 * dtype VSA_F32  = fp32 storage and arithmetic (parity mode, SIMT kernels).
 */
#ifndef VSA_B200_H_
#define VSA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { VSA_OK = 0, VSA_EINVAL = -1 };
enum { VSA_F32 = 0, VSA_BF16 = 1 };
enum { VSA_POOL_MEAN = 0, VSA_POOL_MAX = 1 };            /* PoolMode, coarse.hpp:13 */
/* layout.cpp:10-11 rejects non-divisible grids; the two pad modes are extensions:
 * ZERO: the grid is padded with zero tokens that are ordinary tokens (pooled, attendable) — the
 *       reference run on the padded layout (parity mode);
 * MASK: FastVideo-style — padded keys are excluded from attention (-inf), cube means / maxima are
 *       over the valid tokens only, the mean unpool divides by the valid count. */
enum { VSA_PAD_REJECT = 0, VSA_PAD_ZERO = 1, VSA_PAD_MASK = 2 };
enum { VSA_GATE_IDENTITY = 0, VSA_GATE_SIGMOID = 1 };    /* GateActivation, vsa.hpp:9 */
/* Raster I/O order of the raster-ordered tensors (q, k, v, gates, out, dO, grads).
 * HEAD_MAJOR: [B, H, S, d] (AttnTensor, tensor.hpp:44-123).
 * SEQ_MAJOR : [S/chunk][B][chunk][H][d]; chunk = S is the DiT-native [B, S, H, d]
 *             (SURVEY.md §8f2), chunk = S/P is the receive buffer of a Ulysses
 *             sequence->head all-to-all over P ranks, consumed in place (§8e). */
enum { VSA_IO_HEAD_MAJOR = 0, VSA_IO_SEQ_MAJOR = 1 };

/* Fine-stage epilogue flags (vsa_fine_forward). */
enum {
  VSA_FINE_COMBINE = 1,     /* out = Oc*Gc + Of*Gf (vsa.hpp:118-120); needs gc, gf/ADAPTATION, oc_cube */
  VSA_FINE_UNTILE = 2,      /* write `out` in raster order (layout.hpp:58-70), padded rows dropped */
  VSA_FINE_ADAPTATION = 4,  /* Gf == 1 (vsa.hpp:112): gf may be NULL */
  VSA_FINE_FORCE_SIMT = 8   /* use the SIMT kernels even for bf16 (debug / cross-check) */
};

/* TileLayout (layout.hpp:14-33, layout.cpp:6-31), plus padded extents. */
typedef struct vsa_layout_t {
  int64_t t, h, w;        /* token extents of the raster grid */
  int64_t ct, ch, cw;     /* cube extents */
  int64_t tp, hp, wp;     /* padded extents (== t,h,w unless padded) */
  int64_t nt, nh, nw;     /* cubes per axis */
  int64_t cube;           /* tokens per cube (B) */
  int64_t seq;            /* raster tokens t*h*w (L) */
  int64_t seq_padded;     /* nc*cube */
  int64_t nc;             /* number of cubes */
  int32_t pad_mode;
  int32_t io_order;       /* raster I/O order, VSA_IO_* (vsa_layout_set_io); 0 after vsa_layout_make */
  int64_t io_batch;       /* B (VSA_IO_SEQ_MAJOR only) */
  int64_t io_heads;       /* H (VSA_IO_SEQ_MAJOR only) */
  int64_t io_chunk;       /* sequence chunk, divides seq (VSA_IO_SEQ_MAJOR only) */
} vsa_layout_t;

/* Last error message of the calling thread ("" if none). */
const char* vsa_last_error(void);
/* Library version / build string. */
const char* vsa_version(void);
/* Number of CUDA kernels this library has launched in this process (all entries). */
uint64_t vsa_kernel_launches(void);
/* Debug: record pipeline events (clock64, code, index) of CTA (cta_x, cta_y) of the
 * instrumented kernels into the device buffer `buf` (uint64: [0] = count, then pairs);
 * buf = NULL disables. Not thread-safe; for profiling only. */
int vsa_debug_trace(void* buf, int32_t cap, int32_t cta_x, int32_t cta_y);
/* Debug: MacCounter on the device (tensor.hpp:36-39, fine.hpp:59-63). While set, every
 * fine-forward launch atomically adds the number of (query cube, key cube) tiles its
 * CTAs actually executed to *dev_counter (a device uint64); MACs = tiles * 2 * cube^2 * d.
 * NULL disables. Process-global, not thread-safe; for instrumentation only. */
int vsa_debug_tile_counter(uint64_t* dev_counter);

/* Replaces: TileLayout::TileLayout (layout.cpp:6-31). VSA_PAD_REJECT reproduces
 * the reference's divisibility check (layout.cpp:10-11); VSA_PAD_ZERO rounds the
 * extents up to cube multiples. */
int vsa_layout_make(int64_t t, int64_t h, int64_t w, int64_t ct, int64_t ch, int64_t cw, int32_t pad_mode,
                    vsa_layout_t* out);

/* Extension (no reference counterpart; the reference's AttnTensor is always
 * [B,H,S,d]): select the raster I/O order for every call that takes this layout.
 * SEQ_MAJOR needs batch, heads (bh = batch*heads at each call) and a chunk that
 * divides t*h*w; HEAD_MAJOR ignores them. Tiled/cube tensors are unaffected. */
int vsa_layout_set_io(vsa_layout_t* layout, int32_t order, int64_t batch, int64_t heads, int64_t chunk);

/* Replaces: flatten_index (layout.cpp:40-42); host-side, no device work.
 * Out-of-range coordinates -> VSA_EINVAL (raster_index, layout.cpp:33-38). */
int vsa_flatten_index(const vsa_layout_t* layout, int64_t t, int64_t h, int64_t w, int64_t* out);

/* Replaces: tile<S> / untile<S> (layout.hpp:43-70). x: raster [B*H, seq, d]
 * <-> tiled [B*H, seq_padded, d]; padded rows are written as zeros by tile and
 * dropped by untile. */
int vsa_tile(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* x_raster, void* x_tiled,
             void* stream);
int vsa_untile(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled, void* x_raster,
               void* stream);

/* K1+K2 — Replaces: tile<S> (layout.hpp:43-55) fused with pool_cubes
 * (coarse.hpp:47-65) for n tensors in one pass. pooled[i]: fp32 [B*H, nc, d],
 * mean = sequential fp32 sum over the cube's tokens in tile order / cube.
 * x_tiled[i] may be NULL (pool only). */
int vsa_tile_pool(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, int32_t n,
                  const void* const* x_raster, void* const* x_tiled, float* const* pooled, int32_t pool_mode,
                  void* stream);
/* Replaces: pool_cubes (coarse.hpp:47-65) on an already tile-ordered tensor. */
int vsa_pool_tiled(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled,
                   float* pooled, int32_t pool_mode, void* stream);

/* K3 — Replaces: coarse_forward_select (coarse.hpp:71-117) from pooled inputs.
 * Canonical fp32 order (bit-exact with oracle/): scores = fma-chain dot * fl(1/sqrt(d)),
 * softmax with canon_exp and sequential row sum, top-k (ties -> lower index,
 * ascending), Oc = Ac * Vc. Outputs: ac fp32 [B*H, nc, nc] (probabilities),
 * oc_cube fp32 [B*H, nc, d], sel int32 [B*H, nc, top_k], and the transposed
 * block map in CSR form (the reference's `rev`, fine.hpp:163-170):
 * selT_offs int32 [B*H, nc+1], selT_idx int32 [B*H, nc*top_k], q-cubes ascending.
 * selT_* may be NULL. bitmap_ws: device scratch of vsa_coarse_bitmap_bytes() bytes. */
int vsa_coarse_forward(const vsa_layout_t* layout, int64_t bh, int64_t d, const float* qc, const float* kc,
                       const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel, int32_t* selT_offs,
                       int32_t* selT_idx, void* bitmap_ws, void* stream);
size_t vsa_coarse_bitmap_bytes(const vsa_layout_t* layout, int64_t bh);

/* Coarse-stage precision (north_star kernel 3 / H3):
 * VSA_COARSE_F32 : canonical fp32 order on the SIMT pipes — probabilities and the block map
 *                  bit-exact with the reference's top-k (the parity mode, default);
 * VSA_COARSE_BF16: the coarse products on the tensor cores (tcgen05, TMEM accumulators, TMA)
 *                  from bf16 copies of the pooled cubes, the same fused softmax + top-k +
 *                  transposed-map kernel; the map can differ where bf16 moves a score across
 *                  the top-k boundary (validated by feeding the fine stage the oracle's map).
 * The bf16 mode needs nc % 8 == 0 and a workspace of vsa_coarse_workspace_bytes(); it keeps
 * bf16 Qc/Kc/Vc/P there for vsa_coarse_backward_ex. */
enum { VSA_COARSE_F32 = 0, VSA_COARSE_BF16 = 1 };
size_t vsa_coarse_workspace_bytes(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t precision);
int vsa_coarse_forward_ex(const vsa_layout_t* layout, int64_t bh, int64_t d, const float* qc, const float* kc,
                          const float* vc, int64_t top_k, int32_t precision, float* ac, float* oc_cube, int32_t* sel,
                          int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* coarse_ws, void* stream);
int vsa_coarse_backward_ex(const vsa_layout_t* layout, int64_t bh, int64_t d, const float* qc, const float* kc,
                           const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc, float* dvc,
                           float* scratch, int32_t precision, void* coarse_ws, void* stream);

/* Builds the transposed CSR map from a user-supplied block map (e.g. the
 * sel_override of vsa.hpp:93,115, or random_selection / all_cubes). */
int vsa_selection_transpose(const vsa_layout_t* layout, int64_t bh, const int32_t* sel, int64_t top_k,
                            int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* stream);

/* Replaces: BlockSelection::validate (selection.cpp:24-37) on device. Writes 0
 * to *err_dev if every row is strictly ascending and in [0, nc), else 1. */
int vsa_validate_selection(const int32_t* sel, int64_t rows, int64_t top_k, int64_t nc, int32_t* err_dev,
                           void* stream);

/* K4+K5 — Replaces: fine_forward (fine.hpp:43-99) and, with
 * VSA_FINE_COMBINE|VSA_FINE_UNTILE, the combine of vsa_forward (vsa.hpp:118-120)
 * plus untile (layout.hpp:58-70) in the epilogue.
 *   q,k,v   : tiled [B*H, seq_padded, d] (dtype)
 *   sel     : int32 [B*H, nc, top_k], strictly ascending rows (validated by the caller)
 *   o_fine  : tiled [B*H, seq_padded, d] (dtype), the fine output Of
 *   lse     : fp32 [B*H, seq_padded], row_lse = m + log(l) (fine.hpp:94-96)
 *   row_max : fp32 [B*H, seq_padded] or NULL (fine.hpp:93)
 *   gc, gf  : gates, same order as `out` (raster if UNTILE else tiled), dtype
 *   oc_cube : fp32 [B*H, nc, d] coarse output at cube level
 *   out     : combined output (dtype) or NULL. */
int vsa_fine_forward(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                     const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max,
                     const void* gc, const void* gf, const float* oc_cube, int32_t flags, void* out, void* stream);

/* Task-range variants (a head sub-split across GPUs): the forward computes
 * only query cubes t = u*nc + qc in [task_begin, task_end) (their out / o_fine / lse rows);
 * the backward computes dQ for those query cubes and dK/dV for the key cubes of the same
 * range. lse and delta must hold every query row of the units involved (a rank exchanges
 * its rows with the ranks sharing a unit); dQ then recomputes S / dP (no dS workspace: the
 * dS tiles of a query cube come from other ranks' key cubes). tcgen05 path only. */
int vsa_fine_forward_range(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* q,
                           const void* k, const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse,
                           float* row_max, const void* gc, const void* gf, const float* oc_cube, int32_t flags,
                           void* out, int64_t task_begin, int64_t task_end, void* stream);
int vsa_fine_backward_range(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* q,
                            const void* k, const void* v, const void* dof, const float* lse, const float* delta,
                            const int32_t* sel, int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx,
                            const float* dqc, const float* dkc, const float* dvc, int32_t raster, int32_t flags,
                            void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, int64_t task_begin,
                            int64_t task_end, void* stream);

/* K6a — backward prologue, the elementwise part of vsa_backward (vsa.hpp:142-150)
 * fused with the tile of dO and the fine delta:
 *   dof  = dO*Gf (tiled, dtype)                 dgc = dO*Oc  (same order as dout)
 *   dgf  = dO*Of (0 in adaptation)              doc_cube = sum over each cube's tokens of dO*Gc (fp32)
 *   delta = rowsum(dof * Of)  fp32 [B*H, seq_padded]  (== fine.hpp:142-149's sum P*dP)
 * dout, gc, gf, dgc, dgf are raster when `raster` != 0, else tiled. dgc/dgf may be NULL. */
int vsa_backward_prologue(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, int32_t raster,
                          const void* dout, const void* gc, const void* gf, const float* oc_cube, const void* o_fine,
                          int32_t adaptation, void* dof, float* delta, float* doc_cube, void* dgc, void* dgf,
                          void* stream);

/* K6d — Replaces the cube-level part of coarse_backward (coarse.hpp:143-162):
 * from doc_cube (token dOc summed per cube) produce dqc, dkc, dvc fp32 [B*H, nc, d].
 * scratch: fp32 [B*H, nc, nc]. */
int vsa_coarse_backward(const vsa_layout_t* layout, int64_t bh, int64_t d, const float* qc, const float* kc,
                        const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc, float* dvc,
                        float* scratch, void* stream);

/* K6b+K6c — Replaces: fine_backward (fine.hpp:107-204) plus the coarse unpool
 * (coarse.hpp:164-178, mean mode) and the grad sum of vsa_backward (vsa.hpp:182-187):
 *   dq = dQ_fine + dqc/cube (broadcast), dk, dv likewise; dqc/dkc/dvc may be NULL.
 *   dof, lse, delta as produced by the forward / prologue; selT_* from the
 *   coarse stage or vsa_selection_transpose. Deterministic (no atomics on any
 *   gradient): dQ per query cube, dK/dV per key cube over the transposed map,
 *   q-cubes ascending (key cubes are handed to CTAs by a counter in the workspace;
 *   each is still computed by one CTA in a fixed order).
 *   Unselected key cubes get exactly zero fine gradient (test_fine.cpp:149-169).
 * raster != 0 writes dq/dk/dv in raster order (padded rows dropped).
 * workspace (device, >= vsa_fine_backward_workspace_bytes, may be NULL): with it the
 * tcgen05 path stores the bf16 dS tiles from the dK/dV pass and computes dQ as a
 * block-sparse GEMM over them (no S/dP recompute); without it dQ recomputes S and dP. */
int vsa_fine_backward(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                      const void* v, const void* dof, const float* lse, const float* delta, const int32_t* sel,
                      int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx, const float* dqc,
                      const float* dkc, const float* dvc, int32_t raster, int32_t flags, void* dq, void* dk,
                      void* dv, void* workspace, size_t workspace_bytes, void* stream);
/* Workspace size for the dS-materialising backward: B*H*nc*top_k tiles x (8 KiB + 4 B),
 * plus 256 B for the dK/dV task counter. */
size_t vsa_fine_backward_workspace_bytes(const vsa_layout_t* layout, int64_t bh, int64_t top_k);

/* Max-pool unpool (coarse.hpp:172-176): adds dxc[cube][j] to the first argmax
 * token of x (tiled) per (cube, channel) into dx (raster if `raster` else tiled, dtype). */
int vsa_unpool_max_add(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled,
                       const float* dxc, int32_t raster, void* dx, void* stream);

/* Replaces: the gate projection of vsa_forward (vsa.hpp:100-112): z = hidden . Wg
 * (+ bias), optional sigmoid, split into Gc = z[:, h*d:(h+1)*d] and Gf = z[:, (H+h)*d:...]
 * written as [B, H, S, d] bf16 in the layout's raster I/O order (Gf = 1 in adaptation
 * mode). hidden: bf16 [B, S, model_dim] (S = t*h*w); weight: bf16 [model_dim, 2*H*d]
 * row-major; bias: fp32 [2*H*d] or NULL. tcgen05 GEMM (gemm_sm100.cu); needs
 * model_dim % 64 == 0 and 2*H*d % 256 == 0. */
int vsa_gate_forward(const vsa_layout_t* layout, int64_t batch, int64_t heads, int64_t d, int64_t model_dim,
                     const void* hidden, const void* weight, const float* bias, int32_t activation,
                     int32_t adaptation, void* gc, void* gf, void* stream);
/* Replaces: the gate part of vsa_backward (vsa.hpp:152-176): dz = [dGc, dGf] (times
 * G(1-G) for sigmoid; the Gf half is 0 in adaptation mode), dhidden = dz . Wg^T (bf16
 * [B, S, model_dim]), dWg = hidden^T . dz (fp32 [model_dim, 2*H*d]), dbias = column sums
 * of dz (fp32, NULL to skip). gc/gf are the activated gates of the forward (needed for
 * sigmoid). Workspace: vsa_gate_backward_workspace_bytes. model_dim % 256 == 0. */
int vsa_gate_backward(const vsa_layout_t* layout, int64_t batch, int64_t heads, int64_t d, int64_t model_dim,
                      const void* hidden, const void* weight, const void* gc, const void* gf, const void* dgc,
                      const void* dgf, int32_t activation, int32_t adaptation, void* dz_workspace, void* dhidden,
                      float* dweight, float* dbias, void* stream);
size_t vsa_gate_backward_workspace_bytes(const vsa_layout_t* layout, int64_t batch, int64_t heads, int64_t d);

/* Selection analytics (analysis.hpp:100-147, dense.hpp:214-240).
 * vsa_selection_accuracy_from_lse: acc[u] = mean_i exp(lse_sel[u,i] - lse_all[u,i]) (double),
 * the attention mass captured by a block map, from the row log-sum-exps of vsa_fine_forward
 * run with the selection and with all cubes — equal to selection_accuracy(
 * aggregate_probs_to_cubes(dense_probs(q, k)), sel) without any [S,S] matrix.
 * vsa_aggregate_probs_to_cubes / vsa_selection_accuracy: the reference's diagnostics on
 * materialised fp32 probabilities ([bh,S,S] -> [bh,S,nc]; [bh,S,nc] + sel -> acc), unpadded
 * layouts. */
int vsa_selection_accuracy_from_lse(const float* lse_sel, const float* lse_all, int64_t bh, int64_t seq,
                                    double* acc, void* stream);
int vsa_aggregate_probs_to_cubes(const vsa_layout_t* layout, int64_t bh, const float* probs, float* out,
                                 void* stream);
int vsa_selection_accuracy(const vsa_layout_t* layout, int64_t bh, const float* probs_cube, const int32_t* sel,
                           int64_t top_k, double* acc, void* stream);

/* ============================================================================
 * The operator context (SURVEY.md §8b "device-side context"): vsa_forward /
 * vsa_backward (vsa.hpp:89-93, 129-133) with the forward artifacts (the VsaOutput of
 * vsa.hpp:56-63: pooled cubes, Ac, Oc, block map + transposed map, fine output, lse,
 * gates) resident in HBM between the two calls. One context per (layout, shape); the
 * calls are stream-ordered and asynchronous.
 * ========================================================================== */
typedef struct vsa_op vsa_op_t;

enum {
  VSA_OP_FORCE_SIMT = 1,       /* SIMT fine kernels (fp32 parity mode / debug) even for bf16 */
  VSA_OP_NO_DS_WORKSPACE = 2   /* backward recomputes S / dP for dQ even when a workspace is attached */
};

typedef struct vsa_op_desc_t {
  int64_t batch, heads, head_dim;
  int64_t top_k;       /* VsaParams::top_k (vsa.hpp:20), 1 <= top_k <= nc */
  int64_t max_sel_k;   /* largest k of a sel_override (0 = top_k) */
  int64_t model_dim;   /* > 0: the gate projection of vsa_forward / vsa_backward (VsaParams::gate_weight rows) */
  int32_t dtype;       /* VSA_BF16 (tcgen05) or VSA_F32 (parity mode) */
  int32_t pool_mode;   /* VsaParams::pool (vsa.hpp:21) */
  int32_t activation;  /* VsaParams::activation (vsa.hpp:22) */
  int32_t adaptation;  /* VsaParams::adaptation (vsa.hpp:23): Gf == 1 */
  int32_t raster;      /* 1: q/k/v/gates/out/dO/grads raster-ordered (tiling fused); 0: tile-ordered (vsa.hpp:86) */
  int32_t flags;       /* VSA_OP_* */
  int32_t coarse;      /* VSA_COARSE_F32 (bit-exact map, default) or VSA_COARSE_BF16 (tcgen05) */
  int32_t reserved;
  /* Sub-split: the fine stages compute only the (unit, cube) tasks
   * t = u*nc + c in [task_begin, task_end) of this op's units (0, 0 = all). Between
   * vsa_op_forward and vsa_op_backward_finish the caller completes lse (after the forward)
   * and delta (after vsa_op_backward_prologue) with the rows of the other ranks. */
  int64_t task_begin, task_end;
} vsa_op_desc_t;

/* Device pointers of the context's buffers (views for callers and tests). */
typedef struct vsa_op_buffers_t {
  void* base;
  size_t bytes;
  void *q_t, *k_t, *v_t;                /* tiled copies (raster mode), else NULL */
  float *qc, *kc, *vc, *ac, *oc_cube;   /* CoarseArtifacts (coarse.hpp:18-25), Oc at cube level */
  int32_t *sel, *selT_offs, *selT_idx;  /* coarse top-k map, transposed CSR map of the map the fine stage used */
  void* o_fine;                         /* FineResult::out, tiled */
  float* lse;                           /* FineSaved::row_lse [B*H, Lp] */
  void* dof;
  float *delta, *doc_cube, *dqc, *dkc, *dvc;
  void *gc, *gf, *dgc, *dgf;            /* gates (model_dim > 0) */
  const int32_t* fine_sel;              /* selection the fine stage used (VsaOutput::fine_sel) */
  int64_t fine_k;
  int32_t bwd_used_workspace;           /* last backward: 1 = dS workspace path, 0 = recompute */
} vsa_op_buffers_t;

/* Bytes of device memory vsa_op_create needs (0 for an invalid descriptor). */
size_t vsa_op_memory_bytes(const vsa_layout_t* layout, const vsa_op_desc_t* desc);
/* device_memory: caller-owned block of >= vsa_op_memory_bytes, or NULL (the op cudaMallocs
 * and frees it). The layout (with its raster I/O order) is copied. */
int vsa_op_create(const vsa_layout_t* layout, const vsa_op_desc_t* desc, void* device_memory, size_t bytes,
                  vsa_op_t** op);
int vsa_op_destroy(vsa_op_t* op);
int vsa_op_buffers(const vsa_op_t* op, vsa_op_buffers_t* out);
/* dS workspace of the backward (>= vsa_op_workspace_bytes(op, k)); NULL = recompute path. */
int vsa_op_set_workspace(vsa_op_t* op, void* ws, size_t bytes);
size_t vsa_op_workspace_bytes(const vsa_op_t* op, int64_t sel_k);

/* Attention-level forward (gates given): K1-K3 (vsa_op_forward_coarse) then K4+K5
 * (vsa_op_forward_fine). sel_override (vsa.hpp:93,115): device int32 [B*H, nc, sel_k]
 * replacing the fine stage's map (the coarse stage still computes its own top-k); it is
 * validated with one synchronous flag read. */
int vsa_op_forward(vsa_op_t* op, const void* q, const void* k, const void* v, const void* gc, const void* gf,
                   const int32_t* sel_override, int64_t sel_k, void* out, void* stream);
int vsa_op_forward_coarse(vsa_op_t* op, const void* q, const void* k, const void* v, const int32_t* sel_override,
                          int64_t sel_k, void* stream);
int vsa_op_forward_fine(vsa_op_t* op, const void* gc, const void* gf, void* out, void* stream);
/* Attention-level backward: dO -> dq, dk, dv, dgc, dgf (dgc/dgf may be NULL) =
 * vsa_op_backward_prologue (K6a + K6d: dof, delta, dgc, dgf, coarse cube gradients) then
 * vsa_op_backward_finish (K6b/K6c + unpool). */
int vsa_op_backward(vsa_op_t* op, const void* dout, void* dq, void* dk, void* dv, void* dgc, void* dgf,
                    void* stream);
int vsa_op_backward_prologue(vsa_op_t* op, const void* dout, void* dgc, void* dgf, void* stream);
int vsa_op_backward_finish(vsa_op_t* op, void* dq, void* dk, void* dv, void* stream);

/* Replaces: vsa_forward (vsa.hpp:89-122). hidden: bf16 [B, S, model_dim] in the op's row
 * order (raster tokens, or tile order when desc.raster == 0); gate_weight bf16
 * [model_dim, 2*H*d]; gate_bias fp32 [2*H*d] or NULL. The gates stay in the context. */
int vsa_forward(vsa_op_t* op, const void* hidden, const void* gate_weight, const float* gate_bias, const void* q,
                const void* k, const void* v, const int32_t* sel_override, int64_t sel_k, void* out, void* stream);
/* Replaces: vsa_backward (vsa.hpp:129-189): dq, dk, dv (coarse + fine paths), dhidden
 * bf16 [B, S, model_dim], dgate_weight fp32 [model_dim, 2*H*d], dgate_bias fp32 or NULL.
 * Missing forward artifacts -> VSA_EINVAL (vsa.hpp:137-138). */
int vsa_backward(vsa_op_t* op, const void* hidden, const void* gate_weight, const void* dout, void* dq, void* dk,
                 void* dv, void* dhidden, float* dgate_weight, float* dgate_bias, void* stream);

/* Stage timing without host gaps: with timing on, each call records CUDA events between
 * its stages on the launch stream; vsa_op_stage_ms synchronises once and returns the mean
 * per stage over the timed calls: [tile_pool, coarse_fwd, fine_fwd, prologue, coarse_bwd,
 * fine_bwd]. calls (nullable) = {forward calls, backward calls}. */
enum { VSA_OP_STAGES = 6 };
int vsa_op_timing(vsa_op_t* op, int32_t enable);
int vsa_op_stage_ms(vsa_op_t* op, float* ms, int32_t* calls);

/* Replaces the token-level coarse_backward (coarse.hpp:124-184) on tile-ordered tensors:
 * doc tiled [B*H, Lp, d] -> cube sums -> K6d -> unpool (mean: broadcast dxc/cube; max:
 * first argmax token of x_tiled) into dq, dk, dv tiled. Scratch fp32: doc_cube, dqc,
 * dkc, dvc [B*H, nc, d] and [B*H, nc, nc]. q/k/v tiled are needed for max pooling only. */
int vsa_coarse_backward_tokens(const vsa_layout_t* layout, int64_t bh, int64_t d, int32_t dtype, const float* qc,
                               const float* kc, const float* vc, const float* ac, int32_t pool_mode,
                               const void* doc, const void* q_t, const void* k_t, const void* v_t, float* doc_cube,
                               float* dqc, float* dkc, float* dvc, float* scratch, void* dq, void* dk, void* dv,
                               void* stream);

/* Ulysses resharding copy: dst[i1][i0] = src[i0][i1] over an
 * [n0][n1] grid of contiguous blocks of `block_bytes` (a multiple of 16). With
 * n0 = B*S/P, n1 = P, block = (H/P)*d*elem it packs a sequence shard [B,S/P,H,d]
 * into the per-destination send buffer [P][B][S/P][H/P][d] (and, swapped, unpacks
 * the returned head groups). 128-bit loads and stores, one pass. */
int vsa_transpose_blocks(const void* src, void* dst, int64_t n0, int64_t n1, int64_t block_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VSA_B200_H_ */

#include <cstdlib>
// SPDX-License-Identifier: Apache-2.0
// The C ABI (include/vsa_b200.h): argument validation with the reference's
// precondition messages (std::invalid_argument -> VSA_EINVAL + vsa_last_error),
// then dispatch to the kernel launchers. No CPU compute path exists: every
// entry either launches CUDA work or fails.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "common.cuh"
#include "launch.h"

namespace vsa_host {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return 0;
  set_error("%s: %s", where, cudaGetErrorString(e));
  return int(e);
}

static std::atomic<uint64_t> g_launches{0};
static vsa_dev::TraceCfg g_trace{nullptr, 0, 0, 0};

vsa_dev::TraceCfg debug_trace() { return g_trace; }

static unsigned long long* g_tile_ctr = nullptr;
unsigned long long* debug_tile_counter() { return g_tile_ctr; }

int kernel_status(const char* where) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError(), where);
}

static bool dtype_ok(int32_t dt) { return dt == VSA_F32 || dt == VSA_BF16; }
static int vec_elems(int32_t dt) { return dt == VSA_BF16 ? 8 : 4; }

static int check_layout(const vsa_layout_t* L) {
  VSA_REQUIRE(L != nullptr, "layout: null pointer");
  VSA_REQUIRE(L->nc >= 1 && L->cube >= 1 && L->seq_padded == L->nc * L->cube, "layout: not initialised");
  VSA_REQUIRE(L->io_order == VSA_IO_HEAD_MAJOR || L->io_order == VSA_IO_SEQ_MAJOR, "layout: unknown io order");
  return 0;
}

// Sequence-major raster I/O addresses rows by (b, h) = (u / H, u % H): the unit
// count must be the layout's B*H.
static int check_io(const vsa_layout_t* L, int64_t bh) {
  if (L->io_order == VSA_IO_SEQ_MAJOR)
    VSA_REQUIRE(bh == L->io_batch * L->io_heads, "sequence-major I/O: bh must equal batch*heads of the layout");
  return 0;
}

// Head-dim contract of the vectorised HBM kernels: 16-byte chunks per row,
// chunk count a power of two <= 32.
static int check_vec_dim(int64_t d, int32_t dtype) {
  const int V = vec_elems(dtype);
  VSA_REQUIRE(d >= 1 && d % V == 0, "head_dim must be a multiple of 16 bytes (4 fp32 / 8 bf16)");
  const int64_t chunks = d / V;
  VSA_REQUIRE(chunks <= 32 && (chunks & (chunks - 1)) == 0, "head_dim/16B must be a power of two <= 32");
  return 0;
}

}  // namespace vsa_host

using namespace vsa_host;

#define VSA_CHECKED(expr)   \
  do {                      \
    int _rc = (expr);       \
    if (_rc) return _rc;    \
  } while (0)

extern "C" {

const char* vsa_last_error(void) { return g_err.c_str(); }
const char* vsa_version(void) { return "vsa_b200 0.1 (sm_100a)"; }
uint64_t vsa_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int vsa_debug_trace(void* buf, int32_t cap, int32_t cta_x, int32_t cta_y) {
  g_trace = vsa_dev::TraceCfg{static_cast<unsigned long long*>(buf), cap, cta_x, cta_y};
  return VSA_OK;
}

int vsa_debug_tile_counter(uint64_t* dev_counter) {
  g_tile_ctr = reinterpret_cast<unsigned long long*>(dev_counter);
  return VSA_OK;
}

int vsa_layout_make(int64_t t, int64_t h, int64_t w, int64_t ct, int64_t ch, int64_t cw, int32_t pad_mode,
                    vsa_layout_t* out) {
  VSA_REQUIRE(out != nullptr, "TileLayout: null output");
  VSA_REQUIRE(t >= 1 && h >= 1 && w >= 1, "TileLayout: token extents must be >= 1");
  VSA_REQUIRE(ct >= 1 && ch >= 1 && cw >= 1, "TileLayout: cube extents must be >= 1");
  VSA_REQUIRE(pad_mode == VSA_PAD_REJECT || pad_mode == VSA_PAD_ZERO || pad_mode == VSA_PAD_MASK,
              "TileLayout: unknown pad mode");
  if (pad_mode == VSA_PAD_REJECT)
    VSA_REQUIRE(t % ct == 0 && h % ch == 0 && w % cw == 0,
                "TileLayout: token extents must be integer multiples of cube extents");
  vsa_layout_t L{};
  L.t = t; L.h = h; L.w = w; L.ct = ct; L.ch = ch; L.cw = cw;
  L.tp = (t + ct - 1) / ct * ct;
  L.hp = (h + ch - 1) / ch * ch;
  L.wp = (w + cw - 1) / cw * cw;
  L.nt = L.tp / ct; L.nh = L.hp / ch; L.nw = L.wp / cw;
  L.cube = ct * ch * cw;
  L.seq = t * h * w;
  L.nc = L.nt * L.nh * L.nw;
  L.seq_padded = L.nc * L.cube;
  L.pad_mode = pad_mode;
  VSA_REQUIRE(L.nc < (int64_t(1) << 30) && L.seq_padded < (int64_t(1) << 40), "TileLayout: too large");
  *out = L;
  return VSA_OK;
}

int vsa_layout_set_io(vsa_layout_t* L, int32_t order, int64_t batch, int64_t heads, int64_t chunk) {
  VSA_CHECKED(check_layout(L));
  VSA_REQUIRE(order == VSA_IO_HEAD_MAJOR || order == VSA_IO_SEQ_MAJOR, "layout_set_io: unknown order");
  if (order == VSA_IO_HEAD_MAJOR) {
    L->io_order = order;
    L->io_batch = L->io_heads = L->io_chunk = 0;
    return VSA_OK;
  }
  VSA_REQUIRE(batch >= 1 && heads >= 1, "layout_set_io: batch and heads must be >= 1");
  VSA_REQUIRE(chunk >= 1 && L->seq % chunk == 0, "layout_set_io: chunk must divide the raster sequence length");
  L->io_order = order;
  L->io_batch = batch;
  L->io_heads = heads;
  L->io_chunk = chunk;
  return VSA_OK;
}

int vsa_flatten_index(const vsa_layout_t* L, int64_t t, int64_t h, int64_t w, int64_t* out) {
  VSA_CHECKED(check_layout(L));
  VSA_REQUIRE(t >= 0 && t < L->t && h >= 0 && h < L->h && w >= 0 && w < L->w,
              "raster_index: coordinate out of range");
  const int64_t cube = ((t / L->ct) * L->nh + h / L->ch) * L->nw + w / L->cw;
  const int64_t off = ((t % L->ct) * L->ch + h % L->ch) * L->cw + w % L->cw;
  *out = cube * L->cube + off;
  return VSA_OK;
}

int vsa_tile(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* x_raster, void* x_tiled,
             void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "tile: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(bh >= 1 && x_raster && x_tiled, "tile: bad arguments");
  const void* xr[1] = {x_raster};
  void* xt[1] = {x_tiled};
  return launch_tile_pool(*L, bh, d, dtype, 1, xr, xt, nullptr, VSA_POOL_MEAN, 0, as_stream(stream));
}

int vsa_untile(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled, void* x_raster,
               void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "untile: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(bh >= 1 && x_raster && x_tiled, "untile: bad arguments");
  return launch_untile(*L, bh, d, dtype, x_tiled, x_raster, as_stream(stream));
}

int vsa_tile_pool(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, int32_t n,
                  const void* const* x_raster, void* const* x_tiled, float* const* pooled, int32_t pool_mode,
                  void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "tile_pool: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(n >= 1 && n <= 3 && x_raster && bh >= 1, "tile_pool: 1..3 tensors");
  VSA_REQUIRE(pool_mode == VSA_POOL_MEAN || pool_mode == VSA_POOL_MAX, "pool_cubes: unknown pool mode");
  for (int i = 0; i < n; ++i) VSA_REQUIRE(x_raster[i] != nullptr, "tile_pool: null input");
  return launch_tile_pool(*L, bh, d, dtype, n, x_raster, x_tiled, pooled, pool_mode, 0, as_stream(stream));
}

int vsa_pool_tiled(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled, float* pooled,
                   int32_t pool_mode, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "pool_cubes: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(pool_mode == VSA_POOL_MEAN || pool_mode == VSA_POOL_MAX, "pool_cubes: unknown pool mode");
  VSA_REQUIRE(x_tiled && pooled && bh >= 1, "pool_cubes: bad arguments");
  const void* xr[1] = {x_tiled};
  float* pl[1] = {pooled};
  return launch_tile_pool(*L, bh, d, dtype, 1, xr, nullptr, pl, pool_mode, 1, as_stream(stream));
}

size_t vsa_coarse_bitmap_bytes(const vsa_layout_t* L, int64_t bh) {
  if (!L || bh < 1) return 0;
  return coarse_bitmap_bytes(*L, bh);
}

int vsa_coarse_forward(const vsa_layout_t* L, int64_t bh, int64_t d, const float* qc, const float* kc,
                       const float* vc, int64_t top_k, float* ac, float* oc_cube, int32_t* sel, int32_t* selT_offs,
                       int32_t* selT_idx, void* bitmap_ws, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(top_k >= 1 && top_k <= L->nc, "coarse_forward_select: k must be in [1, num_cubes]");
  VSA_REQUIRE(d >= 1 && d <= 1024, "coarse_forward_select: head_dim out of range");
  VSA_REQUIRE(qc && kc && vc && ac && oc_cube && sel && bh >= 1, "coarse_forward_select: null buffer");
  VSA_REQUIRE((selT_offs == nullptr) == (selT_idx == nullptr), "coarse_forward_select: selT_offs/selT_idx pair");
  VSA_REQUIRE(selT_offs == nullptr || bitmap_ws != nullptr, "coarse_forward_select: transposed map needs bitmap_ws");
  // softmax + top-k keeps 4 rows of nc + 256 words in shared memory (227 KB per CTA)
  VSA_REQUIRE(L->nc <= 14080, "coarse_forward_select: num_cubes > 14080 unsupported");
  return launch_coarse_forward(*L, bh, d, qc, kc, vc, top_k, ac, oc_cube, sel, selT_offs, selT_idx, bitmap_ws,
                               as_stream(stream));
}

size_t vsa_coarse_workspace_bytes(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t precision) {
  if (!L || bh < 1 || d < 1 || precision != VSA_COARSE_BF16) return 0;
  return coarse_bf16_ws_bytes(*L, bh, d);
}

int vsa_coarse_forward_ex(const vsa_layout_t* L, int64_t bh, int64_t d, const float* qc, const float* kc,
                          const float* vc, int64_t top_k, int32_t precision, float* ac, float* oc_cube, int32_t* sel,
                          int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* coarse_ws, void* stream) {
  VSA_REQUIRE(precision == VSA_COARSE_F32 || precision == VSA_COARSE_BF16, "coarse: unknown precision");
  if (precision == VSA_COARSE_F32)
    return vsa_coarse_forward(L, bh, d, qc, kc, vc, top_k, ac, oc_cube, sel, selT_offs, selT_idx, bitmap_ws, stream);
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(top_k >= 1 && top_k <= L->nc, "coarse_forward_select: k must be in [1, num_cubes]");
  VSA_REQUIRE(d >= 8 && d % 8 == 0 && d <= 256, "coarse (bf16): head_dim must be a multiple of 8 in [8, 256]");
  VSA_REQUIRE(L->nc % 8 == 0, "coarse (bf16): num_cubes must be a multiple of 8 (use the fp32 coarse mode)");
  VSA_REQUIRE(L->nc <= 14080, "coarse_forward_select: num_cubes > 14080 unsupported");
  VSA_REQUIRE(qc && kc && vc && ac && oc_cube && sel && coarse_ws && bh >= 1, "coarse_forward_select: null buffer");
  VSA_REQUIRE((selT_offs == nullptr) == (selT_idx == nullptr), "coarse_forward_select: selT_offs/selT_idx pair");
  VSA_REQUIRE(selT_offs == nullptr || bitmap_ws != nullptr, "coarse_forward_select: transposed map needs bitmap_ws");
  return launch_coarse_forward_bf16(*L, bh, d, qc, kc, vc, top_k, ac, oc_cube, sel, selT_offs, selT_idx, bitmap_ws,
                                    coarse_ws, as_stream(stream));
}

int vsa_coarse_backward_ex(const vsa_layout_t* L, int64_t bh, int64_t d, const float* qc, const float* kc,
                           const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc, float* dvc,
                           float* scratch, int32_t precision, void* coarse_ws, void* stream) {
  VSA_REQUIRE(precision == VSA_COARSE_F32 || precision == VSA_COARSE_BF16, "coarse: unknown precision");
  if (precision == VSA_COARSE_F32)
    return vsa_coarse_backward(L, bh, d, qc, kc, vc, ac, doc_cube, dqc, dkc, dvc, scratch, stream);
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(ac != nullptr && coarse_ws != nullptr, "coarse_backward: artifacts do not match layout");
  VSA_REQUIRE(d >= 8 && d % 8 == 0 && d <= 256 && L->nc % 8 == 0, "coarse (bf16): unsupported shape");
  VSA_REQUIRE(doc_cube && dqc && dkc && dvc && scratch && bh >= 1, "coarse_backward: null buffer");
  return launch_coarse_backward_bf16(*L, bh, d, ac, doc_cube, dqc, dkc, dvc, scratch, coarse_ws, as_stream(stream));
}

int vsa_selection_transpose(const vsa_layout_t* L, int64_t bh, const int32_t* sel, int64_t top_k,
                            int32_t* selT_offs, int32_t* selT_idx, void* bitmap_ws, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(top_k >= 1 && top_k <= L->nc, "BlockSelection: k must be in [1, num_cubes]");
  VSA_REQUIRE(sel && selT_offs && selT_idx && bitmap_ws && bh >= 1, "selection_transpose: null buffer");
  return launch_selection_transpose(*L, bh, sel, top_k, selT_offs, selT_idx, bitmap_ws, as_stream(stream));
}

int vsa_validate_selection(const int32_t* sel, int64_t rows, int64_t top_k, int64_t nc, int32_t* err_dev,
                           void* stream) {
  VSA_REQUIRE(sel && err_dev, "BlockSelection: empty selection");
  VSA_REQUIRE(rows >= 1 && top_k >= 1 && top_k <= nc, "BlockSelection: k must be in [1, num_cubes]");
  return launch_validate_selection(sel, rows, top_k, nc, err_dev, as_stream(stream));
}

int vsa_fine_forward_range(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                           const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max,
                           const void* gc, const void* gf, const float* oc_cube, int32_t flags, void* out,
                           int64_t task_begin, int64_t task_end, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "fine stage: unknown dtype");
  VSA_REQUIRE(q && k && v && sel && o_fine && lse && bh >= 1, "fine stage: null buffer");
  VSA_REQUIRE(top_k >= 1 && top_k <= L->nc, "fine stage: selection does not match shapes");
  VSA_REQUIRE(d >= 1 && L->cube <= 128 && L->cube * d <= 8192, "fine stage: cube*head_dim > 8192 unsupported");
  VSA_REQUIRE(task_begin >= 0 && task_begin < task_end && task_end <= bh * L->nc,
              "fine stage: task range must be a non-empty part of [0, bh*nc)");
  if (flags & VSA_FINE_COMBINE)
    VSA_REQUIRE(out && gc && oc_cube && (gf || (flags & VSA_FINE_ADAPTATION)), "combine: missing gates / Oc");
  if (flags & VSA_FINE_UNTILE) VSA_REQUIRE(out != nullptr, "untile: missing output");
  cudaStream_t st = as_stream(stream);
  // bf16 runs on the tcgen05 kernels (64-token cubes, d in {64, 128}); the SIMT kernels
  // serve fp32 and, only when asked for explicitly, bf16 shapes outside that set
  if (dtype == VSA_BF16 && !(flags & VSA_FINE_FORCE_SIMT))
    VSA_REQUIRE(sm100_fine_supported(*L, d, dtype),
                "fine stage: bf16 needs 64-token cubes and head_dim 64 or 128 (VSA_FINE_FORCE_SIMT for the SIMT path)");
  if (!(flags & VSA_FINE_FORCE_SIMT) && sm100_fine_supported(*L, d, dtype))
    return launch_fine_forward_sm100(*L, bh, d, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags,
                                     out, task_begin, task_end, st);
  VSA_REQUIRE(task_begin == 0 && task_end == bh * L->nc, "fine stage: task ranges need the tcgen05 kernels");
  return launch_fine_forward_simt(*L, bh, d, dtype, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube,
                                  flags, out, st);
}

int vsa_fine_forward(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                     const void* v, const int32_t* sel, int64_t top_k, void* o_fine, float* lse, float* row_max,
                     const void* gc, const void* gf, const float* oc_cube, int32_t flags, void* out, void* stream) {
  VSA_CHECKED(check_layout(L));
  return vsa_fine_forward_range(L, bh, d, dtype, q, k, v, sel, top_k, o_fine, lse, row_max, gc, gf, oc_cube, flags,
                                out, 0, bh * L->nc, stream);
}

int vsa_backward_prologue(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, int32_t raster,
                          const void* dout, const void* gc, const void* gf, const float* oc_cube, const void* o_fine,
                          int32_t adaptation, void* dof, float* delta, float* doc_cube, void* dgc, void* dgf,
                          void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "vsa_backward: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(dout && gc && oc_cube && o_fine && dof && delta && bh >= 1,
              "vsa_backward: missing or mismatched forward artifacts");
  VSA_REQUIRE(gf || adaptation, "vsa_backward: missing fine gate");
  return launch_backward_prologue(*L, bh, d, dtype, raster, dout, gc, gf, oc_cube, o_fine, adaptation, dof, delta,
                                  doc_cube, dgc, dgf, as_stream(stream));
}

int vsa_coarse_backward(const vsa_layout_t* L, int64_t bh, int64_t d, const float* qc, const float* kc,
                        const float* vc, const float* ac, const float* doc_cube, float* dqc, float* dkc, float* dvc,
                        float* scratch, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(ac != nullptr, "coarse_backward: artifacts do not match layout");
  VSA_REQUIRE(qc && kc && vc && doc_cube && dqc && dkc && dvc && scratch && bh >= 1 && d >= 1 && d <= 1024,
              "coarse_backward: null buffer");
  return launch_coarse_backward(*L, bh, d, qc, kc, vc, ac, doc_cube, dqc, dkc, dvc, scratch, as_stream(stream));
}

int vsa_fine_backward_range(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                            const void* v, const void* dof, const float* lse, const float* delta, const int32_t* sel,
                            int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx, const float* dqc,
                            const float* dkc, const float* dvc, int32_t raster, int32_t flags, void* dq, void* dk,
                            void* dv, void* workspace, size_t workspace_bytes, int64_t task_begin, int64_t task_end,
                            void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "fine_backward: unknown dtype");
  VSA_REQUIRE(q && k && v && dof && sel && dq && dk && dv && bh >= 1, "fine_backward: null buffer");
  VSA_REQUIRE(lse && delta, "fine_backward: saved statistics do not match shapes");
  VSA_REQUIRE(selT_offs && selT_idx, "fine_backward: transposed block map required");
  VSA_REQUIRE(top_k >= 1 && top_k <= L->nc, "fine stage: selection does not match shapes");
  VSA_REQUIRE(d >= 1 && L->cube <= 128 && L->cube * d <= 8192, "fine stage: cube*head_dim > 8192 unsupported");
  VSA_REQUIRE(task_begin >= 0 && task_begin < task_end && task_end <= bh * L->nc,
              "fine_backward: task range must be a non-empty part of [0, bh*nc)");
  cudaStream_t st = as_stream(stream);
  if (dtype == VSA_BF16 && !(flags & VSA_FINE_FORCE_SIMT))
    VSA_REQUIRE(sm100_fine_bwd_supported(*L, d, dtype),
                "fine_backward: bf16 needs 64-token cubes and head_dim 64 or 128 (VSA_FINE_FORCE_SIMT for the SIMT path)");
  if (!(flags & VSA_FINE_FORCE_SIMT) && sm100_fine_bwd_supported(*L, d, dtype))
    return launch_fine_backward_sm100(*L, bh, d, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc,
                                      dvc, raster, dq, dk, dv, workspace, workspace_bytes, task_begin, task_end, st);
  VSA_REQUIRE(task_begin == 0 && task_end == bh * L->nc, "fine_backward: task ranges need the tcgen05 kernels");
  return launch_fine_backward_simt(*L, bh, d, dtype, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc,
                                   dkc, dvc, raster, dq, dk, dv, st);
}

int vsa_fine_backward(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* q, const void* k,
                      const void* v, const void* dof, const float* lse, const float* delta, const int32_t* sel,
                      int64_t top_k, const int32_t* selT_offs, const int32_t* selT_idx, const float* dqc,
                      const float* dkc, const float* dvc, int32_t raster, int32_t flags, void* dq, void* dk,
                      void* dv, void* workspace, size_t workspace_bytes, void* stream) {
  VSA_CHECKED(check_layout(L));
  return vsa_fine_backward_range(L, bh, d, dtype, q, k, v, dof, lse, delta, sel, top_k, selT_offs, selT_idx, dqc, dkc,
                                 dvc, raster, flags, dq, dk, dv, workspace, workspace_bytes, 0, bh * L->nc, stream);
}

size_t vsa_fine_backward_workspace_bytes(const vsa_layout_t* L, int64_t bh, int64_t top_k) {
  if (!L || bh < 1 || top_k < 1) return 0;
  return fine_backward_ws_bytes(*L, bh, top_k);
}

int vsa_unpool_max_add(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const void* x_tiled,
                       const float* dxc, int32_t raster, void* dx, void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_CHECKED(check_io(L, bh));
  VSA_REQUIRE(dtype_ok(dtype), "unpool: unknown dtype");
  VSA_REQUIRE(x_tiled && dxc && dx && bh >= 1 && d >= 1 && d <= 1024, "unpool: null buffer");
  return launch_unpool_max_add(*L, bh, d, dtype, x_tiled, dxc, raster, dx, as_stream(stream));
}

int vsa_coarse_backward_tokens(const vsa_layout_t* L, int64_t bh, int64_t d, int32_t dtype, const float* qc,
                               const float* kc, const float* vc, const float* ac, int32_t pool_mode,
                               const void* doc, const void* q_t, const void* k_t, const void* v_t, float* doc_cube,
                               float* dqc, float* dkc, float* dvc, float* scratch, void* dq, void* dk, void* dv,
                               void* stream) {
  VSA_CHECKED(check_layout(L));
  VSA_REQUIRE(dtype_ok(dtype), "coarse_backward: unknown dtype");
  VSA_CHECKED(check_vec_dim(d, dtype));
  VSA_REQUIRE(ac != nullptr, "coarse_backward: artifacts do not match layout");
  VSA_REQUIRE(pool_mode == VSA_POOL_MEAN || pool_mode == VSA_POOL_MAX, "pool_cubes: unknown pool mode");
  VSA_REQUIRE(qc && kc && vc && doc && doc_cube && dqc && dkc && dvc && scratch && dq && dk && dv && bh >= 1,
              "coarse_backward: null buffer");
  VSA_REQUIRE(pool_mode == VSA_POOL_MEAN || (q_t && k_t && v_t), "coarse_backward: max pooling needs q, k, v");
  cudaStream_t st = as_stream(stream);
  // dOc_cube = sum of dOc over each cube's tokens (coarse.hpp:146), sequential fp32 in tile order
  const void* xs[1] = {doc};
  float* pl[1] = {doc_cube};
  VSA_CHECKED(launch_tile_pool(*L, bh, d, dtype, 1, xs, nullptr, pl, kPoolSum, 1, st));
  VSA_CHECKED(launch_coarse_backward(*L, bh, d, qc, kc, vc, ac, doc_cube, dqc, dkc, dvc, scratch, st));
  const float* dc[3] = {dqc, dkc, dvc};
  void* gs[3] = {dq, dk, dv};
  const void* xt[3] = {q_t, k_t, v_t};
  for (int i = 0; i < 3; ++i) {
    if (pool_mode == VSA_POOL_MEAN) {
      VSA_CHECKED(launch_unpool_mean(*L, bh, d, dtype, dc[i], gs[i], st));
    } else {
      const size_t n = size_t(bh) * size_t(L->seq_padded) * size_t(d) * (dtype == VSA_BF16 ? 2 : 4);
      VSA_CHECKED(cuda_status(cudaMemsetAsync(gs[i], 0, n, st), "coarse_backward: zero"));
      VSA_CHECKED(launch_unpool_max_add(*L, bh, d, dtype, xt[i], dc[i], 0, gs[i], st));
    }
  }
  return VSA_OK;
}

}  // extern "C"

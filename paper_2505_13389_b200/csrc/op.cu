// SPDX-License-Identifier: Apache-2.0
// The VSA operator as a device-side context: the native
// orchestration of vsa_forward / vsa_backward (vsa.hpp:89-189) over the stage
// kernels, holding the forward artifacts the backward needs (the VsaOutput of
// vsa.hpp:56-63) resident in HBM.
//
//   forward : [gate GEMM] -> K1+K2 tile+pool -> K3 coarse + top-k (+ transposed map)
//             -> K4+K5 fine + gated combine + untile
//   backward: K6a prologue -> K6d coarse backward -> K6b/K6c fine backward
//             (+ max unpool) -> [gate GEMM backward]
//
// Memory: one block carved into 256-byte aligned buffers, either caller-provided
// (torch's caching allocator from Python) or cudaMalloc'ed by the op. The bf16 dS
// workspace of the dS-materialising backward is attached separately
// (vsa_op_set_workspace); without one the backward recomputes S/dP for dQ.
// Stage timing (vsa_op_timing) records CUDA events between the stages on the
// launch stream for up to kMaxTimed calls and averages them after one final
// synchronisation: no host gaps are timed.
#include <cstring>
#include <vector>

#include "common.cuh"
#include "launch.h"

namespace vsa_host {
namespace {

constexpr int kMaxTimed = 256;  // forward or backward calls timed per session

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Plan {
  size_t q_t, k_t, v_t, qc, kc, vc, ac, oc, sel, selT_offs, selT_idx, bitmap, o_f, lse, dof, delta, doc, dqc, dkc,
      dvc, scratch, gc, gf, dgc, dgf, dz, valid_err, coarse_ws, total;
};

Plan make_plan(const vsa_layout_t& L, const vsa_op_desc_t& D) {
  const size_t bh = size_t(D.batch * D.heads), d = size_t(D.head_dim), nc = size_t(L.nc);
  const size_t Lp = size_t(L.seq_padded), es = D.dtype == VSA_BF16 ? 2 : 4;
  const size_t kmax = size_t(std::max<int64_t>(D.top_k, D.max_sel_k));
  const size_t S_io = D.raster ? size_t(L.seq) : Lp;
  Plan p{};
  size_t off = 0;
  auto take = [&](size_t& field, size_t bytes) {
    field = off;
    off += align256(std::max<size_t>(bytes, 1));
  };
  const bool tiled_copies = D.raster != 0;
  take(p.q_t, tiled_copies ? bh * Lp * d * es : 0);
  take(p.k_t, tiled_copies ? bh * Lp * d * es : 0);
  take(p.v_t, tiled_copies ? bh * Lp * d * es : 0);
  take(p.qc, bh * nc * d * 4);
  take(p.kc, bh * nc * d * 4);
  take(p.vc, bh * nc * d * 4);
  take(p.ac, bh * nc * nc * 4);
  take(p.oc, bh * nc * d * 4);
  take(p.sel, bh * nc * size_t(D.top_k) * 4);
  take(p.selT_offs, bh * (nc + 1) * 4);
  take(p.selT_idx, bh * nc * kmax * 4);
  take(p.bitmap, coarse_bitmap_bytes(L, int64_t(bh)));
  take(p.o_f, bh * Lp * d * es);
  take(p.lse, bh * Lp * 4);
  take(p.dof, bh * Lp * d * es);
  take(p.delta, bh * Lp * 4);
  take(p.doc, bh * nc * d * 4);
  take(p.dqc, bh * nc * d * 4);
  take(p.dkc, bh * nc * d * 4);
  take(p.dvc, bh * nc * d * 4);
  take(p.scratch, bh * nc * nc * 4);
  const bool gates = D.model_dim > 0;
  take(p.gc, gates ? bh * S_io * d * es : 0);
  take(p.gf, gates ? bh * S_io * d * es : 0);
  take(p.dgc, gates ? bh * S_io * d * es : 0);
  take(p.dgf, gates ? bh * S_io * d * es : 0);
  take(p.valid_err, 16);
  take(p.coarse_ws, vsa_coarse_workspace_bytes(&L, int64_t(bh), int64_t(d), D.coarse));
  p.dz = 0;
  p.total = off;
  return p;
}

}  // namespace
}  // namespace vsa_host

struct vsa_op {
  vsa_layout_t layout;       // raster I/O order included (vsa_layout_set_io before create)
  vsa_layout_t gate_layout;  // rows of the gate GEMM: the layout itself (raster) or [B,H,Lp,d] (tiled)
  vsa_op_desc_t desc;
  vsa_host::Plan plan;
  uint8_t* base = nullptr;
  bool owns = false;
  void* ws = nullptr;  // dS workspace
  size_t ws_bytes = 0;
  bool owns_ws = false;
  void* gate_ws = nullptr;  // dz workspace of the gate backward (owned)
  size_t gate_ws_bytes = 0;
  // per-forward state
  const void* q_t = nullptr;
  const void* k_t = nullptr;
  const void* v_t = nullptr;
  const void* gc = nullptr;
  const void* gf = nullptr;
  const int32_t* fine_sel = nullptr;
  int64_t fine_k = 0;
  bool have_fwd = false;
  bool have_prologue = false;
  int32_t last_bwd_used_ws = 0;
  // stage timing: events [call][stage boundary]
  bool timing = false;
  int nf = 0, nb = 0;
  std::vector<cudaEvent_t> ev_f, ev_b;  // kMaxTimed x 4

  template <typename T = void>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(base + off);
  }
  int64_t bh() const { return desc.batch * desc.heads; }
  int64_t t0() const { return desc.task_end ? desc.task_begin : 0; }
  int64_t t1() const { return desc.task_end ? desc.task_end : bh() * layout.nc; }
};

namespace {

using namespace vsa_host;

int check_desc(const vsa_layout_t* L, const vsa_op_desc_t* D) {
  VSA_REQUIRE(L != nullptr && D != nullptr, "vsa_op: null layout / descriptor");
  VSA_REQUIRE(L->nc >= 1 && L->seq_padded == L->nc * L->cube, "layout: not initialised");
  VSA_REQUIRE(D->batch >= 1 && D->heads >= 1 && D->head_dim >= 1, "attention: all dimensions must be >= 1");
  VSA_REQUIRE(D->dtype == VSA_BF16 || D->dtype == VSA_F32, "vsa_op: unknown dtype");
  VSA_REQUIRE(D->top_k >= 1 && D->top_k <= L->nc, "coarse_forward_select: k must be in [1, num_cubes]");
  VSA_REQUIRE(D->max_sel_k >= 0 && D->max_sel_k <= L->nc, "vsa_op: max_sel_k must be in [0, num_cubes]");
  VSA_REQUIRE(D->pool_mode == VSA_POOL_MEAN || D->pool_mode == VSA_POOL_MAX, "pool_cubes: unknown pool mode");
  VSA_REQUIRE(D->activation == VSA_GATE_IDENTITY || D->activation == VSA_GATE_SIGMOID,
              "VsaParams: unknown gate activation");
  VSA_REQUIRE(D->model_dim >= 0, "VsaParams: model_dim must be >= 0");
  VSA_REQUIRE(D->coarse == VSA_COARSE_F32 || D->coarse == VSA_COARSE_BF16, "vsa_op: unknown coarse precision");
  if (D->coarse == VSA_COARSE_BF16)
    VSA_REQUIRE(L->nc % 8 == 0 && D->head_dim % 8 == 0, "vsa_op: the bf16 coarse mode needs nc % 8 == 0");
  if (L->io_order == VSA_IO_SEQ_MAJOR) {
    VSA_REQUIRE(D->raster, "sequence-major I/O needs raster order");
    VSA_REQUIRE(L->io_batch == D->batch && L->io_heads == D->heads, "sequence-major I/O: layout batch/heads mismatch");
  }
  const int64_t ntask = D->batch * D->heads * L->nc;
  VSA_REQUIRE((D->task_begin == 0 && D->task_end == 0) ||
                  (D->task_begin >= 0 && D->task_begin < D->task_end && D->task_end <= ntask),
              "vsa_op: task range must be empty (all) or a non-empty part of [0, B*H*nc)");
  if (D->task_end != 0)
    VSA_REQUIRE(D->dtype == VSA_BF16 && !(D->flags & VSA_OP_FORCE_SIMT) && D->pool_mode == VSA_POOL_MEAN,
                "vsa_op: task ranges need the bf16 tcgen05 kernels and mean pooling");
  if (D->dtype == VSA_BF16 && !(D->flags & VSA_OP_FORCE_SIMT))
    VSA_REQUIRE(L->cube == 64 && (D->head_dim == 64 || D->head_dim == 128),
                "vsa_op: the bf16 tcgen05 path needs 64-token cubes and head_dim 64 or 128 "
                "(VSA_OP_FORCE_SIMT selects the SIMT kernels)");
  return VSA_OK;
}

void record(vsa_op* op, std::vector<cudaEvent_t>& ev, int call, int stage, cudaStream_t st) {
  if (op->timing && call < kMaxTimed) cudaEventRecord(ev[size_t(call) * 4 + stage], st);
}

int fine_flags(const vsa_op* op) { return (op->desc.flags & VSA_OP_FORCE_SIMT) ? VSA_FINE_FORCE_SIMT : 0; }

}  // namespace

extern "C" {

size_t vsa_op_memory_bytes(const vsa_layout_t* layout, const vsa_op_desc_t* desc) {
  if (check_desc(layout, desc) != VSA_OK) return 0;
  return make_plan(*layout, *desc).total;
}

int vsa_op_create(const vsa_layout_t* layout, const vsa_op_desc_t* desc, void* device_memory, size_t bytes,
                  vsa_op_t** out) {
  VSA_REQUIRE(out != nullptr, "vsa_op_create: null output");
  *out = nullptr;
  int rc = check_desc(layout, desc);
  if (rc) return rc;
  auto* op = new vsa_op();
  op->layout = *layout;
  op->desc = *desc;
  op->plan = make_plan(*layout, *desc);
  if (desc->raster) {
    op->gate_layout = *layout;
  } else {  // tile-ordered gates [B, H, Lp, d]: a trivial head-major layout over Lp rows
    vsa_layout_make(1, 1, layout->seq_padded, 1, 1, 1, VSA_PAD_REJECT, &op->gate_layout);
  }
  if (device_memory) {
    if (bytes < op->plan.total) {
      delete op;
      VSA_REQUIRE(false, "vsa_op_create: device memory smaller than vsa_op_memory_bytes");
    }
    op->base = static_cast<uint8_t*>(device_memory);
  } else {
    void* p = nullptr;
    rc = cuda_status(cudaMalloc(&p, op->plan.total), "vsa_op_create: cudaMalloc");
    if (rc) {
      delete op;
      return rc;
    }
    op->base = static_cast<uint8_t*>(p);
    op->owns = true;
  }
  op->ev_f.resize(size_t(kMaxTimed) * 4);
  op->ev_b.resize(size_t(kMaxTimed) * 4);
  for (auto* v : {&op->ev_f, &op->ev_b})
    for (auto& e : *v) cudaEventCreate(&e);
  *out = op;
  return VSA_OK;
}

int vsa_op_destroy(vsa_op_t* op) {
  if (!op) return VSA_OK;
  for (auto* v : {&op->ev_f, &op->ev_b})
    for (auto& e : *v) cudaEventDestroy(e);
  if (op->owns) cudaFree(op->base);
  if (op->owns_ws) cudaFree(op->ws);
  if (op->gate_ws) cudaFree(op->gate_ws);
  delete op;
  return VSA_OK;
}

int vsa_op_buffers(const vsa_op_t* op, vsa_op_buffers_t* b) {
  VSA_REQUIRE(op && b, "vsa_op_buffers: null argument");
  const auto& p = op->plan;
  const bool tiled = op->desc.raster != 0, gates = op->desc.model_dim > 0;
  std::memset(b, 0, sizeof(*b));
  b->base = op->base;
  b->bytes = p.total;
  b->q_t = tiled ? op->at(p.q_t) : nullptr;
  b->k_t = tiled ? op->at(p.k_t) : nullptr;
  b->v_t = tiled ? op->at(p.v_t) : nullptr;
  b->qc = op->at<float>(p.qc);
  b->kc = op->at<float>(p.kc);
  b->vc = op->at<float>(p.vc);
  b->ac = op->at<float>(p.ac);
  b->oc_cube = op->at<float>(p.oc);
  b->sel = op->at<int32_t>(p.sel);
  b->selT_offs = op->at<int32_t>(p.selT_offs);
  b->selT_idx = op->at<int32_t>(p.selT_idx);
  b->o_fine = op->at(p.o_f);
  b->lse = op->at<float>(p.lse);
  b->dof = op->at(p.dof);
  b->delta = op->at<float>(p.delta);
  b->doc_cube = op->at<float>(p.doc);
  b->dqc = op->at<float>(p.dqc);
  b->dkc = op->at<float>(p.dkc);
  b->dvc = op->at<float>(p.dvc);
  b->gc = gates ? op->at(p.gc) : nullptr;
  b->gf = gates ? op->at(p.gf) : nullptr;
  b->dgc = gates ? op->at(p.dgc) : nullptr;
  b->dgf = gates ? op->at(p.dgf) : nullptr;
  b->fine_sel = op->fine_sel;
  b->fine_k = op->fine_k;
  b->bwd_used_workspace = op->last_bwd_used_ws;
  return VSA_OK;
}

int vsa_op_set_workspace(vsa_op_t* op, void* ws, size_t bytes) {
  VSA_REQUIRE(op != nullptr, "vsa_op_set_workspace: null op");
  if (op->owns_ws) cudaFree(op->ws);
  op->owns_ws = false;
  op->ws = ws;
  op->ws_bytes = ws ? bytes : 0;
  return VSA_OK;
}

size_t vsa_op_workspace_bytes(const vsa_op_t* op, int64_t sel_k) {
  if (!op) return 0;
  return vsa_fine_backward_workspace_bytes(&op->layout, op->bh(), sel_k > 0 ? sel_k : op->desc.top_k);
}

int vsa_op_forward_coarse(vsa_op_t* op, const void* q, const void* k, const void* v, const int32_t* sel_override,
                          int64_t sel_k, void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  VSA_REQUIRE(q && k && v, "attention: empty tensors");
  const auto& p = op->plan;
  const auto& D = op->desc;
  const vsa_layout_t* L = &op->layout;
  const int64_t bh = op->bh(), d = D.head_dim;
  cudaStream_t st = as_stream(stream);
  const int call = op->nf;
  record(op, op->ev_f, call, 0, st);
  float* pooled[3] = {op->at<float>(p.qc), op->at<float>(p.kc), op->at<float>(p.vc)};
  int rc;
  if (D.raster) {
    const void* xr[3] = {q, k, v};
    void* xt[3] = {op->at(p.q_t), op->at(p.k_t), op->at(p.v_t)};
    rc = vsa_tile_pool(L, bh, d, D.dtype, 3, xr, xt, pooled, D.pool_mode, stream);
    if (rc) return rc;
    op->q_t = xt[0], op->k_t = xt[1], op->v_t = xt[2];
  } else {
    const void* xs[3] = {q, k, v};
    for (int i = 0; i < 3; ++i) {
      rc = vsa_pool_tiled(L, bh, d, D.dtype, xs[i], pooled[i], D.pool_mode, stream);
      if (rc) return rc;
    }
    op->q_t = q, op->k_t = k, op->v_t = v;
  }
  record(op, op->ev_f, call, 1, st);
  const bool override_sel = sel_override != nullptr;
  if (override_sel) {
    VSA_REQUIRE(sel_k >= 1 && sel_k <= std::max<int64_t>(D.top_k, D.max_sel_k),
                "fine stage: selection k exceeds the operator's max_sel_k");
    // BlockSelection::validate on every fine call (fine.hpp:33): the device check, then
    // one synchronous read of its flag (override maps are a control path)
    int32_t* err = op->at<int32_t>(p.valid_err);
    rc = vsa_validate_selection(sel_override, bh * L->nc, sel_k, L->nc, err, stream);
    if (rc) return rc;
    int32_t herr = 0;
    rc = cuda_status(cudaMemcpyAsync(&herr, err, sizeof(herr), cudaMemcpyDeviceToHost, st), "validate: copy");
    if (rc) return rc;
    rc = cuda_status(cudaStreamSynchronize(st), "validate: sync");
    if (rc) return rc;
    VSA_REQUIRE(herr == 0, "BlockSelection: indices must be strictly ascending and in [0, num_cubes)");
  }
  rc = vsa_coarse_forward_ex(L, bh, d, pooled[0], pooled[1], pooled[2], D.top_k, D.coarse, op->at<float>(p.ac),
                             op->at<float>(p.oc), op->at<int32_t>(p.sel),
                             override_sel ? nullptr : op->at<int32_t>(p.selT_offs),
                             override_sel ? nullptr : op->at<int32_t>(p.selT_idx), op->at(p.bitmap),
                             op->at(p.coarse_ws), stream);
  if (rc) return rc;
  if (override_sel) {
    rc = vsa_selection_transpose(L, bh, sel_override, sel_k, op->at<int32_t>(p.selT_offs),
                                 op->at<int32_t>(p.selT_idx), op->at(p.bitmap), stream);
    if (rc) return rc;
    op->fine_sel = sel_override;
    op->fine_k = sel_k;
  } else {
    op->fine_sel = op->at<int32_t>(p.sel);
    op->fine_k = D.top_k;
  }
  record(op, op->ev_f, call, 2, st);
  return VSA_OK;
}

int vsa_op_forward_fine(vsa_op_t* op, const void* gc, const void* gf, void* out, void* stream) {
  VSA_REQUIRE(op != nullptr && op->q_t != nullptr, "vsa_op: forward_fine before forward_coarse");
  const auto& p = op->plan;
  const auto& D = op->desc;
  VSA_REQUIRE(gc != nullptr && out != nullptr, "vsa_forward: missing coarse gate / output");
  VSA_REQUIRE(gf != nullptr || D.adaptation, "vsa_forward: missing fine gate");
  cudaStream_t st = as_stream(stream);
  const int32_t flags = VSA_FINE_COMBINE | (D.raster ? VSA_FINE_UNTILE : 0) | (D.adaptation ? VSA_FINE_ADAPTATION : 0) |
                        fine_flags(op);
  int rc = vsa_fine_forward_range(&op->layout, op->bh(), D.head_dim, D.dtype, op->q_t, op->k_t, op->v_t,
                                  op->fine_sel, op->fine_k, op->at(p.o_f), op->at<float>(p.lse), nullptr, gc, gf,
                                  op->at<float>(p.oc), flags, out, op->t0(), op->t1(), stream);
  if (rc) return rc;
  op->gc = gc;
  op->gf = gf;
  op->have_fwd = true;
  record(op, op->ev_f, op->nf, 3, st);
  if (op->timing) ++op->nf;
  return VSA_OK;
}

int vsa_op_forward(vsa_op_t* op, const void* q, const void* k, const void* v, const void* gc, const void* gf,
                   const int32_t* sel_override, int64_t sel_k, void* out, void* stream) {
  int rc = vsa_op_forward_coarse(op, q, k, v, sel_override, sel_k, stream);
  if (rc) return rc;
  return vsa_op_forward_fine(op, gc, gf, out, stream);
}

int vsa_op_backward_prologue(vsa_op_t* op, const void* dout, void* dgc, void* dgf, void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  VSA_REQUIRE(op->have_fwd, "vsa_backward: missing or mismatched forward artifacts");
  VSA_REQUIRE(dout != nullptr, "vsa_backward: null dO");
  const auto& p = op->plan;
  const auto& D = op->desc;
  const vsa_layout_t* L = &op->layout;
  const int64_t bh = op->bh(), d = D.head_dim;
  const int32_t raster = D.raster ? 1 : 0;
  cudaStream_t st = as_stream(stream);
  const int call = op->nb;
  record(op, op->ev_b, call, 0, st);
  int rc = vsa_backward_prologue(L, bh, d, D.dtype, raster, dout, op->gc, op->gf, op->at<float>(p.oc),
                                 op->at(p.o_f), D.adaptation, op->at(p.dof), op->at<float>(p.delta),
                                 op->at<float>(p.doc), dgc, D.adaptation ? nullptr : dgf, stream);
  if (rc) return rc;
  if (D.adaptation && dgf) {  // the fine gate is fixed: no gradient (vsa.hpp:147)
    const size_t es = D.dtype == VSA_BF16 ? 2 : 4;
    const size_t n = size_t(bh) * size_t(D.raster ? L->seq : L->seq_padded) * size_t(d) * es;
    rc = cuda_status(cudaMemsetAsync(dgf, 0, n, st), "vsa_backward: zero dGf");
    if (rc) return rc;
  }
  record(op, op->ev_b, call, 1, st);
  rc = vsa_coarse_backward_ex(L, bh, d, op->at<float>(p.qc), op->at<float>(p.kc), op->at<float>(p.vc),
                              op->at<float>(p.ac), op->at<float>(p.doc), op->at<float>(p.dqc), op->at<float>(p.dkc),
                              op->at<float>(p.dvc), op->at<float>(p.scratch), D.coarse, op->at(p.coarse_ws), stream);
  if (rc) return rc;
  record(op, op->ev_b, call, 2, st);
  op->have_prologue = true;
  return VSA_OK;
}

int vsa_op_backward_finish(vsa_op_t* op, void* dq, void* dk, void* dv, void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  VSA_REQUIRE(op->have_prologue, "vsa_backward: finish before the prologue");
  VSA_REQUIRE(dq && dk && dv, "vsa_backward: null gradient buffer");
  const auto& p = op->plan;
  const auto& D = op->desc;
  const vsa_layout_t* L = &op->layout;
  const int64_t bh = op->bh(), d = D.head_dim;
  const int32_t raster = D.raster ? 1 : 0;
  cudaStream_t st = as_stream(stream);
  const bool mean = D.pool_mode == VSA_POOL_MEAN;
  const size_t need = vsa_fine_backward_workspace_bytes(L, bh, op->fine_k);
  const bool use_ws = !(D.flags & VSA_OP_NO_DS_WORKSPACE) && op->ws != nullptr && op->ws_bytes >= need &&
                      D.task_end == 0;
  int rc = vsa_fine_backward_range(L, bh, d, D.dtype, op->q_t, op->k_t, op->v_t, op->at(p.dof), op->at<float>(p.lse),
                                   op->at<float>(p.delta), op->fine_sel, op->fine_k, op->at<int32_t>(p.selT_offs),
                                   op->at<int32_t>(p.selT_idx), mean ? op->at<float>(p.dqc) : nullptr,
                                   mean ? op->at<float>(p.dkc) : nullptr, mean ? op->at<float>(p.dvc) : nullptr,
                                   raster, fine_flags(op), dq, dk, dv, use_ws ? op->ws : nullptr,
                                   use_ws ? op->ws_bytes : 0, op->t0(), op->t1(), stream);
  if (rc) return rc;
  op->last_bwd_used_ws = use_ws ? 1 : 0;
  if (!mean) {  // max pooling: route the cube grads to the first argmax tokens (coarse.hpp:172-176)
    const void* xs[3] = {op->q_t, op->k_t, op->v_t};
    const float* dc[3] = {op->at<float>(p.dqc), op->at<float>(p.dkc), op->at<float>(p.dvc)};
    void* gs[3] = {dq, dk, dv};
    for (int i = 0; i < 3; ++i) {
      rc = vsa_unpool_max_add(L, bh, d, D.dtype, xs[i], dc[i], raster, gs[i], stream);
      if (rc) return rc;
    }
  }
  record(op, op->ev_b, op->nb, 3, st);
  if (op->timing) ++op->nb;
  op->have_prologue = false;
  return VSA_OK;
}

int vsa_op_backward(vsa_op_t* op, const void* dout, void* dq, void* dk, void* dv, void* dgc, void* dgf,
                    void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  VSA_REQUIRE(dout && dq && dk && dv, "vsa_backward: null gradient buffer");
  int rc = vsa_op_backward_prologue(op, dout, dgc, dgf, stream);
  if (rc) return rc;
  return vsa_op_backward_finish(op, dq, dk, dv, stream);
}

int vsa_forward(vsa_op_t* op, const void* hidden, const void* gate_weight, const float* gate_bias, const void* q,
                const void* k, const void* v, const int32_t* sel_override, int64_t sel_k, void* out, void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  const auto& D = op->desc;
  VSA_REQUIRE(D.model_dim > 0, "vsa_forward: the operator was created without model_dim (gate projection)");
  VSA_REQUIRE(D.dtype == VSA_BF16, "vsa_forward: the gate projection runs in bf16 (tcgen05 GEMM)");
  VSA_REQUIRE(hidden && gate_weight, "vsa: hidden states / gate weight missing");
  const auto& p = op->plan;
  int rc = vsa_gate_forward(&op->gate_layout, D.batch, D.heads, D.head_dim, D.model_dim, hidden, gate_weight,
                            gate_bias, D.activation, D.adaptation, op->at(p.gc), op->at(p.gf), stream);
  if (rc) return rc;
  return vsa_op_forward(op, q, k, v, op->at(p.gc), op->at(p.gf), sel_override, sel_k, out, stream);
}

int vsa_backward(vsa_op_t* op, const void* hidden, const void* gate_weight, const void* dout, void* dq, void* dk,
                 void* dv, void* dhidden, float* dgate_weight, float* dgate_bias, void* stream) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  const auto& D = op->desc;
  VSA_REQUIRE(D.model_dim > 0, "vsa_backward: the operator was created without model_dim (gate projection)");
  VSA_REQUIRE(hidden && gate_weight && dhidden && dgate_weight, "vsa_backward: null gate buffer");
  const auto& p = op->plan;
  int rc = vsa_op_backward(op, dout, dq, dk, dv, op->at(p.dgc), op->at(p.dgf), stream);
  if (rc) return rc;
  const size_t wsb = vsa_gate_backward_workspace_bytes(&op->gate_layout, D.batch, D.heads, D.head_dim);
  if (op->gate_ws_bytes < wsb) {
    if (op->gate_ws) cudaFree(op->gate_ws);
    op->gate_ws = nullptr;
    op->gate_ws_bytes = 0;
    rc = cuda_status(cudaMalloc(&op->gate_ws, wsb), "vsa_backward: gate workspace");
    if (rc) return rc;
    op->gate_ws_bytes = wsb;
  }
  return vsa_gate_backward(&op->gate_layout, D.batch, D.heads, D.head_dim, D.model_dim, hidden, gate_weight,
                           op->at(p.gc), op->at(p.gf), op->at(p.dgc), D.adaptation ? nullptr : op->at(p.dgf),
                           D.activation, D.adaptation, op->gate_ws, dhidden, dgate_weight, dgate_bias, stream);
}

int vsa_op_timing(vsa_op_t* op, int32_t enable) {
  VSA_REQUIRE(op != nullptr, "vsa_op: null op");
  op->timing = enable != 0;
  op->nf = op->nb = 0;
  return VSA_OK;
}

int vsa_op_stage_ms(vsa_op_t* op, float* ms, int32_t* calls) {
  VSA_REQUIRE(op && ms, "vsa_op_stage_ms: null argument");
  for (int i = 0; i < VSA_OP_STAGES; ++i) ms[i] = 0.f;
  const int nf = std::min(op->nf, kMaxTimed), nb = std::min(op->nb, kMaxTimed);
  if (calls) calls[0] = nf, calls[1] = nb;
  if (nf) {
    int rc = cuda_status(cudaEventSynchronize(op->ev_f[size_t(nf - 1) * 4 + 3]), "vsa_op_stage_ms");
    if (rc) return rc;
  }
  if (nb) {
    int rc = cuda_status(cudaEventSynchronize(op->ev_b[size_t(nb - 1) * 4 + 3]), "vsa_op_stage_ms");
    if (rc) return rc;
  }
  for (int c = 0; c < nf; ++c)
    for (int s = 0; s < 3; ++s) {
      float t = 0.f;
      cudaEventElapsedTime(&t, op->ev_f[size_t(c) * 4 + s], op->ev_f[size_t(c) * 4 + s + 1]);
      ms[s] += t / float(nf);
    }
  for (int c = 0; c < nb; ++c)
    for (int s = 0; s < 3; ++s) {
      float t = 0.f;
      cudaEventElapsedTime(&t, op->ev_b[size_t(c) * 4 + s], op->ev_b[size_t(c) * 4 + s + 1]);
      ms[3 + s] += t / float(nb);
    }
  return VSA_OK;
}

}  // extern "C"

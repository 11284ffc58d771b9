// SPDX-License-Identifier: Apache-2.0
//
// vsa_b200/vsa.hpp — header-only C++ mirror of the reference API
// (/root/reference/proj/include/vsa/*.hpp) over the C ABI in vsa_b200.h.
//
// Same type and function names, argument meaning and error behaviour as the
// reference (precondition failures throw std::invalid_argument, tensor.hpp:18-20),
// but Eigen-free and executed on the GPU: host tensors are copied to device
// buffers, the libvsa_b200 kernels run, results are copied back. Scalar = float
// runs the fp32 parity mode; Scalar = vsa_b200::bf16 runs the tcgen05 path.
// Link with -lvsa_b200 -lcudart.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "vsa_b200.h"

namespace vsa_b200 {

using Index = std::ptrdiff_t;
using bf16 = __nv_bfloat16;

namespace detail {

inline void require(bool cond, const char* msg) {
  if (!cond) throw std::invalid_argument(msg);
}

inline void check(int rc) {
  if (rc == 0) return;
  if (rc < 0) throw std::invalid_argument(vsa_last_error());
  throw std::runtime_error(std::string("vsa_b200 CUDA error: ") + vsa_last_error());
}

inline void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

template <typename S>
constexpr int32_t dtype_of() {
  static_assert(std::is_same_v<S, float> || std::is_same_v<S, bf16>, "vsa_b200: Scalar must be float or bf16");
  return std::is_same_v<S, float> ? VSA_F32 : VSA_BF16;
}

// RAII device buffer.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n) cuda(cudaMalloc(&p_, n * sizeof(T)));
  }
  DeviceBuffer(const T* host, size_t n) : DeviceBuffer(n) {
    if (n) cuda(cudaMemcpy(p_, host, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      if (p_) cudaFree(p_);
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void to_host(T* dst) const {
    if (n_) cuda(cudaMemcpy(dst, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost));
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

}  // namespace detail

// Multiply-accumulate instrumentation (tensor.hpp:36-39).
struct MacCounter {
  std::uint64_t tiles = 0;
  std::uint64_t macs = 0;
};

// AttnTensor (tensor.hpp:44-123): contiguous [batch, heads, seq, dim] on the host.
template <typename Scalar>
class AttnTensor {
 public:
  AttnTensor() = default;
  AttnTensor(Index batch, Index heads, Index seq, Index dim) : b_(batch), h_(heads), s_(seq), d_(dim) {
    detail::require(batch >= 1 && heads >= 1 && seq >= 1 && dim >= 1, "AttnTensor: all dimensions must be >= 1");
    data_.assign(static_cast<size_t>(batch * heads * seq * dim), Scalar(0.f));
  }
  // Same draw as the reference: one normal_distribution<double> per tensor, flat order (tensor.hpp:62-68).
  static AttnTensor randn(Index batch, Index heads, Index seq, Index dim, std::mt19937_64& rng, double stddev = 1.0) {
    AttnTensor t(batch, heads, seq, dim);
    std::normal_distribution<double> dist(0.0, stddev);
    for (auto& x : t.data_) x = Scalar(static_cast<float>(dist(rng)));
    return t;
  }
  Index batch() const { return b_; }
  Index heads() const { return h_; }
  Index seq() const { return s_; }
  Index dim() const { return d_; }
  Index size() const { return static_cast<Index>(data_.size()); }
  Scalar* data() { return data_.data(); }
  const Scalar* data() const { return data_.data(); }
  Scalar& at(Index b, Index h, Index s, Index d) { return data_[((b * h_ + h) * s_ + s) * d_ + d]; }
  const Scalar& at(Index b, Index h, Index s, Index d) const { return data_[((b * h_ + h) * s_ + s) * d_ + d]; }
  bool same_shape(const AttnTensor& o) const { return b_ == o.b_ && h_ == o.h_ && s_ == o.s_ && d_ == o.d_; }

 private:
  Index b_ = 0, h_ = 0, s_ = 0, d_ = 0;
  std::vector<Scalar> data_;
};

// TileLayout (layout.hpp:14-33). `pad = true` enables the zero-pad extension.
class TileLayout {
 public:
  TileLayout(Index t, Index h, Index w, Index ct, Index ch, Index cw, bool pad = false) {
    detail::check(vsa_layout_make(t, h, w, ct, ch, cw, pad ? VSA_PAD_ZERO : VSA_PAD_REJECT, &raw_));
    tokens_t = t; tokens_h = h; tokens_w = w;
    cube_t = ct; cube_h = ch; cube_w = cw;
    cubes_t = raw_.nt; cubes_h = raw_.nh; cubes_w = raw_.nw;
    cube_size = raw_.cube;
    seq_len = raw_.seq_padded;  // tile-ordered length (== t*h*w unless padded)
    num_cubes = raw_.nc;
  }
  Index tokens_t = 0, tokens_h = 0, tokens_w = 0;
  Index cube_t = 0, cube_h = 0, cube_w = 0;
  Index cubes_t = 0, cubes_h = 0, cubes_w = 0;
  Index cube_size = 0, seq_len = 0, num_cubes = 0;
  const vsa_layout_t* raw() const { return &raw_; }

 private:
  vsa_layout_t raw_{};
};

// flatten_index (layout.cpp:40-42).
inline Index flatten_index(const TileLayout& layout, Index t, Index h, Index w) {
  int64_t out = 0;
  detail::check(vsa_flatten_index(layout.raw(), t, h, w, &out));
  return out;
}

// BlockSelection (selection.hpp:17-56).
class BlockSelection {
 public:
  BlockSelection() = default;
  BlockSelection(Index batch, Index heads, Index num_cubes, Index k) : b_(batch), h_(heads), nc_(num_cubes), k_(k) {
    detail::require(batch >= 1 && heads >= 1 && num_cubes >= 1, "BlockSelection: bad shape");
    detail::require(k >= 1 && k <= num_cubes, "BlockSelection: k must be in [1, num_cubes]");
    idx_.assign(static_cast<size_t>(batch * heads * num_cubes * k), 0);
  }
  static BlockSelection all_cubes(Index batch, Index heads, Index num_cubes) {
    BlockSelection s(batch, heads, num_cubes, num_cubes);
    for (size_t i = 0; i < s.idx_.size(); ++i) s.idx_[i] = static_cast<int32_t>(i % num_cubes);
    return s;
  }
  Index batch() const { return b_; }
  Index heads() const { return h_; }
  Index num_cubes() const { return nc_; }
  Index k() const { return k_; }
  bool empty() const { return idx_.empty(); }
  int32_t* row(Index b, Index h, Index qc) { return idx_.data() + ((b * h_ + h) * nc_ + qc) * k_; }
  const int32_t* row(Index b, Index h, Index qc) const { return idx_.data() + ((b * h_ + h) * nc_ + qc) * k_; }
  int32_t* data() { return idx_.data(); }
  const int32_t* data() const { return idx_.data(); }
  // selection.cpp:24-37 (host check; the device path also validates)
  void validate() const {
    detail::require(!idx_.empty(), "BlockSelection: empty selection");
    for (Index r = 0; r < b_ * h_ * nc_; ++r) {
      int32_t prev = -1;
      for (Index j = 0; j < k_; ++j) {
        const int32_t c = idx_[r * k_ + j];
        detail::require(c >= 0 && c < nc_, "BlockSelection: cube index out of range");
        detail::require(c > prev, "BlockSelection: indices must be strictly ascending");
        prev = c;
      }
    }
  }

 private:
  Index b_ = 0, h_ = 0, nc_ = 0, k_ = 0;
  std::vector<int32_t> idx_;
};

// random_selection (selection.cpp:52-70): identical draws.
inline BlockSelection random_selection(Index batch, Index heads, Index num_cubes, Index k, std::mt19937_64& rng) {
  BlockSelection sel(batch, heads, num_cubes, k);
  std::vector<int32_t> pool(static_cast<size_t>(num_cubes));
  for (Index c = 0; c < num_cubes; ++c) pool[static_cast<size_t>(c)] = static_cast<int32_t>(c);
  for (Index r = 0; r < batch * heads * num_cubes; ++r) {
    for (Index i = 0; i < k; ++i) {
      std::uniform_int_distribution<Index> pick(i, num_cubes - 1);
      std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(pick(rng))]);
    }
    int32_t* dst = sel.data() + r * k;
    std::copy(pool.begin(), pool.begin() + k, dst);
    std::sort(dst, dst + k);
  }
  return sel;
}

enum class PoolMode { kMean, kMax };

// tile / untile (layout.hpp:43-70).
template <typename Scalar>
AttnTensor<Scalar> tile(const TileLayout& layout, const AttnTensor<Scalar>& x) {
  detail::require(x.seq() == layout.raw()->seq, "tile: sequence length does not match layout");
  const Index bh = x.batch() * x.heads();
  detail::DeviceBuffer<Scalar> src(x.data(), x.size());
  AttnTensor<Scalar> out(x.batch(), x.heads(), layout.seq_len, x.dim());
  detail::DeviceBuffer<Scalar> dst(out.size());
  detail::check(vsa_tile(layout.raw(), bh, x.dim(), detail::dtype_of<Scalar>(), src.get(), dst.get(), nullptr));
  dst.to_host(out.data());
  return out;
}
template <typename Scalar>
AttnTensor<Scalar> untile(const TileLayout& layout, const AttnTensor<Scalar>& x) {
  detail::require(x.seq() == layout.seq_len, "untile: sequence length does not match layout");
  const Index bh = x.batch() * x.heads();
  detail::DeviceBuffer<Scalar> src(x.data(), x.size());
  AttnTensor<Scalar> out(x.batch(), x.heads(), layout.raw()->seq, x.dim());
  detail::DeviceBuffer<Scalar> dst(out.size());
  detail::check(vsa_untile(layout.raw(), bh, x.dim(), detail::dtype_of<Scalar>(), src.get(), dst.get(), nullptr));
  dst.to_host(out.data());
  return out;
}

// SoftmaxStats / FineSaved (dense.hpp:53-57, fine.hpp:13-14): [batch*heads, seq].
struct SoftmaxStats {
  std::vector<float> row_max, row_lse;
};
template <typename Scalar>
struct FineResult {
  AttnTensor<Scalar> out;
  SoftmaxStats saved;
};
template <typename Scalar>
struct AttnGrads {
  AttnTensor<Scalar> dq, dk, dv;
};

namespace detail {
template <typename Scalar>
void check_fine(const TileLayout& L, const AttnTensor<Scalar>& q, const AttnTensor<Scalar>& k,
                const AttnTensor<Scalar>& v, const BlockSelection& sel) {
  require(q.size() > 0, "attention: empty tensors");
  require(q.same_shape(k) && q.same_shape(v), "attention: Q, K, V must share one shape");
  require(q.seq() == L.seq_len, "fine stage: sequence length does not match layout");
  require(sel.batch() == q.batch() && sel.heads() == q.heads() && sel.num_cubes() == L.num_cubes,
          "fine stage: selection does not match shapes");
  sel.validate();
}
}  // namespace detail

// fine_forward (fine.hpp:43-99) on tile-ordered tensors.
template <typename Scalar>
FineResult<Scalar> fine_forward(const TileLayout& layout, const AttnTensor<Scalar>& q, const AttnTensor<Scalar>& k,
                                const AttnTensor<Scalar>& v, const BlockSelection& sel, MacCounter* counter = nullptr) {
  detail::check_fine(layout, q, k, v, sel);
  const Index bh = q.batch() * q.heads(), d = q.dim(), n = q.size();
  detail::DeviceBuffer<Scalar> dq(q.data(), n), dk(k.data(), n), dv(v.data(), n), dout(n);
  detail::DeviceBuffer<int32_t> dsel(sel.data(), static_cast<size_t>(bh * layout.num_cubes * sel.k()));
  detail::DeviceBuffer<float> lse(static_cast<size_t>(bh * q.seq())), rmax(static_cast<size_t>(bh * q.seq()));
  // MacCounter (fine.hpp:59-63): the kernels count the tiles they execute on the device
  const std::uint64_t zero = 0;
  detail::DeviceBuffer<std::uint64_t> ctr(counter ? &zero : nullptr, counter ? 1 : 0);
  if (counter) detail::check(vsa_debug_tile_counter(ctr.get()));
  const int rc = vsa_fine_forward(layout.raw(), bh, d, detail::dtype_of<Scalar>(), dq.get(), dk.get(), dv.get(),
                                  dsel.get(), sel.k(), dout.get(), lse.get(), rmax.get(), nullptr, nullptr, nullptr, 0,
                                  nullptr, nullptr);
  if (counter) vsa_debug_tile_counter(nullptr);
  detail::check(rc);
  if (counter) {
    std::uint64_t tiles = 0;
    ctr.to_host(&tiles);
    counter->tiles += tiles;
    counter->macs += tiles * 2ull * static_cast<std::uint64_t>(layout.cube_size * layout.cube_size * d);
  }
  FineResult<Scalar> res{AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d), {}};
  dout.to_host(res.out.data());
  res.saved.row_lse.resize(lse.size());
  res.saved.row_max.resize(rmax.size());
  lse.to_host(res.saved.row_lse.data());
  rmax.to_host(res.saved.row_max.data());
  return res;
}

// fine_backward (fine.hpp:107-204). `out` is the fine forward output (delta = rowsum(dO*O)).
template <typename Scalar>
AttnGrads<Scalar> fine_backward(const TileLayout& layout, const AttnTensor<Scalar>& q, const AttnTensor<Scalar>& k,
                                const AttnTensor<Scalar>& v, const BlockSelection& sel,
                                const AttnTensor<Scalar>& dout, const FineResult<Scalar>& fwd) {
  detail::check_fine(layout, q, k, v, sel);
  detail::require(dout.same_shape(q), "fine_backward: dO shape mismatch");
  const Index bh = q.batch() * q.heads(), d = q.dim(), n = q.size(), nc = layout.num_cubes;
  detail::require(static_cast<Index>(fwd.saved.row_lse.size()) == bh * q.seq(),
                  "fine_backward: saved statistics do not match shapes");
  const int32_t dt = detail::dtype_of<Scalar>();
  detail::DeviceBuffer<Scalar> dq_(q.data(), n), dk_(k.data(), n), dv_(v.data(), n), ddo(dout.data(), n),
      dof(n), dout_f(fwd.out.data(), n), gq(n), gk(n), gv(n);
  detail::DeviceBuffer<int32_t> dsel(sel.data(), static_cast<size_t>(bh * nc * sel.k()));
  detail::DeviceBuffer<float> lse(fwd.saved.row_lse.data(), fwd.saved.row_lse.size()), delta(bh * q.seq()),
      doc(bh * nc * d), zoc(bh * nc * d);
  std::vector<Scalar> ones_h(static_cast<size_t>(n), Scalar(1.f));
  detail::DeviceBuffer<Scalar> ones(ones_h.data(), ones_h.size());
  detail::cuda(cudaMemset(zoc.get(), 0, zoc.size() * sizeof(float)));
  detail::DeviceBuffer<int32_t> offs(static_cast<size_t>(bh * (nc + 1))), idx(static_cast<size_t>(bh * nc * sel.k()));
  detail::DeviceBuffer<uint8_t> bitmap(vsa_coarse_bitmap_bytes(layout.raw(), bh));
  detail::check(vsa_selection_transpose(layout.raw(), bh, dsel.get(), sel.k(), offs.get(), idx.get(), bitmap.get(),
                                        nullptr));
  detail::check(vsa_backward_prologue(layout.raw(), bh, d, dt, 0, ddo.get(), ones.get(), nullptr, zoc.get(),
                                      dout_f.get(), 1, dof.get(), delta.get(), doc.get(), nullptr, nullptr, nullptr));
  const size_t wsb = vsa_fine_backward_workspace_bytes(layout.raw(), bh, sel.k());
  detail::DeviceBuffer<uint8_t> ws(wsb);
  detail::check(vsa_fine_backward(layout.raw(), bh, d, dt, dq_.get(), dk_.get(), dv_.get(), dof.get(), lse.get(),
                                  delta.get(), dsel.get(), sel.k(), offs.get(), idx.get(), nullptr, nullptr, nullptr, 0,
                                  0, gq.get(), gk.get(), gv.get(), ws.get(), wsb, nullptr));
  AttnGrads<Scalar> g{AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d),
                      AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d),
                      AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d)};
  gq.to_host(g.dq.data());
  gk.to_host(g.dk.data());
  gv.to_host(g.dv.data());
  return g;
}

// CoarseArtifacts (coarse.hpp:18-25) with Oc at cube level.
struct CoarseArtifacts {
  std::vector<float> qc, kc, vc, ac, oc_cube;
  BlockSelection sel;
  PoolMode pool = PoolMode::kMean;
};

// coarse_forward_select (coarse.hpp:71-117) on tile-ordered tensors.
template <typename Scalar>
CoarseArtifacts coarse_forward_select(const TileLayout& layout, const AttnTensor<Scalar>& q,
                                      const AttnTensor<Scalar>& k, const AttnTensor<Scalar>& v, Index top_k,
                                      PoolMode mode = PoolMode::kMean) {
  detail::require(q.size() > 0, "attention: empty tensors");
  detail::require(q.same_shape(k) && q.same_shape(v), "attention: Q, K, V must share one shape");
  detail::require(q.seq() == layout.seq_len, "coarse_forward_select: shape/layout mismatch");
  detail::require(top_k >= 1 && top_k <= layout.num_cubes, "coarse_forward_select: k must be in [1, num_cubes]");
  const Index bh = q.batch() * q.heads(), d = q.dim(), nc = layout.num_cubes, n = q.size();
  const int32_t dt = detail::dtype_of<Scalar>();
  const int32_t pm = mode == PoolMode::kMean ? VSA_POOL_MEAN : VSA_POOL_MAX;
  detail::DeviceBuffer<Scalar> dq(q.data(), n), dk(k.data(), n), dv(v.data(), n);
  detail::DeviceBuffer<float> qc(bh * nc * d), kc(bh * nc * d), vc(bh * nc * d), ac(bh * nc * nc), oc(bh * nc * d);
  detail::check(vsa_pool_tiled(layout.raw(), bh, d, dt, dq.get(), qc.get(), pm, nullptr));
  detail::check(vsa_pool_tiled(layout.raw(), bh, d, dt, dk.get(), kc.get(), pm, nullptr));
  detail::check(vsa_pool_tiled(layout.raw(), bh, d, dt, dv.get(), vc.get(), pm, nullptr));
  CoarseArtifacts art;
  art.pool = mode;
  art.sel = BlockSelection(q.batch(), q.heads(), nc, top_k);
  detail::DeviceBuffer<int32_t> sel(art.sel.batch() * art.sel.heads() * nc * top_k);
  detail::check(vsa_coarse_forward(layout.raw(), bh, d, qc.get(), kc.get(), vc.get(), top_k, ac.get(), oc.get(),
                                   sel.get(), nullptr, nullptr, nullptr, nullptr));
  art.qc.resize(qc.size()); art.kc.resize(kc.size()); art.vc.resize(vc.size());
  art.ac.resize(ac.size()); art.oc_cube.resize(oc.size());
  qc.to_host(art.qc.data()); kc.to_host(art.kc.data()); vc.to_host(art.vc.data());
  ac.to_host(art.ac.data()); oc.to_host(art.oc_cube.data());
  sel.to_host(art.sel.data());
  return art;
}

// fine_backward with the reference signature (fine.hpp:107-111): only the saved
// softmax statistics are given, so the fine output (needed for delta = rowsum(dO * O))
// is recomputed by one fine forward on the device.
template <typename Scalar>
AttnGrads<Scalar> fine_backward(const TileLayout& layout, const AttnTensor<Scalar>& q, const AttnTensor<Scalar>& k,
                                const AttnTensor<Scalar>& v, const BlockSelection& sel,
                                const AttnTensor<Scalar>& dout, const SoftmaxStats& saved) {
  FineResult<Scalar> fwd = fine_forward(layout, q, k, v, sel);
  detail::require(saved.row_lse.size() == fwd.saved.row_lse.size(),
                  "fine_backward: saved statistics do not match shapes");
  fwd.saved.row_lse = saved.row_lse;  // the caller's lse drives the backward, as in the reference
  return fine_backward(layout, q, k, v, sel, dout, fwd);
}

// pool_cubes (coarse.hpp:47-65) on a tile-ordered tensor -> fp32 [B, H, nc, d].
template <typename Scalar>
AttnTensor<float> pool_cubes(const TileLayout& layout, const AttnTensor<Scalar>& x, PoolMode mode = PoolMode::kMean) {
  detail::require(x.seq() == layout.seq_len, "pool_cubes: sequence length does not match layout");
  const Index bh = x.batch() * x.heads();
  detail::DeviceBuffer<Scalar> dx(x.data(), x.size());
  AttnTensor<float> out(x.batch(), x.heads(), layout.num_cubes, x.dim());
  detail::DeviceBuffer<float> dp(out.size());
  detail::check(vsa_pool_tiled(layout.raw(), bh, x.dim(), detail::dtype_of<Scalar>(), dx.get(), dp.get(),
                               mode == PoolMode::kMean ? VSA_POOL_MEAN : VSA_POOL_MAX, nullptr));
  dp.to_host(out.data());
  return out;
}

// coarse_backward (coarse.hpp:124-184): token-level dOc (tile-ordered) -> (dq, dk, dv).
template <typename Scalar>
AttnGrads<Scalar> coarse_backward(const CoarseArtifacts& art, const TileLayout& layout,
                                  const AttnTensor<Scalar>& doc, const AttnTensor<Scalar>& q,
                                  const AttnTensor<Scalar>& k, const AttnTensor<Scalar>& v) {
  detail::require(doc.same_shape(q), "coarse_backward: dOc shape mismatch");
  const Index bh = q.batch() * q.heads(), d = q.dim(), nc = layout.num_cubes, n = q.size();
  detail::require(static_cast<Index>(art.ac.size()) == bh * nc * nc, "coarse_backward: artifacts do not match layout");
  const int32_t dt = detail::dtype_of<Scalar>();
  detail::DeviceBuffer<float> qc(art.qc.data(), art.qc.size()), kc(art.kc.data(), art.kc.size()),
      vc(art.vc.data(), art.vc.size()), ac(art.ac.data(), art.ac.size()), docc(bh * nc * d), dqc(bh * nc * d),
      dkc(bh * nc * d), dvc(bh * nc * d), scratch(bh * nc * nc);
  detail::DeviceBuffer<Scalar> ddoc(doc.data(), n), dq_(q.data(), n), dk_(k.data(), n), dv_(v.data(), n), gq(n),
      gk(n), gv(n);
  detail::check(vsa_coarse_backward_tokens(layout.raw(), bh, d, dt, qc.get(), kc.get(), vc.get(), ac.get(),
                                           art.pool == PoolMode::kMean ? VSA_POOL_MEAN : VSA_POOL_MAX, ddoc.get(),
                                           dq_.get(), dk_.get(), dv_.get(), docc.get(), dqc.get(), dkc.get(),
                                           dvc.get(), scratch.get(), gq.get(), gk.get(), gv.get(), nullptr));
  AttnGrads<Scalar> g{AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d),
                      AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d),
                      AttnTensor<Scalar>(q.batch(), q.heads(), q.seq(), d)};
  gq.to_host(g.dq.data());
  gk.to_host(g.dk.data());
  gv.to_host(g.dv.data());
  return g;
}

// ============================================================================ the operator
enum class GateActivation { kIdentity, kSigmoid };  // vsa.hpp:9

// VsaParams (vsa.hpp:16-52). gate_weight is row-major [model_dim, 2*heads*head_dim] on the
// host; the gate projection runs on the tcgen05 GEMM in bf16.
template <typename Scalar>
struct VsaParams {
  Index model_dim = 0, cols = 0;
  std::vector<float> gate_weight;  // [model_dim][cols]
  std::vector<float> gate_bias;    // empty or [cols]
  Index top_k = 1;
  PoolMode pool = PoolMode::kMean;
  GateActivation activation = GateActivation::kIdentity;
  bool adaptation = false;

  // random_init (vsa.hpp:25-32): the reference's draws (randn_matrix, tensor.hpp:126-133).
  static VsaParams random_init(Index model_dim, Index heads, Index head_dim, Index top_k, std::mt19937_64& rng) {
    VsaParams p;
    p.model_dim = model_dim;
    p.cols = 2 * heads * head_dim;
    p.gate_weight.resize(static_cast<size_t>(model_dim * p.cols));
    std::normal_distribution<double> dist(0.0, 1.0 / std::sqrt(static_cast<double>(model_dim)));
    for (auto& w : p.gate_weight) w = static_cast<float>(static_cast<Scalar>(static_cast<float>(dist(rng))));
    p.top_k = top_k;
    return p;
  }
  // adaptation_init (vsa.hpp:35-42): zero weights, fine gate fixed to one, k = all cubes.
  static VsaParams adaptation_init(Index model_dim, Index heads, Index head_dim, Index num_cubes) {
    VsaParams p;
    p.model_dim = model_dim;
    p.cols = 2 * heads * head_dim;
    p.gate_weight.assign(static_cast<size_t>(model_dim * p.cols), 0.f);
    p.top_k = num_cubes;
    p.adaptation = true;
    return p;
  }
  void check(Index md, Index heads, Index head_dim) const {
    detail::require(model_dim == md && cols == 2 * heads * head_dim &&
                        static_cast<Index>(gate_weight.size()) == md * cols,
                    "VsaParams: gate projection must map model_dim -> 2*heads*head_dim");
    detail::require(gate_bias.empty() || static_cast<Index>(gate_bias.size()) == cols,
                    "VsaParams: gate bias size mismatch");
    detail::require(top_k >= 1, "VsaParams: k must be >= 1");
  }
};

namespace detail {
// The device operator context (vsa_op_t) with RAII.
struct OpHandle {
  vsa_op_t* op = nullptr;
  DeviceBuffer<uint8_t> ws;
  // the forward's device inputs (the context's artifacts point into q/k/v; the backward
  // reuses them, as the reference's vsa_backward receives the same q, k, v, hidden)
  DeviceBuffer<bf16> hidden, q, k, v, w;
  DeviceBuffer<float> bias;
  ~OpHandle() {
    if (op) vsa_op_destroy(op);
  }
};
}  // namespace detail

// VsaOutput (vsa.hpp:56-63): host copies of the output and artifacts; the device
// context `ctx` keeps them resident for vsa_backward.
template <typename Scalar>
struct VsaOutput {
  AttnTensor<Scalar> out;
  CoarseArtifacts coarse;
  FineResult<Scalar> fine;
  AttnTensor<Scalar> gate_coarse, gate_fine;
  BlockSelection fine_sel;
  std::shared_ptr<detail::OpHandle> ctx;
};

// VsaGrads (vsa.hpp:65-71).
template <typename Scalar>
struct VsaGrads {
  AttnTensor<Scalar> dq, dk, dv;
  AttnTensor<Scalar> dhidden;          // [batch, 1, seq, model_dim]
  std::vector<float> dgate_weight;     // [model_dim][2*heads*head_dim]
  std::vector<float> dgate_bias;       // empty or [2*heads*head_dim]
};

namespace detail {
template <typename Scalar>
void check_hidden(const AttnTensor<Scalar>& hidden, const AttnTensor<Scalar>& q) {  // vsa.hpp:75-80
  require(hidden.heads() == 1, "vsa: hidden states are [batch, 1, seq, model_dim]");
  require(hidden.batch() == q.batch() && hidden.seq() == q.seq(), "vsa: hidden states do not match Q/K/V shapes");
}
inline std::vector<bf16> to_bf16(const std::vector<float>& x) {
  std::vector<bf16> y(x.size());
  for (size_t i = 0; i < x.size(); ++i) y[i] = __float2bfloat16(x[i]);
  return y;
}
}  // namespace detail

// vsa_forward (vsa.hpp:89-122): q, k, v, hidden tile-ordered. Scalar = bf16 (the gate
// projection is a bf16 tcgen05 GEMM; the attention stages run the tcgen05 path).
template <typename Scalar>
VsaOutput<Scalar> vsa_forward(const TileLayout& layout, const AttnTensor<Scalar>& hidden, const AttnTensor<Scalar>& q,
                              const AttnTensor<Scalar>& k, const AttnTensor<Scalar>& v,
                              const VsaParams<Scalar>& params, const BlockSelection* sel_override = nullptr) {
  static_assert(std::is_same_v<Scalar, bf16>, "vsa_b200::vsa_forward: the gate projection runs in bf16");
  detail::require(q.size() > 0, "attention: empty tensors");
  detail::require(q.same_shape(k) && q.same_shape(v), "attention: Q, K, V must share one shape");
  detail::check_hidden(hidden, q);
  const Index B = q.batch(), H = q.heads(), S = q.seq(), d = q.dim(), nc = layout.num_cubes, md = hidden.dim();
  detail::require(S == layout.seq_len, "vsa: sequence length does not match layout");
  params.check(md, H, d);
  detail::require(params.top_k <= nc, "coarse_forward_select: k must be in [1, num_cubes]");
  if (sel_override) {
    detail::require(sel_override->batch() == B && sel_override->heads() == H && sel_override->num_cubes() == nc,
                    "fine stage: selection does not match shapes");
    sel_override->validate();
  }
  vsa_op_desc_t desc{};
  desc.batch = B;
  desc.heads = H;
  desc.head_dim = d;
  desc.top_k = params.top_k;
  desc.max_sel_k = sel_override ? sel_override->k() : 0;
  desc.model_dim = md;
  desc.dtype = VSA_BF16;
  desc.pool_mode = params.pool == PoolMode::kMean ? VSA_POOL_MEAN : VSA_POOL_MAX;
  desc.activation = params.activation == GateActivation::kSigmoid ? VSA_GATE_SIGMOID : VSA_GATE_IDENTITY;
  desc.adaptation = params.adaptation ? 1 : 0;
  desc.raster = 0;  // the reference contract: tile-ordered tensors (vsa.hpp:86)
  VsaOutput<Scalar> res;
  res.ctx = std::make_shared<detail::OpHandle>();
  detail::check(vsa_op_create(layout.raw(), &desc, nullptr, 0, &res.ctx->op));
  const size_t n = static_cast<size_t>(q.size());
  auto& c = *res.ctx;
  c.hidden = detail::DeviceBuffer<bf16>(hidden.data(), static_cast<size_t>(hidden.size()));
  c.q = detail::DeviceBuffer<bf16>(q.data(), n);
  c.k = detail::DeviceBuffer<bf16>(k.data(), n);
  c.v = detail::DeviceBuffer<bf16>(v.data(), n);
  const auto wb = detail::to_bf16(params.gate_weight);
  c.w = detail::DeviceBuffer<bf16>(wb.data(), wb.size());
  c.bias = detail::DeviceBuffer<float>(params.gate_bias.data(), params.gate_bias.size());
  detail::DeviceBuffer<Scalar> dout(n);
  detail::DeviceBuffer<int32_t> dsel(sel_override ? sel_override->data() : nullptr,
                                     sel_override ? static_cast<size_t>(B * H * nc * sel_override->k()) : 0);
  detail::check(::vsa_forward(c.op, c.hidden.get(), c.w.get(), params.gate_bias.empty() ? nullptr : c.bias.get(),
                            c.q.get(), c.k.get(), c.v.get(), sel_override ? dsel.get() : nullptr,
                            sel_override ? sel_override->k() : 0, dout.get(), nullptr));
  detail::cuda(cudaDeviceSynchronize());
  vsa_op_buffers_t b{};
  detail::check(vsa_op_buffers(res.ctx->op, &b));
  auto d2h = [](void* dst, const void* src, size_t bytes) {
    detail::cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  };
  res.out = AttnTensor<Scalar>(B, H, S, d);
  dout.to_host(res.out.data());
  const size_t cub = static_cast<size_t>(B * H * nc * d), es = sizeof(Scalar);
  res.coarse.pool = params.pool;
  res.coarse.qc.resize(cub); res.coarse.kc.resize(cub); res.coarse.vc.resize(cub); res.coarse.oc_cube.resize(cub);
  res.coarse.ac.resize(static_cast<size_t>(B * H * nc * nc));
  d2h(res.coarse.qc.data(), b.qc, cub * 4); d2h(res.coarse.kc.data(), b.kc, cub * 4);
  d2h(res.coarse.vc.data(), b.vc, cub * 4); d2h(res.coarse.oc_cube.data(), b.oc_cube, cub * 4);
  d2h(res.coarse.ac.data(), b.ac, res.coarse.ac.size() * 4);
  res.coarse.sel = BlockSelection(B, H, nc, params.top_k);
  d2h(res.coarse.sel.data(), b.sel, static_cast<size_t>(B * H * nc * params.top_k) * 4);
  res.fine.out = AttnTensor<Scalar>(B, H, S, d);
  d2h(res.fine.out.data(), b.o_fine, n * es);
  res.fine.saved.row_lse.resize(static_cast<size_t>(B * H * S));
  d2h(res.fine.saved.row_lse.data(), b.lse, res.fine.saved.row_lse.size() * 4);
  res.gate_coarse = AttnTensor<Scalar>(B, H, S, d);
  res.gate_fine = AttnTensor<Scalar>(B, H, S, d);
  d2h(res.gate_coarse.data(), b.gc, n * es);
  d2h(res.gate_fine.data(), b.gf, n * es);
  res.fine_sel = sel_override ? *sel_override : res.coarse.sel;
  return res;
}

// vsa_backward (vsa.hpp:129-189) on the device artifacts of `fwd`.
template <typename Scalar>
VsaGrads<Scalar> vsa_backward(const TileLayout& layout, const VsaOutput<Scalar>& fwd, const AttnTensor<Scalar>& hidden,
                              const AttnTensor<Scalar>& q, const AttnTensor<Scalar>& k, const AttnTensor<Scalar>& v,
                              const VsaParams<Scalar>& params, const AttnTensor<Scalar>& dout) {
  detail::require(q.same_shape(k) && q.same_shape(v), "attention: Q, K, V must share one shape");
  detail::check_hidden(hidden, q);
  detail::require(dout.same_shape(q), "vsa_backward: dO shape mismatch");
  detail::require(fwd.ctx && fwd.ctx->op && fwd.out.same_shape(q) && !fwd.fine_sel.empty(),
                  "vsa_backward: missing or mismatched forward artifacts");
  const Index B = q.batch(), H = q.heads(), S = q.seq(), d = q.dim(), md = hidden.dim();
  params.check(md, H, d);
  (void)layout;
  vsa_op_t* op = fwd.ctx->op;
  const size_t wsb = vsa_op_workspace_bytes(op, fwd.fine_sel.k());
  if (fwd.ctx->ws.size() < wsb) {
    fwd.ctx->ws = detail::DeviceBuffer<uint8_t>(wsb);
    detail::check(vsa_op_set_workspace(op, fwd.ctx->ws.get(), wsb));
  }
  const size_t n = static_cast<size_t>(q.size());
  auto& c = *fwd.ctx;
  detail::DeviceBuffer<Scalar> ddo(dout.data(), n), gq(n), gk(n), gv(n), gh(static_cast<size_t>(hidden.size()));
  detail::DeviceBuffer<float> gW(params.gate_weight.size()), gb(params.gate_bias.size());
  detail::check(::vsa_backward(op, c.hidden.get(), c.w.get(), ddo.get(), gq.get(), gk.get(), gv.get(), gh.get(),
                             gW.get(), params.gate_bias.empty() ? nullptr : gb.get(), nullptr));
  detail::cuda(cudaDeviceSynchronize());
  VsaGrads<Scalar> g{AttnTensor<Scalar>(B, H, S, d), AttnTensor<Scalar>(B, H, S, d), AttnTensor<Scalar>(B, H, S, d),
                     AttnTensor<Scalar>(B, 1, S, md), std::vector<float>(params.gate_weight.size()), {}};
  gq.to_host(g.dq.data());
  gk.to_host(g.dk.data());
  gv.to_host(g.dv.data());
  gh.to_host(g.dhidden.data());
  gW.to_host(g.dgate_weight.data());
  if (!params.gate_bias.empty()) {
    g.dgate_bias.resize(params.gate_bias.size());
    gb.to_host(g.dgate_bias.data());
  }
  return g;
}

}  // namespace vsa_b200

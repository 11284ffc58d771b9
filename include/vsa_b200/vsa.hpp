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
  if (counter) {
    counter->tiles += static_cast<std::uint64_t>(bh * layout.num_cubes * sel.k());
    counter->macs += static_cast<std::uint64_t>(bh * layout.num_cubes * sel.k()) * 2ull * layout.cube_size *
                     layout.cube_size * static_cast<std::uint64_t>(d);
  }
  detail::DeviceBuffer<Scalar> dq(q.data(), n), dk(k.data(), n), dv(v.data(), n), dout(n);
  detail::DeviceBuffer<int32_t> dsel(sel.data(), static_cast<size_t>(bh * layout.num_cubes * sel.k()));
  detail::DeviceBuffer<float> lse(static_cast<size_t>(bh * q.seq())), rmax(static_cast<size_t>(bh * q.seq()));
  detail::check(vsa_fine_forward(layout.raw(), bh, d, detail::dtype_of<Scalar>(), dq.get(), dk.get(), dv.get(),
                                 dsel.get(), sel.k(), dout.get(), lse.get(), rmax.get(), nullptr, nullptr, nullptr, 0,
                                 nullptr, nullptr));
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

}  // namespace vsa_b200

// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — NOT PART OF THE PRODUCT.
//
// CPU restatement of the reference VSA operator (/root/reference/proj), used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
// checker. The reference itself cannot be compiled here (it needs Eigen3,
// absent from the image: proj/include/vsa/tensor.hpp:4, proj/CMakeLists.txt:12),
// so every Eigen expression is restated as plain loops with ONE fixed
// evaluation order (the "canonical order"):
//   * reductions run sequentially in ascending index order;
//   * dot products are fma chains  acc = fma(a_i, b_i, acc), i ascending;
//   * exp() on the coarse path is canon_exp (explicit-fma double polynomial),
//     rounded to float for Scalar=float, so a GPU kernel can replicate the
//     cube-level probabilities — and therefore the Top-K block map — bit-exactly.
// Build flags: -O3 -fopenmp -ffp-contract=off (no implicit contraction).
//
// Parity pinning: tests/test_oracle_*.py run every known-answer test and
// property test of the reference suite for this path (proj/tests/test_tiling.cpp,
// test_dense.cpp, test_coarse.cpp, test_fine.cpp, test_vsa.cpp, verify.hpp,
// gradcheck.hpp) against this file, with the reference's seeds and tolerances.

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using Index = std::ptrdiff_t;  // Eigen::Index (tensor.hpp:14)

static thread_local std::string g_err;

inline void require(bool cond, const char* msg) {  // tensor.hpp:18-20
  if (!cond) throw std::invalid_argument(msg);
}

// ---------------------------------------------------------------------------
// canonical exp: double-precision Cody-Waite reduction + degree-13 Taylor
// polynomial, every step an explicit IEEE op (fma / mul / add), so the same
// code gives identical bits on any IEEE host or device.
double canon_exp(double x) {
  if (std::isnan(x)) return x;
  if (x > 709.782712893384) return std::numeric_limits<double>::infinity();
  if (x < -745.1332191019412) return 0.0;
  const double log2e = 1.4426950408889634;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double kd = std::nearbyint(x * log2e);
  double r = std::fma(-kd, ln2_hi, x);
  r = std::fma(-kd, ln2_lo, r);
  // Taylor coefficients 1/n!, n = 13 .. 0
  static const double c[14] = {1.6059043836821613e-10, 2.08767569878681e-09,  2.505210838544172e-08,
                               2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
                               1.984126984126984e-04,  1.388888888888889e-03,  8.333333333333333e-03,
                               4.1666666666666664e-02, 1.6666666666666666e-01, 0.5,
                               1.0,                    1.0};
  double p = c[0];
  for (int i = 1; i < 14; ++i) p = std::fma(p, r, c[i]);
  return std::scalbn(p, static_cast<int>(kd));
}

template <typename S>
inline S coarse_exp(S x);
template <>
inline float coarse_exp<float>(float x) {
  return static_cast<float>(canon_exp(static_cast<double>(x)));
}
template <>
inline double coarse_exp<double>(double x) {
  return std::exp(x);
}

// ---------------------------------------------------------------------------
// TileLayout (layout.hpp:14-33, layout.cpp:6-31)
struct Layout {
  Index t = 0, h = 0, w = 0, ct = 0, ch = 0, cw = 0;
  Index nt = 0, nh = 0, nw = 0, cube = 0, seq = 0, nc = 0;
  std::vector<Index> tile_of_raster, raster_of_tile;
};

Layout make_layout(Index t, Index h, Index w, Index ct, Index ch, Index cw) {
  require(t >= 1 && h >= 1 && w >= 1, "TileLayout: token extents must be >= 1");
  require(ct >= 1 && ch >= 1 && cw >= 1, "TileLayout: cube extents must be >= 1");
  require(t % ct == 0 && h % ch == 0 && w % cw == 0,
          "TileLayout: token extents must be integer multiples of cube extents");
  Layout L;
  L.t = t; L.h = h; L.w = w; L.ct = ct; L.ch = ch; L.cw = cw;
  L.nt = t / ct; L.nh = h / ch; L.nw = w / cw;
  L.cube = ct * ch * cw;
  L.seq = t * h * w;
  L.nc = L.seq / L.cube;
  L.tile_of_raster.assign(L.seq, 0);
  L.raster_of_tile.assign(L.seq, 0);
  Index r = 0;
  for (Index a = 0; a < t; ++a)
    for (Index b = 0; b < h; ++b)
      for (Index c = 0; c < w; ++c, ++r) {
        const Index cube_rank = ((a / ct) * L.nh + b / ch) * L.nw + c / cw;
        const Index within = ((a % ct) * ch + b % ch) * cw + c % cw;
        const Index pos = cube_rank * L.cube + within;
        L.tile_of_raster[r] = pos;
        L.raster_of_tile[pos] = r;
      }
  return L;
}

// raster_index / flatten_index (layout.cpp:33-42)
Index raster_index(const Layout& L, Index t, Index h, Index w) {
  require(t >= 0 && t < L.t && h >= 0 && h < L.h && w >= 0 && w < L.w, "raster_index: coordinate out of range");
  return (t * L.h + h) * L.w + w;
}

// tile / untile (layout.hpp:43-70): seq-axis permutation of [B,H,L,d]
template <typename S>
void tile(const Layout& L, const S* x, Index bh, Index d, S* out, bool inverse) {
  for (Index u = 0; u < bh; ++u) {
    const S* src = x + u * L.seq * d;
    S* dst = out + u * L.seq * d;
    for (Index r = 0; r < L.seq; ++r) {
      const Index p = L.tile_of_raster[r];
      if (!inverse)
        std::memcpy(dst + p * d, src + r * d, sizeof(S) * d);
      else
        std::memcpy(dst + r * d, src + p * d, sizeof(S) * d);
    }
  }
}

// ---------------------------------------------------------------------------
// small dense helpers, canonical order
template <typename S>
inline S dot(const S* a, const S* b, Index n) {
  S acc = S(0);
  for (Index i = 0; i < n; ++i) acc = std::fma(a[i], b[i], acc);
  return acc;
}

// C[m x n] = A[m x k] * B[n x k]^T  (row-major), canonical fma chains: every
// C[i][j] is fma-accumulated over k ascending from 0 — bit-identical to
// dot(A_i, B_j), but laid out i-k-j over B^T so the j loop vectorises.
template <typename S>
void gemm_abt(const S* A, const S* B, S* C, Index m, Index n, Index k) {
  std::vector<S> bt(static_cast<size_t>(k * n));
  for (Index j = 0; j < n; ++j)
    for (Index p = 0; p < k; ++p) bt[p * n + j] = B[j * k + p];
  for (Index i = 0; i < m; ++i) {
    S* c = C + i * n;
    std::fill(c, c + n, S(0));
    for (Index p = 0; p < k; ++p) {
      const S a = A[i * k + p];
      const S* b = bt.data() + p * n;
      for (Index j = 0; j < n; ++j) c[j] = std::fma(a, b[j], c[j]);
    }
  }
}
// C[m x n] (+)= A[m x k] * B[k x n]; sum over k ascending per element.
template <typename S>
void gemm_ab(const S* A, const S* B, S* C, Index m, Index n, Index k, bool accumulate) {
  for (Index i = 0; i < m; ++i) {
    S* c = C + i * n;
    if (!accumulate) std::fill(c, c + n, S(0));
    for (Index p = 0; p < k; ++p) {
      const S a = A[i * k + p];
      const S* b = B + p * n;
      for (Index j = 0; j < n; ++j) c[j] = std::fma(a, b[j], c[j]);
    }
  }
}
// C[m x n] (+)= A[k x m]^T * B[k x n]
template <typename S>
void gemm_atb(const S* A, const S* B, S* C, Index m, Index n, Index k, bool accumulate) {
  if (!accumulate) std::fill(C, C + m * n, S(0));
  for (Index p = 0; p < k; ++p)
    for (Index i = 0; i < m; ++i) {
      const S a = A[p * m + i];
      const S* b = B + p * n;
      S* c = C + i * n;
      for (Index j = 0; j < n; ++j) c[j] = std::fma(a, b[j], c[j]);
    }
}

// ---------------------------------------------------------------------------
// BlockSelection (selection.hpp:17-56, selection.cpp)
struct Sel {
  Index B = 0, H = 0, nc = 0, k = 0;
  const int32_t* idx = nullptr;
  const int32_t* row(Index b, Index h, Index qc) const { return idx + ((b * H + h) * nc + qc) * k; }
};

void validate(const Sel& s) {  // selection.cpp:24-37
  require(s.idx != nullptr && s.B * s.H * s.nc * s.k > 0, "BlockSelection: empty selection");
  for (Index r = 0; r < s.B * s.H * s.nc; ++r) {
    int32_t prev = -1;
    for (Index j = 0; j < s.k; ++j) {
      const int32_t c = s.idx[r * s.k + j];
      require(c >= 0 && c < s.nc, "BlockSelection: cube index out of range");
      require(c > prev, "BlockSelection: indices must be strictly ascending");
      prev = c;
    }
  }
}

// topk_row (coarse.hpp:30-42): descending value, ties -> lower index, reported ascending.
template <typename S>
void topk_row(const S* values, Index n, Index k, int32_t* out) {
  require(k >= 1 && k <= n, "topk_row: k must be in [1, n]");
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  auto better = [values](int32_t a, int32_t b) {
    if (values[a] != values[b]) return values[a] > values[b];
    return a < b;
  };
  std::partial_sort(order.begin(), order.begin() + k, order.end(), better);
  std::sort(order.begin(), order.begin() + k);
  std::copy(order.begin(), order.begin() + k, out);
}

// ---------------------------------------------------------------------------
// pool_cubes (coarse.hpp:47-65). mode 0 = mean, 1 = max. Mean = sequential sum / B.
template <typename S>
void pool_cubes(const Layout& L, const S* x, Index bh, Index d, int mode, S* out) {
  const Index B = L.cube;
#pragma omp parallel for schedule(static)
  for (Index u = 0; u < bh; ++u)
    for (Index c = 0; c < L.nc; ++c)
      for (Index j = 0; j < d; ++j) {
        const S* col = x + (u * L.seq + c * B) * d + j;
        S acc = col[0];
        if (mode == 0) {
          acc = S(0);
          for (Index i = 0; i < B; ++i) acc = acc + col[i * d];
          acc = acc / static_cast<S>(B);
        } else {
          for (Index i = 1; i < B; ++i) acc = std::max(acc, col[i * d]);
        }
        out[(u * L.nc + c) * d + j] = acc;
      }
}

// coarse_forward_select (coarse.hpp:71-117)
template <typename S>
void coarse_forward(const Layout& L, const S* q, const S* k, const S* v, Index Bt, Index H, Index d, Index top_k,
                    int mode, S* qc, S* kc, S* vc, S* ac, S* oc_cube, S* oc_tok, int32_t* sel) {
  require(top_k >= 1 && top_k <= L.nc, "coarse_forward_select: k must be in [1, num_cubes]");
  const Index nc = L.nc, bh = Bt * H;
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  pool_cubes(L, q, bh, d, mode, qc);
  pool_cubes(L, k, bh, d, mode, kc);
  pool_cubes(L, v, bh, d, mode, vc);
#pragma omp parallel for schedule(static)
  for (Index u = 0; u < bh; ++u) {
    const S* Q = qc + u * nc * d;
    const S* K = kc + u * nc * d;
    const S* V = vc + u * nc * d;
    S* A = ac + u * nc * nc;
    gemm_abt(Q, K, A, nc, nc, d);
    for (Index i = 0; i < nc; ++i) {
      S* row = A + i * nc;
      for (Index j = 0; j < nc; ++j) row[j] = row[j] * scale;
      S m = row[0];
      for (Index j = 1; j < nc; ++j) m = std::max(m, row[j]);
      S sum = S(0);
      for (Index j = 0; j < nc; ++j) {
        row[j] = coarse_exp<S>(row[j] - m);
        sum = sum + row[j];
      }
      for (Index j = 0; j < nc; ++j) row[j] = row[j] / sum;
      topk_row(row, nc, top_k, sel + (u * nc + i) * top_k);
      S* o = oc_cube + (u * nc + i) * d;
      std::fill(o, o + d, S(0));
      for (Index j = 0; j < nc; ++j)
        for (Index c = 0; c < d; ++c) o[c] = std::fma(row[j], V[j * d + c], o[c]);
      if (oc_tok)
        for (Index t = 0; t < L.cube; ++t) std::memcpy(oc_tok + (u * L.seq + i * L.cube + t) * d, o, sizeof(S) * d);
    }
  }
}

// coarse_backward (coarse.hpp:124-184). doc_tok: token-level dOc [B,H,L,d].
// Outputs token-level grads (overwritten). Also returns cube-level dqc/dkc/dvc if non-null.
template <typename S>
void coarse_backward(const Layout& L, const S* q, const S* k, const S* v, const S* qc, const S* kc, const S* vc,
                     const S* ac, int mode, const S* doc_tok, Index Bt, Index H, Index d, S* dq, S* dk, S* dv,
                     S* dqc_out, S* dkc_out, S* dvc_out) {
  const Index nc = L.nc, B = L.cube, bh = Bt * H;
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  std::fill(dq, dq + bh * L.seq * d, S(0));
  std::fill(dk, dk + bh * L.seq * d, S(0));
  std::fill(dv, dv + bh * L.seq * d, S(0));
#pragma omp parallel for schedule(static)
  for (Index u = 0; u < bh; ++u) {
    const S* A = ac + u * nc * nc;
    const S* Qc = qc + u * nc * d;
    const S* Kc = kc + u * nc * d;
    const S* Vc = vc + u * nc * d;
    std::vector<S> doc(nc * d, S(0)), dvc(nc * d), dp(nc * nc), ds(nc * nc), dqc(nc * d), dkc(nc * d);
    for (Index c = 0; c < nc; ++c)
      for (Index t = 0; t < B; ++t) {
        const S* g = doc_tok + (u * L.seq + c * B + t) * d;
        for (Index j = 0; j < d; ++j) doc[c * d + j] = doc[c * d + j] + g[j];
      }
    gemm_atb(A, doc.data(), dvc.data(), nc, d, nc, false);     // Ac^T dOc
    gemm_abt(doc.data(), Vc, dp.data(), nc, nc, d);             // dOc Vc^T
    for (Index i = 0; i < nc; ++i) {
      S delta = S(0);
      for (Index j = 0; j < nc; ++j) delta = std::fma(A[i * nc + j], dp[i * nc + j], delta);
      for (Index j = 0; j < nc; ++j) ds[i * nc + j] = A[i * nc + j] * (dp[i * nc + j] - delta) * scale;
    }
    gemm_ab(ds.data(), Kc, dqc.data(), nc, d, nc, false);      // dS Kc
    gemm_atb(ds.data(), Qc, dkc.data(), nc, d, nc, false);     // dS^T Qc
    if (dqc_out) std::memcpy(dqc_out + u * nc * d, dqc.data(), sizeof(S) * nc * d);
    if (dkc_out) std::memcpy(dkc_out + u * nc * d, dkc.data(), sizeof(S) * nc * d);
    if (dvc_out) std::memcpy(dvc_out + u * nc * d, dvc.data(), sizeof(S) * nc * d);
    auto unpool = [&](const std::vector<S>& dc, const S* src, S* dst) {
      for (Index c = 0; c < nc; ++c)
        for (Index j = 0; j < d; ++j) {
          if (mode == 0) {
            const S g = dc[c * d + j] / static_cast<S>(B);
            for (Index t = 0; t < B; ++t) dst[(u * L.seq + c * B + t) * d + j] = g;
          } else {  // first argmax (Eigen maxCoeff)
            Index am = 0;
            S best = src[(u * L.seq + c * B) * d + j];
            for (Index t = 1; t < B; ++t) {
              const S val = src[(u * L.seq + c * B + t) * d + j];
              if (val > best) { best = val; am = t; }
            }
            dst[(u * L.seq + c * B + am) * d + j] += dc[c * d + j];
          }
        }
    };
    unpool(dqc, q, dq);
    unpool(dkc, k, dk);
    unpool(dvc, v, dv);
  }
}

// ---------------------------------------------------------------------------
// dense_forward / dense_backward (dense.hpp:94-209). mask: uint8 [mh, S, S] or null.
template <typename S>
void dense_forward(const S* q, const S* k, const S* v, Index Bt, Index H, Index Sq, Index d, const uint8_t* mask,
                   Index mh, S* out, S* row_max, S* row_lse) {
  const Index n = Bt * H * Sq * d;
  for (Index i = 0; i < n; ++i)
    require(std::isfinite(q[i]) && std::isfinite(k[i]) && std::isfinite(v[i]), "dense_forward: non-finite input");
  if (mask) {
    require(mh == 1 || mh == H, "attention: mask head count must be 1 or match heads");
    for (Index h = 0; h < mh; ++h)
      for (Index i = 0; i < Sq; ++i) {
        bool any = false;
        for (Index j = 0; j < Sq; ++j) any |= mask[(h * Sq + i) * Sq + j] != 0;
        require(any, "attention: fully masked query row");
      }
  }
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  const S ninf = -std::numeric_limits<S>::infinity();
#pragma omp parallel for schedule(static)
  for (Index u = 0; u < Bt * H; ++u) {
    const Index h = u % H;
    const uint8_t* m = mask ? mask + (mh == 1 ? 0 : h) * Sq * Sq : nullptr;
    const S* Q = q + u * Sq * d;
    const S* K = k + u * Sq * d;
    const S* V = v + u * Sq * d;
    std::vector<S> s(Sq), kt(Sq * d);
    for (Index j = 0; j < Sq; ++j)
      for (Index c = 0; c < d; ++c) kt[c * Sq + j] = K[j * d + c];
    for (Index i = 0; i < Sq; ++i) {
      std::fill(s.begin(), s.end(), S(0));
      for (Index c = 0; c < d; ++c) {
        const S a = Q[i * d + c];
        for (Index j = 0; j < Sq; ++j) s[j] = std::fma(a, kt[c * Sq + j], s[j]);
      }
      for (Index j = 0; j < Sq; ++j) {
        s[j] = s[j] * scale;
        if (m && !m[i * Sq + j]) s[j] = ninf;
      }
      S mx = s[0];
      for (Index j = 1; j < Sq; ++j) mx = std::max(mx, s[j]);
      S sum = S(0);
      for (Index j = 0; j < Sq; ++j) {
        s[j] = std::exp(s[j] - mx);
        sum = sum + s[j];
      }
      S* o = out + (u * Sq + i) * d;
      std::fill(o, o + d, S(0));
      for (Index j = 0; j < Sq; ++j)
        for (Index c = 0; c < d; ++c) o[c] = std::fma(s[j], V[j * d + c], o[c]);
      for (Index c = 0; c < d; ++c) o[c] = o[c] / sum;
      row_max[u * Sq + i] = mx;
      row_lse[u * Sq + i] = mx + std::log(sum);
    }
  }
}

template <typename S>
void dense_backward(const S* q, const S* k, const S* v, Index Bt, Index H, Index Sq, Index d, const uint8_t* mask,
                    Index mh, const S* dout, const S* row_lse, S* dq, S* dk, S* dv) {
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  const S ninf = -std::numeric_limits<S>::infinity();
#pragma omp parallel for schedule(static)
  for (Index u = 0; u < Bt * H; ++u) {
    const Index h = u % H;
    const uint8_t* m = mask ? mask + (mh == 1 ? 0 : h) * Sq * Sq : nullptr;
    const S* Q = q + u * Sq * d;
    const S* K = k + u * Sq * d;
    const S* V = v + u * Sq * d;
    const S* dO = dout + u * Sq * d;
    S* dQ = dq + u * Sq * d;
    S* dK = dk + u * Sq * d;
    S* dV = dv + u * Sq * d;
    std::fill(dQ, dQ + Sq * d, S(0));
    std::fill(dK, dK + Sq * d, S(0));
    std::fill(dV, dV + Sq * d, S(0));
    std::vector<S> p(Sq), dp(Sq);
    for (Index i = 0; i < Sq; ++i) {
      const S lse = row_lse[u * Sq + i];
      S delta = S(0);
      for (Index j = 0; j < Sq; ++j) {
        S sc = dot(Q + i * d, K + j * d, d) * scale;
        if (m && !m[i * Sq + j]) sc = ninf;
        p[j] = std::exp(sc - lse);
        dp[j] = dot(dO + i * d, V + j * d, d);
        delta = std::fma(p[j], dp[j], delta);
      }
      for (Index j = 0; j < Sq; ++j) {
        const S ds = p[j] * (dp[j] - delta) * scale;
        for (Index c = 0; c < d; ++c) {
          dQ[i * d + c] = std::fma(ds, K[j * d + c], dQ[i * d + c]);
          dK[j * d + c] = std::fma(ds, Q[i * d + c], dK[j * d + c]);
          dV[j * d + c] = std::fma(p[j], dO[i * d + c], dV[j * d + c]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fine_forward (fine.hpp:43-99): per (b,h,qc), streaming softmax over the
// selected key cubes in ascending order.
template <typename S>
void fine_forward(const Layout& L, const S* q, const S* k, const S* v, const Sel& sel, Index d, S* out,
                  S* row_max, S* row_lse) {
  const Index B = L.cube, nc = L.nc, H = sel.H;
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  const S ninf = -std::numeric_limits<S>::infinity();
#pragma omp parallel for schedule(static)
  for (Index w = 0; w < sel.B * H * nc; ++w) {
    const Index u = w / nc, qc = w % nc;
    const S* Q = q + (u * L.seq + qc * B) * d;
    std::vector<S> mx(B, ninf), sum(B, S(0)), acc(B * d, S(0)), s(B * B);
    const int32_t* r = sel.idx + w * sel.k;
    for (Index t = 0; t < sel.k; ++t) {
      const Index kc = r[t];
      const S* K = k + (u * L.seq + kc * B) * d;
      const S* V = v + (u * L.seq + kc * B) * d;
      gemm_abt(Q, K, s.data(), B, B, d);
      for (Index i = 0; i < B; ++i) {
        S tmax = ninf;
        for (Index j = 0; j < B; ++j) {
          s[i * B + j] = s[i * B + j] * scale;
          tmax = std::max(tmax, s[i * B + j]);
        }
        const S nm = std::max(mx[i], tmax);
        const S resc = std::exp(mx[i] - nm);
        S rs = S(0);
        for (Index j = 0; j < B; ++j) {
          s[i * B + j] = std::exp(s[i * B + j] - nm);
          rs = rs + s[i * B + j];
        }
        sum[i] = sum[i] * resc + rs;
        for (Index c = 0; c < d; ++c) acc[i * d + c] = acc[i * d + c] * resc;
        mx[i] = nm;
      }
      gemm_ab(s.data(), V, acc.data(), B, d, B, true);
    }
    for (Index i = 0; i < B; ++i) {
      S* o = out + (u * L.seq + qc * B + i) * d;
      for (Index c = 0; c < d; ++c) o[c] = acc[i * d + c] / sum[i];
      row_max[u * L.seq + qc * B + i] = mx[i];
      row_lse[u * L.seq + qc * B + i] = mx[i] + std::log(sum[i]);
    }
  }
}

// fine_backward (fine.hpp:107-204): pass A (delta), pass B (dQ), reverse map,
// dK/dV per key cube with query cubes in ascending order.
template <typename S>
void fine_backward(const Layout& L, const S* q, const S* k, const S* v, const Sel& sel, Index d, const S* dout,
                   const S* row_lse, S* dq, S* dk, S* dv, S* delta_out) {
  const Index B = L.cube, nc = L.nc, H = sel.H, bh = sel.B * H;
  const S scale = S(1) / std::sqrt(static_cast<S>(d));
  std::vector<S> delta(bh * L.seq, S(0));
  std::fill(dq, dq + bh * L.seq * d, S(0));
  std::fill(dk, dk + bh * L.seq * d, S(0));
  std::fill(dv, dv + bh * L.seq * d, S(0));

  auto tile_p_dp = [&](Index u, Index qc, Index kc, std::vector<S>& p, std::vector<S>& dp) {
    const S* Q = q + (u * L.seq + qc * B) * d;
    const S* dO = dout + (u * L.seq + qc * B) * d;
    const S* K = k + (u * L.seq + kc * B) * d;
    const S* V = v + (u * L.seq + kc * B) * d;
    gemm_abt(Q, K, p.data(), B, B, d);
    for (Index i = 0; i < B; ++i) {
      const S lse = row_lse[u * L.seq + qc * B + i];
      for (Index j = 0; j < B; ++j) p[i * B + j] = std::exp(p[i * B + j] * scale - lse);
    }
    gemm_abt(dO, V, dp.data(), B, B, d);
  };

#pragma omp parallel for schedule(static)
  for (Index w = 0; w < bh * nc; ++w) {
    const Index u = w / nc, qc = w % nc;
    std::vector<S> p(B * B), dp(B * B), dl(B, S(0)), dqb(B * d, S(0));
    const int32_t* r = sel.idx + w * sel.k;
    for (Index t = 0; t < sel.k; ++t) {
      tile_p_dp(u, qc, r[t], p, dp);
      for (Index i = 0; i < B; ++i) {
        S rs = S(0);
        for (Index j = 0; j < B; ++j) rs = std::fma(p[i * B + j], dp[i * B + j], rs);
        dl[i] = dl[i] + rs;
      }
    }
    for (Index i = 0; i < B; ++i) delta[u * L.seq + qc * B + i] = dl[i];
    for (Index t = 0; t < sel.k; ++t) {
      const Index kc = r[t];
      tile_p_dp(u, qc, kc, p, dp);
      for (Index i = 0; i < B; ++i)
        for (Index j = 0; j < B; ++j) dp[i * B + j] = p[i * B + j] * (dp[i * B + j] - dl[i]) * scale;
      gemm_ab(dp.data(), k + (u * L.seq + kc * B) * d, dqb.data(), B, d, B, true);
    }
    std::memcpy(dq + (u * L.seq + qc * B) * d, dqb.data(), sizeof(S) * B * d);
  }

  std::vector<std::vector<int32_t>> rev(bh * nc);
  for (Index u = 0; u < bh; ++u)
    for (Index qc = 0; qc < nc; ++qc)
      for (Index t = 0; t < sel.k; ++t) rev[u * nc + sel.idx[(u * nc + qc) * sel.k + t]].push_back(int32_t(qc));

#pragma omp parallel for schedule(static)
  for (Index w = 0; w < bh * nc; ++w) {
    const Index u = w / nc, kc = w % nc;
    if (rev[w].empty()) continue;
    std::vector<S> p(B * B), dp(B * B), dkb(B * d, S(0)), dvb(B * d, S(0));
    for (int32_t qc : rev[w]) {
      tile_p_dp(u, qc, kc, p, dp);
      const S* Q = q + (u * L.seq + qc * B) * d;
      const S* dO = dout + (u * L.seq + qc * B) * d;
      gemm_atb(p.data(), dO, dvb.data(), B, d, B, true);
      for (Index i = 0; i < B; ++i) {
        const S dli = delta[u * L.seq + qc * B + i];
        for (Index j = 0; j < B; ++j) dp[i * B + j] = p[i * B + j] * (dp[i * B + j] - dli) * scale;
      }
      gemm_atb(dp.data(), Q, dkb.data(), B, d, B, true);
    }
    std::memcpy(dk + (u * L.seq + kc * B) * d, dkb.data(), sizeof(S) * B * d);
    std::memcpy(dv + (u * L.seq + kc * B) * d, dvb.data(), sizeof(S) * B * d);
  }
  if (delta_out) std::memcpy(delta_out, delta.data(), sizeof(S) * bh * L.seq);
}

}  // namespace orc

// ===========================================================================
// C ABI (ctypes). Every entry returns 0 on success, -1 on std::invalid_argument
// (message via orc_last_error), -2 on any other exception.
using orc::Index;

#define ORC_TRY(...)                      \
  try {                                   \
    __VA_ARGS__;                          \
    return 0;                             \
  } catch (const std::invalid_argument& e) { \
    orc::g_err = e.what();                \
    return -1;                            \
  } catch (const std::exception& e) {     \
    orc::g_err = e.what();                \
    return -2;                            \
  }

extern "C" {

const char* orc_last_error() { return orc::g_err.c_str(); }
int orc_max_threads() { return omp_get_max_threads(); }
void orc_set_num_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
}
double orc_canon_exp(double x) { return orc::canon_exp(x); }

// layout: out[0..5] = nt,nh,nw,cube,seq,nc
int orc_layout(int64_t t, int64_t h, int64_t w, int64_t ct, int64_t ch, int64_t cw, int64_t* out6) {
  ORC_TRY({
    orc::Layout L = orc::make_layout(t, h, w, ct, ch, cw);
    out6[0] = L.nt; out6[1] = L.nh; out6[2] = L.nw; out6[3] = L.cube; out6[4] = L.seq; out6[5] = L.nc;
  })
}
int orc_tile_of_raster(int64_t t, int64_t h, int64_t w, int64_t ct, int64_t ch, int64_t cw, int64_t* out) {
  ORC_TRY({
    orc::Layout L = orc::make_layout(t, h, w, ct, ch, cw);
    for (Index i = 0; i < L.seq; ++i) out[i] = L.tile_of_raster[i];
  })
}
int orc_flatten_index(int64_t t, int64_t h, int64_t w, int64_t ct, int64_t ch, int64_t cw, int64_t a, int64_t b,
                      int64_t c, int64_t* out) {
  ORC_TRY({
    orc::Layout L = orc::make_layout(t, h, w, ct, ch, cw);
    *out = L.tile_of_raster[orc::raster_index(L, a, b, c)];
  })
}

#define ORC_LAYOUT_ARGS int64_t lt, int64_t lh, int64_t lw, int64_t lct, int64_t lch, int64_t lcw
#define ORC_MAKE_LAYOUT orc::Layout L = orc::make_layout(lt, lh, lw, lct, lch, lcw)

#define ORC_DEFINE(SUF, S)                                                                                       \
  int orc_tile_##SUF(ORC_LAYOUT_ARGS, const S* x, int64_t bh, int64_t seq, int64_t d, int inverse, S* out) {    \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, inverse ? "untile: sequence length does not match layout"                      \
                                         : "tile: sequence length does not match layout");                      \
      orc::tile(L, x, bh, d, out, inverse != 0);                                                                 \
    })                                                                                                           \
  }                                                                                                              \
  int orc_pool_##SUF(ORC_LAYOUT_ARGS, const S* x, int64_t bh, int64_t seq, int64_t d, int mode, S* out) {       \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, "pool_cubes: sequence length does not match layout");                          \
      orc::pool_cubes(L, x, bh, d, mode, out);                                                                   \
    })                                                                                                           \
  }                                                                                                              \
  int orc_topk_row_##SUF(const S* values, int64_t n, int64_t k, int32_t* out) {                                  \
    ORC_TRY(orc::topk_row(values, n, k, out))                                                                    \
  }                                                                                                              \
  int orc_coarse_forward_##SUF(ORC_LAYOUT_ARGS, const S* q, const S* k, const S* v, int64_t B, int64_t H,       \
                               int64_t seq, int64_t d, int64_t top_k, int mode, S* qc, S* kc, S* vc, S* ac,     \
                               S* oc_cube, S* oc_tok, int32_t* sel) {                                            \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, "coarse_forward_select: shape/layout mismatch");                               \
      orc::coarse_forward(L, q, k, v, B, H, d, top_k, mode, qc, kc, vc, ac, oc_cube, oc_tok, sel);               \
    })                                                                                                           \
  }                                                                                                              \
  int orc_coarse_backward_##SUF(ORC_LAYOUT_ARGS, const S* q, const S* k, const S* v, const S* qc, const S* kc,  \
                                const S* vc, const S* ac, int mode, const S* doc, int64_t B, int64_t H,          \
                                int64_t seq, int64_t d, S* dq, S* dk, S* dv, S* dqc, S* dkc, S* dvc) {           \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, "coarse_backward: dOc shape mismatch");                                        \
      orc::coarse_backward(L, q, k, v, qc, kc, vc, ac, mode, doc, B, H, d, dq, dk, dv, dqc, dkc, dvc);           \
    })                                                                                                           \
  }                                                                                                              \
  int orc_dense_forward_##SUF(const S* q, const S* k, const S* v, int64_t B, int64_t H, int64_t seq, int64_t d,  \
                              const uint8_t* mask, int64_t mh, S* out, S* row_max, S* row_lse) {                 \
    ORC_TRY(orc::dense_forward(q, k, v, B, H, seq, d, mask, mh, out, row_max, row_lse))                          \
  }                                                                                                              \
  int orc_dense_backward_##SUF(const S* q, const S* k, const S* v, int64_t B, int64_t H, int64_t seq, int64_t d, \
                               const uint8_t* mask, int64_t mh, const S* dout, const S* row_lse, S* dq, S* dk,   \
                               S* dv) {                                                                          \
    ORC_TRY(orc::dense_backward(q, k, v, B, H, seq, d, mask, mh, dout, row_lse, dq, dk, dv))                     \
  }                                                                                                              \
  int orc_fine_forward_##SUF(ORC_LAYOUT_ARGS, const S* q, const S* k, const S* v, int64_t B, int64_t H,         \
                             int64_t seq, int64_t d, const int32_t* sel, int64_t sb, int64_t sh, int64_t snc,    \
                             int64_t top_k, S* out, S* row_max, S* row_lse) {                                    \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, "fine stage: sequence length does not match layout");                          \
      orc::require(sb == B && sh == H && snc == L.nc, "fine stage: selection does not match shapes");           \
      orc::Sel s{sb, sh, snc, top_k, sel};                                                                       \
      orc::validate(s);                                                                                          \
      orc::fine_forward(L, q, k, v, s, d, out, row_max, row_lse);                                                \
    })                                                                                                           \
  }                                                                                                              \
  int orc_fine_backward_##SUF(ORC_LAYOUT_ARGS, const S* q, const S* k, const S* v, int64_t B, int64_t H,        \
                              int64_t seq, int64_t d, const int32_t* sel, int64_t sb, int64_t sh, int64_t snc,   \
                              int64_t top_k, const S* dout, const S* row_lse, S* dq, S* dk, S* dv, S* delta) {   \
    ORC_TRY({                                                                                                    \
      ORC_MAKE_LAYOUT;                                                                                           \
      orc::require(seq == L.seq, "fine stage: sequence length does not match layout");                          \
      orc::require(sb == B && sh == H && snc == L.nc, "fine stage: selection does not match shapes");           \
      orc::Sel s{sb, sh, snc, top_k, sel};                                                                       \
      orc::validate(s);                                                                                          \
      orc::fine_backward(L, q, k, v, s, d, dout, row_lse, dq, dk, dv, delta);                                    \
    })                                                                                                           \
  }

ORC_DEFINE(f32, float)
ORC_DEFINE(f64, double)

int orc_validate_selection(const int32_t* sel, int64_t B, int64_t H, int64_t nc, int64_t k) {
  ORC_TRY({
    orc::Sel s{B, H, nc, k, sel};
    orc::validate(s);
  })
}

// ---------------------------------------------------------------------------
// Random generation exactly as the reference test fixtures draw it.
struct OrcRng {
  std::mt19937_64 g;
};
void* orc_rng_new(uint64_t seed) { return new OrcRng{std::mt19937_64(seed)}; }
void orc_rng_free(void* r) { delete static_cast<OrcRng*>(r); }
// AttnTensor::randn / randn_matrix (tensor.hpp:62-68, 126-133): one fresh
// normal_distribution per tensor, values drawn in flat order.
void orc_rng_randn(void* r, int64_t n, double stddev, double* out) {
  std::normal_distribution<double> dist(0.0, stddev);
  auto& g = static_cast<OrcRng*>(r)->g;
  for (int64_t i = 0; i < n; ++i) out[i] = dist(g);
}
int64_t orc_rng_uniform_int(void* r, int64_t a, int64_t b) {
  std::uniform_int_distribution<Index> d(a, b);
  return d(static_cast<OrcRng*>(r)->g);
}
uint64_t orc_rng_uniform_size(void* r, uint64_t a, uint64_t b) {
  std::uniform_int_distribution<std::size_t> d(a, b);
  return d(static_cast<OrcRng*>(r)->g);
}
int orc_rng_uniform_int32(void* r, int a, int b) {
  std::uniform_int_distribution<int> d(a, b);
  return d(static_cast<OrcRng*>(r)->g);
}
double orc_rng_uniform_real(void* r, double a, double b) {
  std::uniform_real_distribution<double> d(a, b);
  return d(static_cast<OrcRng*>(r)->g);
}
int orc_rng_bernoulli(void* r, double p) {
  std::bernoulli_distribution d(p);
  return d(static_cast<OrcRng*>(r)->g) ? 1 : 0;
}
void orc_rng_shuffle(void* r, int64_t* arr, int64_t n) { std::shuffle(arr, arr + n, static_cast<OrcRng*>(r)->g); }
// random_selection (selection.cpp:52-70)
int orc_rng_random_selection(void* r, int64_t B, int64_t H, int64_t nc, int64_t k, int32_t* out) {
  ORC_TRY({
    orc::require(B >= 1 && H >= 1 && nc >= 1, "BlockSelection: bad shape");
    orc::require(k >= 1 && k <= nc, "BlockSelection: k must be in [1, num_cubes]");
    auto& g = static_cast<OrcRng*>(r)->g;
    std::vector<int32_t> pool(nc);
    for (Index c = 0; c < nc; ++c) pool[c] = int32_t(c);
    for (Index row = 0; row < B * H * nc; ++row) {
      for (Index i = 0; i < k; ++i) {
        std::uniform_int_distribution<Index> pick(i, nc - 1);
        std::swap(pool[i], pool[pick(g)]);
      }
      int32_t* dst = out + row * k;
      std::copy(pool.begin(), pool.begin() + k, dst);
      std::sort(dst, dst + k);
    }
  })
}

}  // extern "C"

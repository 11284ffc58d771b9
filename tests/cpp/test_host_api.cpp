// SPDX-License-Identifier: Apache-2.0
// GPU parity test of the C++ host mirror (include/vsa_b200/vsa.hpp): the
// reference's entry points, called the way a C++ user of /root/reference/proj
// would call them, checked against the oracle (oracle/_build/liboracle.so,
// linked as the checker). Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "vsa_b200/vsa.hpp"

extern "C" {
int orc_fine_forward_f32(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const float*, const float*,
                         const float*, int64_t, int64_t, int64_t, int64_t, const int32_t*, int64_t, int64_t, int64_t,
                         int64_t, float*, float*, float*);
int orc_fine_backward_f32(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const float*, const float*,
                          const float*, int64_t, int64_t, int64_t, int64_t, const int32_t*, int64_t, int64_t, int64_t,
                          int64_t, const float*, const float*, float*, float*, float*, float*);
int orc_coarse_forward_f32(int64_t, int64_t, int64_t, int64_t, int64_t, int64_t, const float*, const float*,
                           const float*, int64_t, int64_t, int64_t, int64_t, int64_t, int, float*, float*, float*,
                           float*, float*, float*, int32_t*);
}

using namespace vsa_b200;

static int failures = 0;
#define CHECK(cond, ...)                    \
  do {                                      \
    if (!(cond)) {                          \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);             \
      std::printf("\n");                    \
      ++failures;                           \
    }                                       \
  } while (0)

template <typename F>
static bool throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static float bfr(float x) { return __bfloat162float(__float2bfloat16(x)); }

int main() {
  // ---- tiling known answers (test_tiling.cpp:40-56, 137-146)
  {
    const TileLayout L(4, 4, 4, 2, 2, 2);
    CHECK(L.cube_size == 8 && L.seq_len == 64 && L.num_cubes == 8, "layout sizes");
    CHECK(flatten_index(L, 0, 0, 0) == 0 && flatten_index(L, 1, 1, 1) == 7 && flatten_index(L, 2, 0, 0) == 32,
          "flatten_index known answers");
    CHECK(throws_invalid([] { TileLayout(5, 4, 4, 2, 2, 2); }), "non-divisible layout must throw");
    CHECK(throws_invalid([&] { flatten_index(L, 4, 0, 0); }), "out-of-range coordinate must throw");
  }
  const TileLayout L(8, 16, 16, 4, 4, 4);
  const Index B = 1, H = 2, d = 64, k = 4, nc = L.num_cubes, S = L.seq_len;
  std::mt19937_64 rng(52);
  auto q = AttnTensor<float>::randn(B, H, S, d, rng);
  auto kk = AttnTensor<float>::randn(B, H, S, d, rng);
  auto v = AttnTensor<float>::randn(B, H, S, d, rng);
  auto dout = AttnTensor<float>::randn(B, H, S, d, rng);
  const auto sel = random_selection(B, H, nc, k, rng);
  const int64_t la[6] = {8, 16, 16, 4, 4, 4};
  // ---- tile / untile round trip
  {
    const auto rt = untile(L, tile(L, q));
    bool same = true;
    for (Index i = 0; i < q.size(); ++i) same &= rt.data()[i] == q.data()[i];
    CHECK(same, "untile(tile(x)) == x");
  }
  // ---- fp32 fine forward / backward vs oracle (1e-4)
  {
    const auto res = fine_forward(L, q, kk, v, sel);
    std::vector<float> out(q.size()), rmax(B * H * S), lse(B * H * S);
    CHECK(orc_fine_forward_f32(la[0], la[1], la[2], la[3], la[4], la[5], q.data(), kk.data(), v.data(), B, H, S, d,
                               sel.data(), B, H, nc, k, out.data(), rmax.data(), lse.data()) == 0,
          "oracle fine_forward");
    double e = 0;
    for (Index i = 0; i < q.size(); ++i) e = std::max(e, double(std::fabs(res.out.data()[i] - out[i])));
    CHECK(e < 1e-4, "fp32 fine_forward err %.3e", e);
    const auto g = fine_backward(L, q, kk, v, sel, dout, res);
    std::vector<float> dq(q.size()), dk(q.size()), dv(q.size()), delta(B * H * S);
    CHECK(orc_fine_backward_f32(la[0], la[1], la[2], la[3], la[4], la[5], q.data(), kk.data(), v.data(), B, H, S, d,
                                sel.data(), B, H, nc, k, dout.data(), lse.data(), dq.data(), dk.data(), dv.data(),
                                delta.data()) == 0,
          "oracle fine_backward");
    double eq = 0, ek = 0, ev = 0;
    for (Index i = 0; i < q.size(); ++i) {
      eq = std::max(eq, double(std::fabs(g.dq.data()[i] - dq[i])) / std::max(1.0, double(std::fabs(dq[i]))));
      ek = std::max(ek, double(std::fabs(g.dk.data()[i] - dk[i])) / std::max(1.0, double(std::fabs(dk[i]))));
      ev = std::max(ev, double(std::fabs(g.dv.data()[i] - dv[i])) / std::max(1.0, double(std::fabs(dv[i]))));
    }
    CHECK(eq < 1e-4 && ek < 1e-4 && ev < 1e-4, "fp32 fine_backward err %.3e %.3e %.3e", eq, ek, ev);
  }
  // ---- coarse_forward_select: block map bit-exact with the oracle
  {
    const auto art = coarse_forward_select(L, q, kk, v, k);
    std::vector<float> qc(B * H * nc * d), kc(qc.size()), vc(qc.size()), ac(B * H * nc * nc), oc(qc.size());
    std::vector<int32_t> osel(B * H * nc * k);
    CHECK(orc_coarse_forward_f32(la[0], la[1], la[2], la[3], la[4], la[5], q.data(), kk.data(), v.data(), B, H, S, d,
                                 k, 0, qc.data(), kc.data(), vc.data(), ac.data(), oc.data(), nullptr, osel.data()) == 0,
          "oracle coarse");
    bool same = true;
    for (size_t i = 0; i < osel.size(); ++i) same &= art.sel.data()[i] == osel[i];
    for (size_t i = 0; i < ac.size(); ++i) same &= art.ac[i] == ac[i];
    CHECK(same, "coarse block map / probabilities bit-exact");
  }
  // ---- bf16 (tcgen05) fine forward vs oracle on the rounded inputs
  {
    AttnTensor<bf16> qb(B, H, S, d), kb(B, H, S, d), vb(B, H, S, d);
    AttnTensor<float> qr(B, H, S, d), kr(B, H, S, d), vr(B, H, S, d);
    for (Index i = 0; i < q.size(); ++i) {
      qb.data()[i] = __float2bfloat16(q.data()[i]);
      kb.data()[i] = __float2bfloat16(kk.data()[i]);
      vb.data()[i] = __float2bfloat16(v.data()[i]);
      qr.data()[i] = bfr(q.data()[i]);
      kr.data()[i] = bfr(kk.data()[i]);
      vr.data()[i] = bfr(v.data()[i]);
    }
    const auto res = fine_forward(L, qb, kb, vb, sel);
    std::vector<float> out(q.size()), rmax(B * H * S), lse(B * H * S);
    orc_fine_forward_f32(la[0], la[1], la[2], la[3], la[4], la[5], qr.data(), kr.data(), vr.data(), B, H, S, d,
                         sel.data(), B, H, nc, k, out.data(), rmax.data(), lse.data());
    double worst = 0;
    for (Index i = 0; i < q.size(); ++i) {
      const double err = std::fabs(__bfloat162float(res.out.data()[i]) - out[i]);
      worst = std::max(worst, err / (2e-2 + 1e-2 * std::fabs(out[i])));
    }
    CHECK(worst <= 1.0, "bf16 fine_forward outside 2e-2 + 1e-2|ref| (ratio %.3f)", worst);
  }
  // ---- invalid selections throw (test_fine.cpp:89-114)
  {
    BlockSelection bad(B, H, nc, 2);
    for (Index r = 0; r < B * H * nc; ++r) {
      bad.data()[2 * r] = 3;
      bad.data()[2 * r + 1] = 1;
    }
    CHECK(throws_invalid([&] { fine_forward(L, q, kk, v, bad); }), "unsorted selection must throw");
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}

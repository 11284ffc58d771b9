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
  // ---- vsa_forward / vsa_backward with hidden states and VsaParams (vsa.hpp:89-189)
  {
    const Index md = 256;
    std::mt19937_64 r2(71);
    auto qf = AttnTensor<float>::randn(B, H, S, d, r2);
    auto kf = AttnTensor<float>::randn(B, H, S, d, r2);
    auto vf = AttnTensor<float>::randn(B, H, S, d, r2);
    auto hf = AttnTensor<float>::randn(B, 1, S, md, r2);
    auto df = AttnTensor<float>::randn(B, H, S, d, r2);
    auto tob = [](const AttnTensor<float>& x) {
      AttnTensor<bf16> y(x.batch(), x.heads(), x.seq(), x.dim());
      for (Index i = 0; i < x.size(); ++i) y.data()[i] = __float2bfloat16(x.data()[i]);
      return y;
    };
    auto rnd = [](const AttnTensor<float>& x) {
      AttnTensor<float> y(x.batch(), x.heads(), x.seq(), x.dim());
      for (Index i = 0; i < x.size(); ++i) y.data()[i] = bfr(x.data()[i]);
      return y;
    };
    const auto qb = tob(qf), kb = tob(kf), vb = tob(vf), hb = tob(hf), db = tob(df);
    const auto qr = rnd(qf), kr = rnd(kf), vr = rnd(vf), dr = rnd(df);
    // adaptation_init: Wg = 0, Gf = 1, k = nc -> the dense attention (test_vsa.cpp:32-52)
    const auto pa = VsaParams<bf16>::adaptation_init(md, H, d, nc);
    const auto fa = vsa_forward(L, hb, qb, kb, vb, pa);
    const auto all = BlockSelection::all_cubes(B, H, nc);
    std::vector<float> out(q.size()), rmax(B * H * S), lse(B * H * S);
    orc_fine_forward_f32(la[0], la[1], la[2], la[3], la[4], la[5], qr.data(), kr.data(), vr.data(), B, H, S, d,
                         all.data(), B, H, nc, nc, out.data(), rmax.data(), lse.data());
    double worst = 0;
    for (Index i = 0; i < q.size(); ++i)
      worst = std::max(worst, std::fabs(__bfloat162float(fa.out.data()[i]) - out[i]) / (2e-2 + 1e-2 * std::fabs(out[i])));
    CHECK(worst <= 1.0, "adaptation_init vsa_forward != dense attention (ratio %.3f)", worst);
    const auto ga = vsa_backward(L, fa, hb, qb, kb, vb, pa, db);
    std::vector<float> dq(q.size()), dk(q.size()), dv(q.size()), delta(B * H * S);
    orc_fine_backward_f32(la[0], la[1], la[2], la[3], la[4], la[5], qr.data(), kr.data(), vr.data(), B, H, S, d,
                          all.data(), B, H, nc, nc, dr.data(), lse.data(), dq.data(), dk.data(), dv.data(),
                          delta.data());
    // Gc = 0 in adaptation_init, so the coarse path contributes no Q/K/V gradient
    double wq = 0, wk = 0, wv = 0;
    for (Index i = 0; i < q.size(); ++i) {
      wq = std::max(wq, std::fabs(__bfloat162float(ga.dq.data()[i]) - dq[i]) / (2e-2 + 1e-2 * std::fabs(dq[i])));
      wk = std::max(wk, std::fabs(__bfloat162float(ga.dk.data()[i]) - dk[i]) / (2e-2 + 1e-2 * std::fabs(dk[i])));
      wv = std::max(wv, std::fabs(__bfloat162float(ga.dv.data()[i]) - dv[i]) / (2e-2 + 1e-2 * std::fabs(dv[i])));
    }
    CHECK(wq <= 1.0 && wk <= 1.0 && wv <= 1.0, "adaptation vsa_backward != dense backward (%.3f %.3f %.3f)", wq, wk, wv);
    const Index cols = 2 * H * d;
    bool right_zero = true;
    for (Index r = 0; r < md; ++r)
      for (Index c = H * d; c < cols; ++c) right_zero &= ga.dgate_weight[size_t(r * cols + c)] == 0.f;
    CHECK(right_zero, "adaptation: the fine half of dWg must be exactly 0");
    // random_init (sigmoid): the output is the gated sum of the returned artifacts
    auto pr = VsaParams<bf16>::random_init(md, H, d, k, r2);
    pr.activation = GateActivation::kSigmoid;
    const auto fr = vsa_forward(L, hb, qb, kb, vb, pr);
    double wc = 0;
    for (Index b = 0; b < B; ++b)
      for (Index h = 0; h < H; ++h)
        for (Index s = 0; s < S; ++s)
          for (Index j = 0; j < d; ++j) {
            const float oc = fr.coarse.oc_cube[size_t(((b * H + h) * nc + s / L.cube_size) * d + j)];
            const float ref = oc * __bfloat162float(fr.gate_coarse.at(b, h, s, j)) +
                              __bfloat162float(fr.fine.out.at(b, h, s, j)) * __bfloat162float(fr.gate_fine.at(b, h, s, j));
            const float g = __bfloat162float(fr.out.at(b, h, s, j));
            wc = std::max(wc, double(std::fabs(g - ref)) / (1e-2 + 1e-2 * std::fabs(ref)));
          }
    CHECK(wc <= 1.0, "vsa_forward out != Oc*Gc + Of*Gf of its artifacts (ratio %.3f)", wc);
    bool sig_ok = true;
    for (Index i = 0; i < fr.gate_coarse.size(); ++i) {
      const float g = __bfloat162float(fr.gate_coarse.data()[i]);
      sig_ok &= g > 0.f && g < 1.f;
    }
    CHECK(sig_ok, "sigmoid gates outside (0, 1)");
    const auto gr = vsa_backward(L, fr, hb, qb, kb, vb, pr, db);
    bool finite = true;
    for (Index i = 0; i < gr.dhidden.size(); ++i) finite &= std::isfinite(__bfloat162float(gr.dhidden.data()[i]));
    for (float x : gr.dgate_weight) finite &= std::isfinite(x);
    CHECK(finite && gr.dhidden.dim() == md, "vsa_backward gate gradients");
    CHECK(throws_invalid([&] { vsa_forward(L, hb, qb, kb, vb, VsaParams<bf16>::random_init(md + 64, H, d, k, r2)); }),
          "mismatched gate projection must throw");
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

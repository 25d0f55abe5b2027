// test_shim.cpp — the C++ host API (include/modulora_b200.hpp) on a B200,
// written like the reference's own suites (proj/tests/test_lowprec.cpp,
// test_lora.cpp, test_quantize.cpp). Plain g++ -std=c++20 consumer of
// libmlra.so. Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>

#include "modulora_b200.hpp"

using namespace modulora_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)

template <typename E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// LSB-first bitstream (bitpack.cpp:68-91), test-side restatement.
static PackedCodes ref_pack(const std::vector<uint32_t>& codes, int bits) {
  PackedCodes p;
  p.bits = bits;
  p.count = codes.size();
  p.words.assign(packed_word_count(codes.size(), bits), 0u);
  for (std::size_t i = 0; i < codes.size(); ++i) {
    const std::size_t bit = i * bits, w = bit / 32, off = bit % 32;
    p.words[w] |= codes[i] << off;
    if (off + bits > 32) p.words[w + 1] |= codes[i] >> (32 - off);
  }
  return p;
}

static QuantizedMatrix random_q(std::size_t rows, std::size_t cols, int bits, std::size_t group,
                                uint64_t seed) {
  std::mt19937_64 g(seed);
  std::vector<uint32_t> codes(rows * cols);
  for (auto& c : codes) c = static_cast<uint32_t>(g() % (1u << bits));
  QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.bits = bits;
  q.group_size = group;
  q.codes = ref_pack(codes, bits);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (std::size_t i = 0; i < rows * (cols / group); ++i) {
    q.scales.push_back(static_cast<float>(0.002 + 0.01 * u(g)));
    q.zeros.push_back(static_cast<float>(-0.05 * u(g)));
  }
  return q;
}

// (float) of the reference f64 value (quantize.cpp:123-137), test-side.
static HostMatrix ref_deq(const QuantizedMatrix& q) {
  HostMatrix w(q.rows, q.cols);
  const std::size_t ng = q.num_groups();
  for (std::size_t i = 0; i < q.rows; ++i)
    for (std::size_t j = 0; j < q.cols; ++j) {
      const std::size_t idx = i * q.cols + j, bit = idx * q.bits, wd = bit / 32, off = bit % 32;
      uint64_t v = q.codes.words[wd] >> off;
      if (off + q.bits > 32) v |= static_cast<uint64_t>(q.codes.words[wd + 1]) << (32 - off);
      const uint32_t c = static_cast<uint32_t>(v) & ((1u << q.bits) - 1u);
      const std::size_t gi = i * ng + j / q.group_size;
      w(i, j) = static_cast<float>(static_cast<double>(q.scales[gi]) * c +
                                   static_cast<double>(q.zeros[gi]));
    }
  return w;
}

static double bf(double v) { return __bfloat162float(__float2bfloat16_rn(static_cast<float>(v))); }

static HostMatrix randn(std::size_t r, std::size_t c, uint64_t seed, double sd = 1.0) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> nd(0.0, sd);
  HostMatrix m(r, c);
  for (double& v : m.data) v = bf(nd(g));  // exactly representable on the device
  return m;
}

static double rel_fro(const HostMatrix& a, const HostMatrix& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.data.size(); ++i) {
    num += (a.data[i] - b.data[i]) * (a.data[i] - b.data[i]);
    den += b.data[i] * b.data[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1.0));
}

int main(int argc, char** argv) {
  const std::string golden = argc > 1 ? argv[1] : "tests/golden";
  if (mlra_device_check() != MLRA_OK) {
    std::printf("SKIP: %s\n", mlra_last_error());
    return 0;
  }
  // --- dequantize is bit-exact with (float) of the reference value (test_quantize.cpp:34-60)
  {
    QuantizedMatrix q;  // codes [[0,1],[2,3]], b=2, g=2, s=[0.5,1], z=[-1,0]
    q.rows = 2;
    q.cols = 2;
    q.bits = 2;
    q.group_size = 2;
    q.codes = ref_pack({0, 1, 2, 3}, 2);
    q.scales = {0.5f, 1.0f};
    q.zeros = {-1.0f, 0.0f};
    DeviceQuantizedMatrix dq(q);
    const HostMatrix w = dequantize(dq);
    CHECK(w(0, 0) == -1.0 && w(0, 1) == -0.5 && w(1, 0) == 2.0 && w(1, 1) == 3.0);
    CHECK(dequantize_row(dq, 1)[1] == 3.0);
    CHECK(throws<RangeError>([&] { dequantize_row(dq, 2); }));
  }
  for (int bits : {2, 3, 4, 8}) {
    const QuantizedMatrix q = random_q(96, 384, bits, 128, 7 + bits);
    DeviceQuantizedMatrix dq(q);
    const HostMatrix got = dequantize(dq), want = ref_deq(q);
    bool same = true;
    for (std::size_t i = 0; i < got.data.size(); ++i) same = same && got.data[i] == want.data[i];
    CHECK(same);
  }
  // --- identity weights pass inputs and gradients through (test_lowprec.cpp:73-82)
  {
    const std::size_t n = 256;
    std::vector<uint32_t> codes(n * n, 0);
    for (std::size_t i = 0; i < n; ++i) codes[i * n + i] = 1;
    QuantizedMatrix q;
    q.rows = q.cols = n;
    q.bits = 8;
    q.group_size = n;
    q.codes = ref_pack(codes, 8);
    q.scales.assign(n, 1.0f);
    q.zeros.assign(n, 0.0f);
    auto dq = std::make_shared<const DeviceQuantizedMatrix>(q);
    const HostMatrix x = randn(300, n, 1), g = randn(300, n, 2);
    for (auto s : {MaterializationStrategy::WeightMaterialize, MaterializationStrategy::RowMaterialize,
                   MaterializationStrategy::QuantizerMatvec}) {
      LpLinearContext ctx{dq, s, "eye"};
      CHECK(lp_forward(ctx, x).data == x.data);
      CHECK(lp_backward(ctx, g).data == g.data);
    }
  }
  // --- lp_forward / lp_backward vs the f64 product on the same bf16 operands
  {
    const QuantizedMatrix q = random_q(512, 768, 3, 128, 99);
    auto dq = std::make_shared<const DeviceQuantizedMatrix>(q);
    HostMatrix w = ref_deq(q);
    for (double& v : w.data) v = bf(v);  // the tensor cores see bf16(Ŵ)
    const HostMatrix x = randn(600, 768, 3), g = randn(600, 512, 4);
    HostMatrix yr(600, 512), dxr(600, 768);
    for (std::size_t t = 0; t < 600; ++t)
      for (std::size_t n = 0; n < 512; ++n) {
        double a = 0;
        for (std::size_t k = 0; k < 768; ++k) a += x(t, k) * w(n, k);
        yr(t, n) = a;
        for (std::size_t k = 0; k < 768; ++k) dxr(t, k) += g(t, n) * w(n, k);
      }
    for (auto s : {MaterializationStrategy::WeightMaterialize, MaterializationStrategy::RowMaterialize}) {
      LpLinearContext ctx{dq, s, "l"};
      CHECK(rel_fro(lp_forward(ctx, x), yr) <= 1e-5);
      CHECK(rel_fro(lp_backward(ctx, g), dxr) <= 1e-5);
    }
    LpLinearContext wctx{dq, MaterializationStrategy::WeightMaterialize, "l"};
    LpLinearContext rctx{dq, MaterializationStrategy::RowMaterialize, "l"};
    CHECK(wctx.ledger_bytes() == 512u * 768u * 2u);  // bf16 Ŵ per pass
    CHECK(rctx.ledger_bytes() == 0u);                // fused: nothing in HBM
  }
  // --- layer: fresh layer == base; closed-form adapter gradients (test_lora.cpp:91-228)
  {
    const QuantizedMatrix q = random_q(256, 512, 4, 128, 5);
    auto dq = std::make_shared<const DeviceQuantizedMatrix>(q);
    ModuLoraLayer L = make_layer("c", dq, 8, 16.0, 31, MaterializationStrategy::RowMaterialize);
    const HostMatrix x = randn(300, 512, 33);
    LpLinearContext ctx{dq, MaterializationStrategy::RowMaterialize, "c"};
    LayerActivations s;
    CHECK(layer_forward(L, x, &s).data == lp_forward(ctx, x).data);
    CHECK(throws<ContractError>([&] { grads_of_adapter(L); }));
    // move A off zero, then check dA = s·gᵀ·(xB), dB = s·xᵀ·(gA)
    std::vector<float> ha(256 * 8), hb(512 * 8);
    std::mt19937_64 gen(7);
    std::normal_distribution<double> nd(0.0, 0.5);
    for (float& v : ha) v = static_cast<float>(nd(gen));
    L.adapter.a.upload(ha.data());
    L.adapter.b.download(hb.data());
    layer_forward(L, x, &s);
    const HostMatrix g = randn(300, 256, 34);
    layer_backward(L, s, g);
    const auto [ga, gb] = grads_of_adapter(L);
    const double sc = L.adapter.scaling();
    HostMatrix xb(300, 8), gA(300, 8), wa(256, 8), wb(512, 8);
    for (std::size_t t = 0; t < 300; ++t)
      for (std::size_t j = 0; j < 8; ++j) {
        for (std::size_t k = 0; k < 512; ++k) xb(t, j) += x(t, k) * hb[k * 8 + j];
        for (std::size_t n = 0; n < 256; ++n) gA(t, j) += g(t, n) * ha[n * 8 + j];
      }
    for (std::size_t t = 0; t < 300; ++t)
      for (std::size_t j = 0; j < 8; ++j) {
        for (std::size_t n = 0; n < 256; ++n) wa(n, j) += sc * g(t, n) * xb(t, j);
        for (std::size_t k = 0; k < 512; ++k) wb(k, j) += sc * x(t, k) * gA(t, j);
      }
    CHECK(rel_fro(ga, wa) <= 1e-4);
    CHECK(rel_fro(gb, wb) <= 1e-4);
  }
  // --- error taxonomy (errors.hpp; quantize.cpp:82-115; lowprec_linear.cpp:153-156)
  {
    CHECK(throws<ConfigError>([] { parse_strategy("column"); }));
    CHECK(parse_strategy(strategy_name(MaterializationStrategy::QuantizerMatvec)) ==
          MaterializationStrategy::QuantizerMatvec);
    QuantizedMatrix q = random_q(8, 16, 4, 8, 1);
    q.scales[3] = 0.0f;
    CHECK(throws<NumericError>([&] { DeviceQuantizedMatrix d(q); }));
    QuantizedMatrix q2 = random_q(8, 16, 4, 8, 1);
    q2.codes.words.pop_back();
    CHECK(throws<FormatError>([&] { DeviceQuantizedMatrix d(q2); }));
    QuantizedMatrix q3 = random_q(8, 16, 4, 8, 1);
    q3.group_size = 5;
    CHECK(throws<ConfigError>([&] { DeviceQuantizedMatrix d(q3); }));
    auto dq = std::make_shared<const DeviceQuantizedMatrix>(random_q(8, 16, 4, 8, 2));
    LpLinearContext ctx{dq, MaterializationStrategy::RowMaterialize, "e"};
    CHECK(throws<DimensionError>([&] { lp_forward(ctx, HostMatrix(2, 15)); }));
    CHECK(throws<DimensionError>([&] { lp_backward(ctx, HostMatrix(2, 9)); }));
    LpLinearContext empty;
    CHECK(throws<ContractError>([&] { lp_forward(empty, HostMatrix(2, 16)); }));
    CHECK(throws<ConfigError>([&] { init_adapter(16, 8, 0, 16.0, 1); }));
    CHECK(throws<ConfigError>([&] { init_adapter(16, 8, 2, 0.0, 1); }));
  }
  // --- the matvec hook is consulted under QuantizerMatvec only (test_lowprec.cpp:354-377)
  {
    auto dq = std::make_shared<const DeviceQuantizedMatrix>(random_q(40, 64, 4, 16, 33));
    const HostMatrix x = randn(3, 64, 34), g = randn(3, 40, 35);
    LpLinearContext plain{dq, MaterializationStrategy::QuantizerMatvec, "p"};
    LpLinearContext hooked = plain;
    hooked.matvec_hook = std::make_shared<DoublingQuantizer>();
    const HostMatrix y0 = lp_forward(plain, x), y1 = lp_forward(hooked, x);
    HostMatrix y2 = y0;
    for (double& v : y2.data) v *= 2.0;
    CHECK(rel_fro(y1, y2) <= 1e-6);
    const HostMatrix d0 = lp_backward(plain, g), d1 = lp_backward(hooked, g);
    HostMatrix d2 = d0;
    for (double& v : d2.data) v *= 2.0;
    CHECK(rel_fro(d1, d2) <= 1e-6);
    LpLinearContext w0{dq, MaterializationStrategy::WeightMaterialize, "w"};
    LpLinearContext w1 = w0;
    w1.matvec_hook = hooked.matvec_hook;
    CHECK(lp_forward(w0, x).data == lp_forward(w1, x).data);
  }
  // --- cb2 plugin: decode law known answer (tests/test_cb2.py::test_cb2_known_answer)
  {
    std::vector<float> cb(256 * 8, 0.0f);
    const float e3[8] = {0.5f, 1.5f, 2.5f, 3.5f, 0.25f, 0.0f, 1.0f, 2.0f};
    for (int j = 0; j < 8; ++j) cb[3 * 8 + j] = e3[j];
    const std::vector<std::uint16_t> codes = {static_cast<std::uint16_t>(3 | (1 << 9) | (1 << 15)), 3};
    auto q = upload_cb2(1, 16, 8, codes, cb, {2.0f, 0.5f});
    const HostMatrix w = dequantize(*q);
    const double want[16] = {1, -3, 5, 7, 0.5, 0, 2, -4, 0.25, 0.75, 1.25, 1.75, 0.125, 0, 0.5, 1};
    bool ok = true;
    for (int j = 0; j < 16; ++j) ok = ok && w(0, j) == want[j];
    CHECK(ok);
    CHECK(throws<NumericError>([&] { upload_cb2(1, 16, 8, codes, cb, {2.0f, -1.0f}); }));
  }
  // --- lut plugin: decode law known answer (tests/test_lut.py::test_lut_known_answer)
  {
    // the header's pack() against the test-side restatement, all widths
    bool same = true;
    for (int b : {2, 3, 4, 8}) {
      std::vector<std::uint32_t> cs(1000);
      for (std::size_t i = 0; i < cs.size(); ++i) cs[i] = static_cast<std::uint32_t>(i * 2654435761u >> 7) & ((1u << b) - 1u);
      same = same && pack(cs, b).words == ref_pack(cs, b).words;
    }
    CHECK(same);
    CHECK(throws<RangeError>([] { pack(std::vector<std::uint32_t>{4}, 2); }));
    PackedCodes pc = pack(std::vector<std::uint32_t>{0, 1, 2, 3, 3, 2, 1, 0, 0, 1, 2, 3, 3, 2, 1, 0}, 2);
    auto q = upload_lut(2, 8, 8, pc, {-1.0f, -0.25f, 0.5f, 3.0f}, {2.0f, 0.5f});
    const HostMatrix w = dequantize(*q);
    const double want[2][8] = {{-2, -0.5, 1, 6, 6, 1, -0.5, -2},
                               {-0.5, -0.125, 0.25, 1.5, 1.5, 0.25, -0.125, -0.5}};
    bool ok = true;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 8; ++j) ok = ok && w(i, j) == want[i][j];
    CHECK(ok);
    CHECK(throws<NumericError>([&] { upload_lut(2, 8, 8, pc, {-1.0f, NAN, 0.5f, 3.0f}, {2.0f, 0.5f}); }));
    CHECK(throws<ConfigError>([&] { upload_lut(2, 8, 4, pc, {-1.0f, 0.0f, 0.5f, 3.0f}, {1, 1, 1, 1}); }));
  }
  // --- device RTN / OPTQ through the C++ mirror: the KAT of test_quantize.cpp:34-60 style
  // shapes, checked for the grid law and against the host restatement of compute_grid
  {
    HostMatrix w(2, 4);
    const double wv[8] = {-1.0, -0.5, 0.5, 1.0, 2.0, 2.0, 2.0, 2.0};
    for (int i = 0; i < 8; ++i) w.data[i] = wv[i];
    const QuantizedMatrix q = quantize_rtn(w, 2, 4);
    // row 0: lo -1, hi 1 -> scale 2/3, zero -1; row 1 flat -> scale 1, zero 2
    CHECK(q.scales.size() == 2 && q.zeros[0] == -1.0f && q.scales[0] == static_cast<float>(2.0 / 3.0));
    CHECK(q.scales[1] == 1.0f && q.zeros[1] == 2.0f);
    CHECK(q.codes.words.size() == 1 && q.codes.words[0] == ((0u) | (1u << 2) | (2u << 4) | (3u << 6)));
    HostMatrix x(6, 4);
    for (std::size_t i = 0; i < x.data.size(); ++i) x.data[i] = std::sin(1.0 + 0.7 * static_cast<double>(i));
    const QuantizedMatrix o = quantize_optq(w, x, 2, 4, 0.01);
    CHECK(o.scales == q.scales && o.zeros == q.zeros);  // grids come from the original weights
    CHECK(throws<DimensionError>([&] { quantize_optq(w, HostMatrix(3, 5), 2, 4); }));
    CHECK(throws<ConfigError>([&] { quantize_rtn(w, 5, 4); }));
  }
  // --- AdamW first step replicates the update arithmetic (test_train.cpp:145-167)
  {
    const double p0[3] = {1.0, -2.0, 3.0}, g0[3] = {0.1, -0.2, 0.3};
    DeviceBuffer<double> p(3), gr(3);
    p.upload(p0);
    gr.upload(g0);
    AdamW opt(0.9, 0.999, 1e-8, 0.0);
    opt.step(p.get(), gr.get(), MLRA_F64, {3}, {"p"}, 0, 0.01);
    double got[3];
    p.download(got);
    bool ok = true;
    for (int j = 0; j < 3; ++j) {
      const double m = (1.0 - 0.9) * g0[j], v = (1.0 - 0.999) * g0[j] * g0[j];
      const double mhat = m / (1.0 - std::pow(0.9, 1.0)), vhat = v / (1.0 - std::pow(0.999, 1.0));
      ok = ok && got[j] == p0[j] * (1.0 - 0.01 * 0.0) - 0.01 * mhat / (std::sqrt(vhat) + 1e-8);
    }
    CHECK(ok);
    const double bad[3] = {0.1, NAN, 0.3};
    gr.upload(bad);
    CHECK(throws<NumericError>([&] { opt.step(p.get(), gr.get(), MLRA_F64, {3}, {"p"}, 1, 0.01); }));
  }
  // --- checkpoint: the reference's golden.mlra digests (acceptance.cpp:462-463)
  {
    Checkpoint c(golden + "/golden.mlra");
    CHECK(c.file_hash() == 0xb48207d130703ee4ull);
    CHECK(c.frozen_state_hash() == 0xa3d66a9e729158ffull);
    CHECK(c.size() == 2);
    auto q = c.upload(0);
    CHECK(q->rows() == static_cast<std::size_t>(c.layer(0).rows));
    CHECK(throws<IoError>([&] { Checkpoint bad(golden + "/missing.mlra"); }));
    bool kind_ok = false;
    try {
      Checkpoint bad(golden + "/layer.npz");
    } catch (const FormatError& e) {
      kind_ok = e.kind == FormatError::Kind::BadMagic && e.offset == 0;
    }
    CHECK(kind_ok);
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail;
}

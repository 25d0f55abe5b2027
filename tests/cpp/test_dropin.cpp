// test_dropin.cpp — the reference's own tape running the B200 path.
//
// Built by oracle/Makefile (target `dropin`) against the REFERENCE HEADERS and
// linked with the reference's own objects (oracle/_ref/obj/*.o, compiled in
// place from /root/reference/proj/src) plus libmlra.so, through the binding a
// reference maintainer adds (integration/modulora_gpu.hpp). The test bodies
// re-run the reference's acceptance criteria with the GPU function registered
// on the reference Tape:
//
//  C1  (acceptance.cpp:98-157): 20 seeded layers, tape gradients of A, B and
//      bias vs central differences at the reference's own 1e-4 bar — exact
//      even with the bf16 base, because the finite differences see the same
//      deterministic device base; dX vs the reference's CPU tape at the bf16
//      bar (4e-3 normwise per bf16 operand rounding; dX
//      carries two: bf16(dY) and bf16(Ŵ) -> 8e-3). Inputs x are bf16-exact.
//  C1w the whole layer as ONE GpuModuLoraFunction record: Y, dX, dA, dB, dbias
//      vs the reference's CPU tape on the same inputs (bf16 bars).
//  C8  (acceptance.cpp:421-457): 50 cases, the three strategies are the same
//      linear map — bit-identical on the device — and within the bf16 bar of
//      the reference's lp_forward / lp_backward.
//  ERR the reference's error taxonomy through the binding (DimensionError,
//      ContractError).
//
// Prints one [PASS]/[FAIL] line per check; exit code = failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "../../integration/modulora_gpu.hpp"
#include "modulora/rng.hpp"

using namespace modulora;

namespace {

double max_rel_diff(const DenseMatrix& a, const DenseMatrix& b) {  // test_util.hpp:18-32
  if (a.rows() != b.rows() || a.cols() != b.cols()) return 1e300;
  double w = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double x = a.data()[i], y = b.data()[i];
    w = std::max(w, std::abs(x - y) / std::max({1.0, std::abs(x), std::abs(y)}));
  }
  return w;
}

double rel_fro(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return 1e300;
  double n = 0.0, d = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double e = a.data()[i] - b.data()[i];
    n += e * e;
    d += b.data()[i] * b.data()[i];
  }
  return std::sqrt(n) / (d > 0 ? std::sqrt(d) : 1.0);
}

bool bits_equal(const DenseMatrix& a, const DenseMatrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (a.data()[i] != b.data()[i]) return false;
  return true;
}

double bf16_value(double v) {
  const uint16_t h = gpu::to_bf16(v);
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

int failures = 0;
void report(const char* name, bool pass, const std::string& details) {
  std::printf("[%s] %s: %s\n", pass ? "PASS" : "FAIL", name, details.c_str());
  if (!pass) ++failures;
}

constexpr MaterializationStrategy kStrategies[] = {MaterializationStrategy::WeightMaterialize,
                                                   MaterializationStrategy::RowMaterialize,
                                                   MaterializationStrategy::QuantizerMatvec};

// The acceptance C1 layer construction (acceptance.cpp:101-121).
struct C1Case {
  std::shared_ptr<const QuantizedMatrix> q;
  ModuLoraLayer layer;
  DenseMatrix x, target;
};
C1Case c1_case(size_t k) {
  const size_t ranks[] = {1, 2, 4};
  const int widths[] = {2, 3, 4, 8};
  const size_t d_in = 4 + (5 * k) % 13, d_out = 4 + (7 * k) % 13, rank = ranks[k % 3];
  Rng rng(mix_seed(0xACC1, k));
  auto q = std::make_shared<const QuantizedMatrix>(
      quantize_rtn(DenseMatrix::gaussian(d_out, d_in, rng), widths[k % 4], 0));
  ModuLoraLayer layer = make_layer("l", q, rank, 2.0 * static_cast<double>(rank),
                                   mix_seed(0xACC2, k), kStrategies[k % 3], true);
  layer.adapter.a.set_value(scale(DenseMatrix::gaussian(d_out, rank, rng), 0.5));
  layer.bias.set_value(scale(DenseMatrix::gaussian(1, d_out, rng), 0.3));
  DenseMatrix x = DenseMatrix::gaussian(3, d_in, rng);
  // activations as the device sees them (bf16-exact), so the CPU and GPU tapes
  // start from the same input ("on the same bf16-rounded inputs")
  for (double& v : x.data()) v = bf16_value(v);
  DenseMatrix target = DenseMatrix::gaussian(3, d_out, rng);
  return {q, std::move(layer), std::move(x), std::move(target)};
}

void zero_grads(ModuLoraLayer& L) {
  L.adapter.a.zero_grad();
  L.adapter.b.zero_grad();
  L.bias.zero_grad();
}

void check_c1_gpu_base() {
  double worst_fd = 0.0, worst_dx = 0.0;
  for (size_t k = 0; k < 20; ++k) {
    C1Case c = c1_case(k);
    auto w = std::make_shared<const gpu::DeviceWeights>(*c.q);
    // the reference's CPU tape (its own layer_forward) for dX
    Tape tc;
    Variable xc = Variable::leaf(c.x, true);
    backward(tc, mse(tc, layer_forward(tc, c.layer, xc), c.target));
    const DenseMatrix dx_cpu = xc.grad();
    zero_grads(c.layer);
    // the same tape with the base on the B200
    Tape t;
    Variable xv = Variable::leaf(c.x, true);
    backward(t, mse(t, gpu::gpu_base_layer_forward(t, c.layer, xv, w), c.target));
    auto loss_with = [&](Variable& param, const DenseMatrix& v) {
      const DenseMatrix saved = param.value();
      param.set_value(v);
      Tape t2;
      Variable x2 = Variable::leaf(c.x);
      const double out =
          mse(t2, gpu::gpu_base_layer_forward(t2, c.layer, x2, w), c.target).value()(0, 0);
      param.set_value(saved);
      return out;
    };
    Variable* params[] = {&c.layer.adapter.a, &c.layer.adapter.b, &c.layer.bias};
    for (Variable* p : params) {
      const DenseMatrix fd = finite_diff_grad(
          [&](const DenseMatrix& v) { return loss_with(*p, v); }, p->value(), 1e-5);
      worst_fd = std::max(worst_fd, max_rel_diff(fd, p->grad()));
    }
    worst_dx = std::max(worst_dx, rel_fro(xv.grad(), dx_cpu));
  }
  // dX = bf16(dY)·bf16(Ŵ): two bf16 roundings of 4..16-term dot products (the
  // upstream dY comes off the tape, not bf16-exact) -> 2 x the 4e-3 bar
  char buf[256];
  std::snprintf(buf, sizeof(buf),
                "20 seeded layers on the reference tape, GPU base: A/B/bias vs central "
                "differences max rel err %.2e (tol 1e-4); dX vs the CPU tape %.2e (tol 8e-3)",
                worst_fd, worst_dx);
  report("C1 gpu base", worst_fd <= 1e-4 && worst_dx <= 8e-3, buf);
}

void check_c1_whole_layer() {
  double w_y = 0.0, w_dx = 0.0, w_da = 0.0, w_db = 0.0, w_dbias = 0.0;
  for (size_t k = 0; k < 20; ++k) {
    C1Case c = c1_case(k);
    auto w = std::make_shared<const gpu::DeviceWeights>(*c.q);
    Tape tc;
    Variable xc = Variable::leaf(c.x, true);
    Variable yc = layer_forward(tc, c.layer, xc);
    backward(tc, mse(tc, yc, c.target));
    const DenseMatrix y_cpu = yc.value(), dx_cpu = xc.grad();
    const auto [da_cpu, db_cpu] = grads_of_adapter(c.layer);
    const DenseMatrix dbias_cpu = c.layer.bias.grad();
    zero_grads(c.layer);
    Tape t;
    Variable xv = Variable::leaf(c.x, true);
    Variable y = gpu::gpu_layer_forward(t, c.layer, xv, w);
    backward(t, mse(t, y, c.target));
    const auto [da, db] = grads_of_adapter(c.layer);
    w_y = std::max(w_y, rel_fro(y.value(), y_cpu));
    w_dx = std::max(w_dx, rel_fro(xv.grad(), dx_cpu));
    w_da = std::max(w_da, rel_fro(da, da_cpu));
    w_db = std::max(w_db, rel_fro(db, db_cpu));
    w_dbias = std::max(w_dbias, rel_fro(c.layer.bias.grad(), dbias_cpu));
  }
  // Y: bf16 Ŵ only (x is bf16-exact) -> 4e-3; dX: bf16(dY) and bf16 Ŵ -> 8e-3;
  // dA/dB/dbias depend on dY = 2(Y - target)/n, which inherits Y's bf16 error
  const double tol_y = 4e-3, tol_dx = 8e-3, tol_g = 2e-2;
  char buf[320];
  std::snprintf(buf, sizeof(buf),
                "20 layers as one GpuModuLoraFunction record vs the CPU tape: Y %.2e (tol %.0e), "
                "dX %.2e (tol %.0e); dA %.2e, dB %.2e, dbias %.2e (tol %.0e)",
                w_y, tol_y, w_dx, tol_dx, w_da, w_db, w_dbias, tol_g);
  report("C1 gpu whole layer", w_y <= tol_y && w_dx <= tol_dx && w_da <= tol_g &&
                                   w_db <= tol_g && w_dbias <= tol_g,
         buf);
}

void check_c8_strategies() {
  double w_cross = 0.0, w_ref = 0.0;
  bool bitwise = true;
  const int widths[] = {2, 3, 4, 8};
  for (uint64_t k = 0; k < 50; ++k) {  // acceptance.cpp:421-457
    Rng rng(mix_seed(0x57A7, k));
    const size_t d_in = 4 + 2 * rng.uniform_index(11);
    const size_t d_out = 3 + rng.uniform_index(22);
    const size_t group_opts[] = {0, 2, d_in / 2};
    const size_t group = group_opts[k % 3];
    const double mag = std::pow(10.0, rng.uniform(-1.0, 1.0));
    auto q = std::make_shared<const QuantizedMatrix>(
        quantize_rtn(scale(DenseMatrix::gaussian(d_out, d_in, rng), mag), widths[k % 4], group));
    const size_t m = 1 + rng.uniform_index(4);
    const DenseMatrix x = DenseMatrix::gaussian(m, d_in, rng);
    const DenseMatrix gout = DenseMatrix::gaussian(m, d_out, rng);
    auto w = std::make_shared<const gpu::DeviceWeights>(*q);
    DenseMatrix fwd[3], bwd[3];
    for (size_t si = 0; si < 3; ++si) {
      gpu::GpuLpLinearFunction f(w, kStrategies[si]);
      FunctionContext ctx;
      const DenseMatrix* in[] = {&x};
      fwd[si] = f.forward(ctx, in);
      bwd[si] = *f.backward(ctx, gout)[0];
    }
    for (size_t si = 1; si < 3; ++si) {
      bitwise = bitwise && bits_equal(fwd[0], fwd[si]) && bits_equal(bwd[0], bwd[si]);
      w_cross = std::max({w_cross, max_rel_diff(fwd[0], fwd[si]), max_rel_diff(bwd[0], bwd[si])});
    }
    LpLinearContext ctx;
    ctx.q = q;
    ctx.strategy = MaterializationStrategy::RowMaterialize;
    ctx.layer_name = "l";
    w_ref = std::max({w_ref, rel_fro(fwd[0], lp_forward(ctx, x)), rel_fro(bwd[0], lp_backward(ctx, gout))});
  }
  char buf[256];
  std::snprintf(buf, sizeof(buf),
                "50 cases: cross-strategy rel diff %.2e (bit-identical: %s); vs the reference's "
                "lp_forward/lp_backward %.2e (tol 1e-2: bf16 x and bf16 Ŵ at 4-24 wide reductions)",
                w_cross, bitwise ? "yes" : "no", w_ref);
  report("C8 gpu strategies", bitwise && w_ref <= 1e-2, buf);
}

void check_errors() {
  Rng rng(7);
  auto q = std::make_shared<const QuantizedMatrix>(
      quantize_rtn(DenseMatrix::gaussian(8, 16, rng), 4, 0));
  auto w = std::make_shared<const gpu::DeviceWeights>(*q);
  bool dim = false, contract = false;
  try {
    gpu::GpuLpLinearFunction f(w, MaterializationStrategy::RowMaterialize);
    FunctionContext ctx;
    const DenseMatrix bad(2, 15);
    const DenseMatrix* in[] = {&bad};
    f.forward(ctx, in);
  } catch (const DimensionError&) {
    dim = true;
  }
  try {
    gpu::GpuLpLinearFunction f(w, MaterializationStrategy::RowMaterialize);
    FunctionContext ctx;
    const DenseMatrix a(2, 16), b(2, 16);
    const DenseMatrix* in[] = {&a, &b};
    f.forward(ctx, in);
  } catch (const ContractError&) {
    contract = true;
  }
  report("errors", dim && contract,
         std::string("DimensionError on a 15-col input: ") + (dim ? "yes" : "no") +
             "; ContractError on two inputs: " + (contract ? "yes" : "no"));
}

}  // namespace

int main() {
  if (mlra_device_check() != MLRA_OK) {
    std::printf("[FAIL] device: %s\n", mlra_last_error());
    return 1;
  }
  check_c1_gpu_base();
  check_c1_whole_layer();
  check_c8_strategies();
  check_errors();
  return failures;
}

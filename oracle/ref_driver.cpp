// ref_driver.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/mlra_oracle.c header). Built by
// oracle/Makefile into oracle/_ref/libmlra_ref.so, compiling the reference's
// own sources in place from /root/reference/proj/src with the reference's
// Release flags (-std=c++20 -O3 -DNDEBUG, proj/CMakeLists.txt:1-16). No
// reference source is copied into this repository. Uses:
//   * tests/golden/make_golden.py — golden fixtures pinning the C oracle;
//   * bench.py --impl reference / cpu_baseline — the reference's own CPU
//     hot path timed on the host cores (token-sharded replicas, one Tape per
//     thread as SPEC.md:310 allows).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "modulora/autodiff.hpp"
#include "modulora/errors.hpp"
#include "modulora/lora.hpp"
#include "modulora/lowprec_linear.hpp"
#include "modulora/quantize.hpp"
#include "modulora/rng.hpp"
#include "modulora/train.hpp"
#include "modulora/checkpoint.hpp"
#include "modulora/hash.hpp"
#include "modulora/model.hpp"
#include "modulora/tasks.hpp"

using namespace modulora;

namespace {

thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const RangeError& e) {
    g_err = e.what();
    return 4;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 5;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 6;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

QuantizedMatrix make_q(const uint32_t* words, uint64_t rows, uint64_t cols,
                       int bits, uint64_t group, const float* scales,
                       const float* zeros) {
  QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.bits = bits;
  q.group_size = group;
  q.codes.bits = bits;
  q.codes.count = rows * cols;
  q.codes.words.assign(words, words + packed_word_count(rows * cols, bits));
  const uint64_t ng = rows * (cols / group);
  q.scales.assign(scales, scales + ng);
  q.zeros.assign(zeros, zeros + ng);
  return q;
}

DenseMatrix dm(const double* p, uint64_t r, uint64_t c) {
  return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

void put(const DenseMatrix& m, double* out) {
  std::memcpy(out, m.data().data(), m.size() * sizeof(double));
}

// Scalar loss Σ y∘G whose backward injects exactly G as dL/dy
// (grad_out(0,0) == 1.0, so 1.0*G == G bit-for-bit).
class GradInjector final : public CustomFunction {
 public:
  explicit GradInjector(DenseMatrix g) : g_(std::move(g)) {}
  std::string_view name() const override { return "grad_injector"; }
  DenseMatrix forward(FunctionContext&,
                      std::span<const DenseMatrix* const> in) override {
    DenseMatrix out(1, 1);
    const DenseMatrix& y = *in[0];
    for (std::size_t i = 0; i < y.size(); ++i)
      out(0, 0) += y.data()[i] * g_.data()[i];
    return out;
  }
  std::vector<std::optional<DenseMatrix>> backward(
      FunctionContext&, const DenseMatrix& grad_out) override {
    std::vector<std::optional<DenseMatrix>> r;
    r.emplace_back(scale(g_, grad_out(0, 0)));
    return r;
  }

 private:
  DenseMatrix g_;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_gaussian(uint64_t seed, uint64_t rows, uint64_t cols, double mean,
                  double stddev, double* out) {
  Rng rng(seed);
  put(DenseMatrix::gaussian(rows, cols, rng, mean, stddev), out);
}

uint64_t ref_mix_seed(uint64_t seed, uint64_t salt) {
  return mix_seed(seed, salt);
}

// Rng(seed).uniform_index(2^bits) stream, as test_bitpack.cpp:19-26 draws it.
void ref_random_codes(uint64_t n, int bits, uint64_t seed, uint32_t* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < n; ++i)
    out[i] = static_cast<uint32_t>(rng.uniform_index(1u << bits));
}

uint64_t ref_packed_word_count(uint64_t count, int bits) {
  return packed_word_count(count, bits);
}

int ref_pack(const uint32_t* codes, uint64_t count, int bits, uint32_t* words) {
  try {
    PackedCodes p = pack(std::span<const uint32_t>(codes, count), bits);
    std::memcpy(words, p.words.data(), p.words.size() * 4);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_unpack(const uint32_t* words, uint64_t word_count, uint64_t count,
               int bits, uint32_t* out) {
  try {
    PackedCodes p;
    p.bits = bits;
    p.count = count;
    p.words.assign(words, words + word_count);
    std::vector<uint32_t> c = unpack(p);
    std::memcpy(out, c.data(), c.size() * 4);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_quantize_rtn(const double* w, uint64_t rows, uint64_t cols, int bits,
                     uint64_t group, uint32_t* words, float* scales,
                     float* zeros) {
  try {
    QuantizedMatrix q = quantize_rtn(dm(w, rows, cols), bits, group);
    std::memcpy(words, q.codes.words.data(), q.codes.words.size() * 4);
    std::memcpy(scales, q.scales.data(), q.scales.size() * 4);
    std::memcpy(zeros, q.zeros.data(), q.zeros.size() * 4);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// quantize_optq (quantize.cpp:213-255) and build_optq_workspace (:186-211).
int ref_quantize_optq(const double* w, const double* calib, uint64_t rows, uint64_t cols,
                      uint64_t m, int bits, uint64_t group, double damping, uint32_t* words,
                      float* scales, float* zeros) {
  try {
    QuantizedMatrix q = quantize_optq(dm(w, rows, cols), dm(calib, m, cols), bits, group, damping);
    std::memcpy(words, q.codes.words.data(), q.codes.words.size() * 4);
    std::memcpy(scales, q.scales.data(), q.scales.size() * 4);
    std::memcpy(zeros, q.zeros.data(), q.zeros.size() * 4);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_optq_workspace(const double* calib, uint64_t m, uint64_t dim, double damping,
                       double* hessian, double* upper) {
  try {
    OptqWorkspace ws = build_optq_workspace(dm(calib, m, dim), dim, damping);
    for (uint64_t i = 0; i < dim; ++i)
      for (uint64_t j = 0; j < dim; ++j) {
        hessian[i * dim + j] = ws.hessian(i, j);
        upper[i * dim + j] = ws.inv_chol_upper(i, j);
      }
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_validate(const uint32_t* words, uint64_t rows, uint64_t cols, int bits,
                 uint64_t group, const float* scales, const float* zeros) {
  try {
    make_q(words, rows, cols, bits, group, scales, zeros).validate();
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_dequantize(const uint32_t* words, uint64_t rows, uint64_t cols,
                   int bits, uint64_t group, const float* scales,
                   const float* zeros, double* out) {
  try {
    put(dequantize(make_q(words, rows, cols, bits, group, scales, zeros)), out);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// strategy: 0 weight, 1 row, 2 matvec (lowprec_linear.hpp:29-30)
int ref_lp_forward(const uint32_t* words, uint64_t rows, uint64_t cols,
                   int bits, uint64_t group, const float* scales,
                   const float* zeros, int strategy, const double* x,
                   uint64_t m, double* out) {
  try {
    LpLinearContext ctx;
    ctx.q = std::make_shared<const QuantizedMatrix>(
        make_q(words, rows, cols, bits, group, scales, zeros));
    ctx.strategy = static_cast<MaterializationStrategy>(strategy);
    put(lp_forward(ctx, dm(x, m, cols)), out);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

int ref_lp_backward(const uint32_t* words, uint64_t rows, uint64_t cols,
                    int bits, uint64_t group, const float* scales,
                    const float* zeros, int strategy, const double* g,
                    uint64_t m, double* out) {
  try {
    LpLinearContext ctx;
    ctx.q = std::make_shared<const QuantizedMatrix>(
        make_q(words, rows, cols, bits, group, scales, zeros));
    ctx.strategy = static_cast<MaterializationStrategy>(strategy);
    put(lp_backward(ctx, dm(g, m, rows)), out);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// Adapter init exactly as the reference does it (lora.cpp:14-32): writes
// B [d_in × r] (A is zero by construction).
int ref_init_adapter_b(uint64_t d_in, uint64_t d_out, uint64_t rank,
                       double alpha, uint64_t seed, double* b_out) {
  try {
    LoraAdapter ad = init_adapter(d_in, d_out, rank, alpha, seed);
    put(ad.b.value(), b_out);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// One ModuLoRA layer forward + backward through the reference's tape
// (lora.cpp:52-72, autodiff.cpp:101-139) with upstream gradient G injected.
// Any of dx / dbias may be NULL (x frozen / bias frozen).
int ref_layer_fwd_bwd(const uint32_t* words, uint64_t rows, uint64_t cols,
                      int bits, uint64_t group, const float* scales,
                      const float* zeros, int strategy, const double* a,
                      const double* b, uint64_t rank, double alpha,
                      const double* bias, const double* x, uint64_t m,
                      const double* G, double* y, double* dx, double* da,
                      double* db, double* dbias) {
  try {
    auto q = std::make_shared<const QuantizedMatrix>(
        make_q(words, rows, cols, bits, group, scales, zeros));
    ModuLoraLayer layer =
        make_layer("ref", q, rank, alpha, /*seed=*/1,
                   static_cast<MaterializationStrategy>(strategy),
                   /*bias_trainable=*/dbias != nullptr);
    layer.adapter.a.set_value(dm(a, rows, rank));
    layer.adapter.b.set_value(dm(b, cols, rank));
    if (bias) layer.bias.set_value(dm(bias, 1, rows));
    Tape t;
    Variable xv = Variable::leaf(dm(x, m, cols), dx != nullptr);
    Variable yv = layer_forward(t, layer, xv);
    put(yv.value(), y);
    Variable loss = register_custom(
        t, std::make_shared<GradInjector>(dm(G, m, rows)), {yv});
    backward(t, loss);
    auto [ga, gb] = grads_of_adapter(layer);
    put(ga, da);
    put(gb, db);
    if (dx) put(xv.grad(), dx);
    if (dbias) put(layer.bias.grad(), dbias);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// CPU baseline: `threads` token-sharded single-thread replicas of the
// reference hot path (layer_forward + tape backward, x requires grad), each
// on `m_per_thread` tokens of the same layer. Returns wall seconds of the
// slowest replica via *seconds. Inputs are seeded with the reference Rng.
int ref_bench_layer(const uint32_t* words, uint64_t rows, uint64_t cols,
                    int bits, uint64_t group, const float* scales,
                    const float* zeros, int strategy, uint64_t rank,
                    double alpha, uint64_t m_per_thread, int threads,
                    uint64_t seed, double* seconds) {
  try {
    auto q = std::make_shared<const QuantizedMatrix>(
        make_q(words, rows, cols, bits, group, scales, zeros));
    std::vector<double> secs(threads, 0.0);
    std::vector<std::exception_ptr> errs(threads);
    std::vector<std::thread> pool;
    for (int ti = 0; ti < threads; ++ti) {
      pool.emplace_back([&, ti] {
        try {
          Rng rng(mix_seed(seed, static_cast<uint64_t>(ti)));
          ModuLoraLayer layer =
              make_layer("bench", q, rank, alpha, mix_seed(seed, 0xADA9),
                         static_cast<MaterializationStrategy>(strategy));
          layer.adapter.a.set_value(
              DenseMatrix::gaussian(rows, rank, rng, 0.0, 0.02));
          const DenseMatrix x = DenseMatrix::gaussian(m_per_thread, cols, rng);
          const DenseMatrix g = DenseMatrix::gaussian(m_per_thread, rows, rng);
          const auto t0 = std::chrono::steady_clock::now();
          Tape t;
          Variable xv = Variable::leaf(x, true);
          Variable yv = layer_forward(t, layer, xv);
          Variable loss =
              register_custom(t, std::make_shared<GradInjector>(g), {yv});
          backward(t, loss);
          const auto t1 = std::chrono::steady_clock::now();
          secs[ti] = std::chrono::duration<double>(t1 - t0).count();
        } catch (...) {
          errs[ti] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    double mx = 0.0;
    for (double s : secs) mx = s > mx ? s : mx;
    *seconds = mx;
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// The CLI's `quantize` command (modulora_main.cpp:93-110, QuantizeOpts
// defaults :78-87): the recipe of the reference's golden.mlra fixture
// (test_checkpoint.cpp:28: --task regression --bits 3 --seed 11). `task`
// "regression" or "parity".
int ref_make_checkpoint(const char* path, const char* task, int bits, uint64_t seed,
                        uint64_t group_size) {
  try {
    ModelConfig mc;
    mc.task = parse_task(task);
    mc.kind = mc.task == TaskKind::TeacherResidualRegression ? ModelKind::Mlp
                                                             : ModelKind::ParityTransformer;
    mc.bits = bits;
    mc.quantizer = "rtn";
    mc.group_size = group_size;
    mc.calib_samples = 0;
    mc.rank = 8;
    mc.alpha = 32.0;
    mc.strategy = parse_strategy("weight");
    mc.base_seed = seed;
    mc.adapter_seed = mix_seed(seed, 0xADA9);
    BuiltModel built = build_model(mc);
    save_model(built.model, path);
    return 0;
  } catch (...) {
    return map_exc();
  }
}

// fnv1a64_file (hash.cpp:11-20) and load_model(path).frozen_state_hash();
// on a load failure returns the status with FormatError kind/offset.
int ref_checkpoint_probe(const char* path, uint64_t* file_hash, uint64_t* frozen_hash,
                         int* fmt_kind, uint64_t* fmt_offset) {
  *fmt_kind = -1;
  *fmt_offset = 0;
  try {
    *file_hash = fnv1a64_file(path);
    *frozen_hash = load_model(path).frozen_state_hash();
    return 0;
  } catch (const FormatError& e) {
    *fmt_kind = static_cast<int>(e.kind);
    *fmt_offset = e.offset;
    g_err = e.what();
    return 7;
  } catch (const IoError& e) {
    g_err = e.what();
    return 10;
  } catch (...) {
    return map_exc();
  }
}

// AdamW::step (train.cpp:81-134) driven for `steps` steps over n_params
// parameters (sizes[i] entries each, values concatenated, updated in place);
// grads: steps x total f64, lrs: steps. On NumericError returns 6 with the
// failing step in *bad_step (values hold the partial update of that step).
int ref_adamw_run(double beta1, double beta2, double eps, double wd, uint64_t n_params,
                  const uint64_t* sizes, double* values, const double* grads, uint64_t steps,
                  const double* lrs, uint64_t* bad_step) {
  uint64_t total = 0;
  for (uint64_t i = 0; i < n_params; ++i) total += sizes[i];
  AdamW opt(beta1, beta2, eps, wd);
  std::vector<std::string> names;
  for (uint64_t i = 0; i < n_params; ++i) names.push_back("p" + std::to_string(i));
  std::vector<Variable> params;
  uint64_t off = 0;
  for (uint64_t i = 0; i < n_params; ++i) {
    params.push_back(Variable::leaf(
        DenseMatrix(1, sizes[i], std::vector<double>(values + off, values + off + sizes[i])),
        true));
    off += sizes[i];
  }
  for (uint64_t s = 0; s < steps; ++s) {
    off = 0;
    for (uint64_t i = 0; i < n_params; ++i) {
      params[i].zero_grad();
      const double* g = grads + s * total + off;
      accumulate_grad(params[i], DenseMatrix(1, sizes[i], std::vector<double>(g, g + sizes[i])));
      off += sizes[i];
    }
    int rc = 0;
    try {
      opt.step(params, names, s, lrs[s]);
    } catch (...) {
      rc = map_exc();
      *bad_step = s;
    }
    off = 0;
    for (uint64_t i = 0; i < n_params; ++i) {
      const auto d = params[i].value().data();
      std::memcpy(values + off, d.data(), sizes[i] * sizeof(double));
      off += sizes[i];
    }
    if (rc) return rc;
  }
  return 0;
}

// model_loss of the parity transformer (model.cpp:226-292: transformer_forward
// per sequence, cross_entropy, mean) on the model saved at `path`, for caller
// sequences xs [n x seq x d] (row-major f64) and labels [n]; then the tape
// backward (autodiff.cpp:101-139). Writes the loss and every trainable
// parameter's gradient, trainable_params order (model.cpp:186-197), flat.
int ref_parity_loss_grads(const char* path, const double* xs, const int* labels, uint64_t n,
                          uint64_t seq, uint64_t d, double* loss, double* grads,
                          uint64_t grads_len) {
  try {
    ToyModel m = load_model(path);
    Tape t;
    Variable total;
    for (uint64_t i = 0; i < n; ++i) {
      DenseMatrix x(seq, d);
      for (uint64_t r = 0; r < seq; ++r)
        for (uint64_t c = 0; c < d; ++c) x(r, c) = xs[(i * seq + r) * d + c];
      Variable logits = transformer_forward(t, m, Variable::leaf(std::move(x)), nullptr);
      const int lab[] = {labels[i]};
      Variable ce = cross_entropy(t, logits, lab);
      total = total.defined() ? add(t, total, ce) : ce;
    }
    Variable L = scalar_mul(t, total, 1.0 / static_cast<double>(n));
    std::vector<Variable> params = m.trainable_params();
    for (Variable& p : params) p.zero_grad();
    backward(t, L);
    *loss = L.value()(0, 0);
    uint64_t off = 0;
    for (Variable& p : params) {
      const std::size_t cnt = p.value().rows() * p.value().cols();
      if (off + cnt > grads_len) throw ContractError("ref_parity_loss_grads: grads buffer too small");
      if (p.has_grad()) {
        const DenseMatrix& g = p.grad();
        for (std::size_t r = 0; r < g.rows(); ++r)
          for (std::size_t c = 0; c < g.cols(); ++c) grads[off + r * g.cols() + c] = g(r, c);
      } else {
        std::fill(grads + off, grads + off + cnt, 0.0);
      }
      off += cnt;
    }
    if (off != grads_len) throw ContractError("ref_parity_loss_grads: grads buffer size mismatch");
    return 0;
  } catch (...) {
    return map_exc();
  }
}

}  // extern "C"

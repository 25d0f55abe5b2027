// modulora_b200.hpp — C++20 host API over the C ABI (include/mlra.h).
//
// Mirrors the reference's hot-path headers — names, argument meaning and the
// exception taxonomy — so reference callers switch by changing a namespace:
//
//   reference (/root/reference/proj/include/modulora)      here (modulora_b200::)
//   errors.hpp  DimensionError … FormatError               same classes (thrown from mlra_status)
//   bitpack.hpp packed_word_count                           packed_word_count
//   quantize.hpp QuantizedMatrix (+validate)                QuantizedMatrix (host) → DeviceQuantizedMatrix
//               dequantize / dequantize_row(_into)          dequantize / dequantize_row (f64 host result,
//                                                           bit-exact (float) of the reference value)
//   lowprec_linear.hpp MaterializationStrategy,             same; lp_forward / lp_backward over HostMatrix
//               parse_strategy, strategy_name,              (f64 host, like DenseMatrix) or DeviceMatrix
//               LpLinearContext, lp_forward, lp_backward
//   lora.hpp    LoraAdapter, ModuLoraLayer, make_layer,     same; layer_forward / layer_backward,
//               layer_forward, grads_of_adapter             grads_of_adapter
//
// Device data are bf16 activations and fp32 adapter factors/gradients; host
// f64 overloads convert at the boundary (the reference computes in f64).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "mlra.h"

namespace modulora_b200 {

// ----------------------------------------------------------------- errors.hpp:15-63
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct RangeError : Error {
  using Error::Error;
};
struct ContractError : Error {
  using Error::Error;
};
struct NumericError : Error {
  using Error::Error;
};
struct FormatError : Error {
  enum class Kind { BadMagic, BadVersion, Truncated, BadField };
  FormatError(Kind k, std::size_t off, const std::string& msg) : Error(msg), kind(k), offset(off) {}
  Kind kind;
  std::size_t offset;
};
struct CudaError : Error {
  using Error::Error;
};

inline void check(mlra_status st) {
  if (st == MLRA_OK) return;
  const std::string m = mlra_last_error();
  switch (st) {
    case MLRA_ERR_DIMENSION: throw DimensionError(m);
    case MLRA_ERR_CONFIG: throw ConfigError(m);
    case MLRA_ERR_RANGE: throw RangeError(m);
    case MLRA_ERR_CONTRACT: throw ContractError(m);
    case MLRA_ERR_NUMERIC: throw NumericError(m);
    case MLRA_ERR_FORMAT: throw FormatError(FormatError::Kind::BadField, 0, m);
    default: throw CudaError(m);
  }
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ----------------------------------------------------------------- bitpack.hpp
inline std::size_t packed_word_count(std::size_t count, int bits) {
  return static_cast<std::size_t>(mlra_packed_word_count(count, bits));
}

// Row-major f64 host matrix (the reference's DenseMatrix layout, matrix.hpp:17-68).
struct HostMatrix {
  std::size_t rows = 0, cols = 0;
  std::vector<double> data;
  HostMatrix() = default;
  HostMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
  double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
};

// RAII device buffer.
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) : n_(n) {
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)), "cudaMalloc");
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(o.n_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  void upload(const T* h) { cuda_check(cudaMemcpy(p_, h, n_ * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
  void download(T* h) const { cuda_check(cudaMemcpy(h, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

inline std::vector<__nv_bfloat16> to_bf16(const std::vector<double>& v) {
  std::vector<__nv_bfloat16> o(v.size());
  for (std::size_t i = 0; i < v.size(); ++i) o[i] = __float2bfloat16_rn(static_cast<float>(v[i]));
  return o;
}

// ----------------------------------------------------------------- quantize.hpp:29-48
struct PackedCodes {
  int bits = 0;
  std::size_t count = 0;
  std::vector<std::uint32_t> words;
  std::size_t packed_bytes() const { return words.size() * 4; }
};

struct QuantizedMatrix {
  std::size_t rows = 0, cols = 0;
  int bits = 0;
  std::size_t group_size = 0;
  PackedCodes codes;
  std::vector<float> scales, zeros;
  std::size_t num_groups() const { return group_size ? cols / group_size : 0; }
};

// The frozen weight resident in HBM; validation on upload mirrors
// QuantizedMatrix::validate (quantize.cpp:82-115) and throws the same types.
class DeviceQuantizedMatrix {
 public:
  explicit DeviceQuantizedMatrix(const QuantizedMatrix& q, cudaStream_t st = nullptr)
      : rows_(q.rows), cols_(q.cols) {
    if (q.codes.bits != q.bits) throw ConfigError("QuantizedMatrix: packed bits mismatch");
    static const std::uint32_t kZeroWord = 0;
    static const float kZeroF = 0.0f;
    check(mlra_qweight_create(static_cast<int64_t>(q.rows), static_cast<int64_t>(q.cols), q.bits,
                              static_cast<int64_t>(q.group_size),
                              q.codes.words.empty() ? &kZeroWord : q.codes.words.data(),
                              q.codes.words.size(), q.codes.count,
                              q.scales.empty() ? &kZeroF : q.scales.data(),
                              q.zeros.empty() ? &kZeroF : q.zeros.data(), q.scales.size(), st, &h_));
  }
  ~DeviceQuantizedMatrix() { mlra_qweight_destroy(h_); }
  DeviceQuantizedMatrix(const DeviceQuantizedMatrix&) = delete;
  DeviceQuantizedMatrix& operator=(const DeviceQuantizedMatrix&) = delete;
  const mlra_qweight* handle() const { return h_; }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }

 private:
  mlra_qweight* h_ = nullptr;
  std::size_t rows_, cols_;
};

// dequantize (quantize.cpp:117-137): f64 host matrix holding (float)RN_f64(s·c+z)
// — the materialize() contract, bit-exact with (float) of the reference value.
inline HostMatrix dequantize(const DeviceQuantizedMatrix& q) {
  DeviceBuffer<float> d(q.rows() * q.cols());
  check(mlra_materialize(q.handle(), d.get(), MLRA_F32, static_cast<int64_t>(q.cols()), nullptr));
  std::vector<float> h(d.size());
  d.download(h.data());
  HostMatrix m(q.rows(), q.cols());
  for (std::size_t i = 0; i < h.size(); ++i) m.data[i] = h[i];
  return m;
}
// dequantize_row (quantize.cpp:139-161); RangeError past the last row.
inline std::vector<double> dequantize_row(const DeviceQuantizedMatrix& q, std::size_t row) {
  DeviceBuffer<float> d(q.cols());
  check(mlra_materialize_rows(q.handle(), static_cast<int64_t>(row), 1, d.get(), MLRA_F32,
                              static_cast<int64_t>(q.cols()), nullptr));
  std::vector<float> h(q.cols());
  d.download(h.data());
  return std::vector<double>(h.begin(), h.end());
}

// ----------------------------------------------------------------- lowprec_linear.hpp:29-112
enum class MaterializationStrategy { WeightMaterialize = MLRA_WEIGHT, RowMaterialize = MLRA_ROW,
                                     QuantizerMatvec = MLRA_MATVEC };

inline MaterializationStrategy parse_strategy(std::string_view name) {
  if (name == "weight") return MaterializationStrategy::WeightMaterialize;
  if (name == "row") return MaterializationStrategy::RowMaterialize;
  if (name == "matvec") return MaterializationStrategy::QuantizerMatvec;
  throw ConfigError("unknown materialization strategy '" + std::string(name) +
                    "' (expected weight, row or matvec)");
}
inline std::string_view strategy_name(MaterializationStrategy s) {
  switch (s) {
    case MaterializationStrategy::WeightMaterialize: return "weight";
    case MaterializationStrategy::RowMaterialize: return "row";
    case MaterializationStrategy::QuantizerMatvec: return "matvec";
  }
  return "?";
}

struct LpLinearContext {
  std::shared_ptr<const DeviceQuantizedMatrix> q;
  MaterializationStrategy strategy = MaterializationStrategy::RowMaterialize;
  std::string layer_name;
  // bytes the strategy materializes per pass (MemoryLedger charge)
  std::size_t ledger_bytes() const {
    return q ? static_cast<std::size_t>(mlra_ledger_bytes(q->handle(), static_cast<mlra_strategy>(strategy)))
             : 0;
  }
};

namespace detail {
inline const mlra_qweight* need_q(const LpLinearContext& ctx) {
  if (!ctx.q) throw ContractError("lp_linear: missing quantized weights");
  return ctx.q->handle();
}
inline HostMatrix download_f32(const DeviceBuffer<float>& d, std::size_t r, std::size_t c) {
  std::vector<float> h(r * c);
  if (r * c) d.download(h.data());
  HostMatrix m(r, c);
  for (std::size_t i = 0; i < h.size(); ++i) m.data[i] = h[i];
  return m;
}
}  // namespace detail

// lp_forward (lowprec_linear.cpp:150-196): x [m x d_in] (f64 host) -> [m x d_out]
inline HostMatrix lp_forward(const LpLinearContext& ctx, const HostMatrix& x) {
  const mlra_qweight* q = detail::need_q(ctx);
  if (x.cols != ctx.q->cols())
    throw DimensionError("lp_forward: input cols " + std::to_string(x.cols) + " != weight cols " +
                         std::to_string(ctx.q->cols()));
  DeviceBuffer<__nv_bfloat16> dx(x.rows * x.cols);
  DeviceBuffer<float> dy(x.rows * ctx.q->rows());
  if (x.rows) dx.upload(to_bf16(x.data).data());
  check(mlra_lp_forward(q, static_cast<mlra_strategy>(ctx.strategy), dx.get(),
                        static_cast<int64_t>(x.cols), static_cast<int64_t>(x.rows), dy.get(), MLRA_F32,
                        static_cast<int64_t>(ctx.q->rows()), nullptr));
  return detail::download_f32(dy, x.rows, ctx.q->rows());
}

// lp_backward (lowprec_linear.cpp:198-247): grad_out [m x d_out] -> [m x d_in]
inline HostMatrix lp_backward(const LpLinearContext& ctx, const HostMatrix& g) {
  const mlra_qweight* q = detail::need_q(ctx);
  if (g.cols != ctx.q->rows())
    throw DimensionError("lp_backward: grad cols " + std::to_string(g.cols) + " != weight rows " +
                         std::to_string(ctx.q->rows()));
  DeviceBuffer<__nv_bfloat16> dg(g.rows * g.cols);
  DeviceBuffer<float> dx(g.rows * ctx.q->cols());
  if (g.rows) dg.upload(to_bf16(g.data).data());
  check(mlra_lp_backward(q, static_cast<mlra_strategy>(ctx.strategy), dg.get(),
                         static_cast<int64_t>(g.cols), static_cast<int64_t>(g.rows), dx.get(), MLRA_F32,
                         static_cast<int64_t>(ctx.q->cols()), nullptr));
  return detail::download_f32(dx, g.rows, ctx.q->cols());
}

// ----------------------------------------------------------------- lora.hpp:24-83
inline constexpr double kAdapterInitStd = 0.02;

struct LoraAdapter {
  DeviceBuffer<float> a;  // [d_out x r], zero-init
  DeviceBuffer<float> b;  // [d_in x r], N(0, 0.02^2)
  std::size_t rank = 0;
  double alpha = 0.0;
  HostMatrix grad_a, grad_b;
  bool has_grad = false;
  double scaling() const { return alpha / static_cast<double>(rank); }
};

struct ModuLoraLayer {
  std::string name;
  std::shared_ptr<const DeviceQuantizedMatrix> weights;
  LoraAdapter adapter;
  DeviceBuffer<float> bias;  // [d_out]
  bool bias_trainable = false;
  HostMatrix grad_bias;
  MaterializationStrategy strategy = MaterializationStrategy::RowMaterialize;
  std::size_t d_in() const { return weights->cols(); }
  std::size_t d_out() const { return weights->rows(); }
};

// init_adapter semantics (lora.cpp:14-32): A = 0, B ~ N(0, 0.02^2) (std::mt19937_64
// stream, not the reference's hand-written Box-Muller), ConfigError on rank 0 / alpha <= 0.
inline LoraAdapter init_adapter(std::size_t d_in, std::size_t d_out, std::size_t rank, double alpha,
                                std::uint64_t seed) {
  if (rank == 0) throw ConfigError("adapter rank must be >= 1");
  if (!(alpha > 0.0)) throw ConfigError("adapter alpha must be positive");
  LoraAdapter ad;
  ad.rank = rank;
  ad.alpha = alpha;
  ad.a = DeviceBuffer<float>(d_out * rank);
  ad.b = DeviceBuffer<float>(d_in * rank);
  std::vector<float> za(d_out * rank, 0.0f), hb(d_in * rank);
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> nd(0.0, kAdapterInitStd);
  for (float& v : hb) v = static_cast<float>(nd(gen));
  ad.a.upload(za.data());
  ad.b.upload(hb.data());
  return ad;
}

inline ModuLoraLayer make_layer(std::string name, std::shared_ptr<const DeviceQuantizedMatrix> w,
                                std::size_t rank, double alpha, std::uint64_t seed,
                                MaterializationStrategy strategy, bool bias_trainable = false) {
  if (!w) throw ContractError("make_layer: null weights");
  ModuLoraLayer L;
  L.name = std::move(name);
  L.weights = std::move(w);
  L.adapter = init_adapter(L.weights->cols(), L.weights->rows(), rank, alpha, seed);
  L.bias = DeviceBuffer<float>(L.weights->rows());
  cuda_check(cudaMemset(L.bias.get(), 0, L.weights->rows() * sizeof(float)), "cudaMemset");
  L.bias_trainable = bias_trainable;
  L.strategy = strategy;
  return L;
}

// One layer step's saved state (the tape keeps x and x·B; Ŵ is never saved).
struct LayerActivations {
  DeviceBuffer<__nv_bfloat16> x;
  DeviceBuffer<float> xb;
  std::size_t m = 0;
};

inline mlra_lora c_layer(const ModuLoraLayer& L) {
  mlra_lora c{};
  c.q = L.weights->handle();
  c.strategy = static_cast<mlra_strategy>(L.strategy);
  c.rank = static_cast<int64_t>(L.adapter.rank);
  c.alpha = L.adapter.alpha;
  c.a = L.adapter.a.get();
  c.b = L.adapter.b.get();
  c.bias = L.bias.get();
  return c;
}

// layer_forward (lora.cpp:52-72): y = x·Ŵᵀ + (α/r)(x·B)·Aᵀ + bias, f64 host in/out.
inline HostMatrix layer_forward(const ModuLoraLayer& L, const HostMatrix& x, LayerActivations* saved) {
  if (x.cols != L.d_in())
    throw DimensionError("layer '" + L.name + "': input cols " + std::to_string(x.cols) +
                         " != d_in " + std::to_string(L.d_in()));
  LayerActivations s;
  s.m = x.rows;
  s.x = DeviceBuffer<__nv_bfloat16>(x.rows * x.cols);
  s.xb = DeviceBuffer<float>(x.rows * L.adapter.rank);
  if (x.rows) s.x.upload(to_bf16(x.data).data());
  DeviceBuffer<float> y(x.rows * L.d_out());
  const mlra_lora c = c_layer(L);
  check(mlra_lora_forward(&c, s.x.get(), static_cast<int64_t>(x.cols), static_cast<int64_t>(x.rows),
                          y.get(), MLRA_F32, static_cast<int64_t>(L.d_out()), s.xb.get(), nullptr));
  HostMatrix out = detail::download_f32(y, x.rows, L.d_out());
  if (saved) *saved = std::move(s);
  return out;
}

// Tape replay of layer_forward's records (autodiff.cpp:101-193): returns dx
// (empty when !need_dx, as autodiff.cpp:136 skips a frozen input); dA/dB (and
// dbias when trainable) land on the layer for grads_of_adapter.
inline HostMatrix layer_backward(ModuLoraLayer& L, const LayerActivations& s, const HostMatrix& g,
                                 bool need_dx = true) {
  if (g.cols != L.d_out() || g.rows != s.m)
    throw DimensionError("layer '" + L.name + "' backward: grad shape mismatch");
  const std::size_t r = L.adapter.rank;
  DeviceBuffer<__nv_bfloat16> dg(g.rows * g.cols);
  if (g.rows) dg.upload(to_bf16(g.data).data());
  DeviceBuffer<float> dx(need_dx ? s.m * L.d_in() : 0), da(L.d_out() * r), db(L.d_in() * r),
      dbias(L.bias_trainable ? L.d_out() : 0);
  const mlra_lora c = c_layer(L);
  check(mlra_lora_backward(&c, s.x.get(), static_cast<int64_t>(L.d_in()), s.xb.get(), dg.get(),
                           static_cast<int64_t>(L.d_out()), static_cast<int64_t>(s.m),
                           need_dx ? dx.get() : nullptr, MLRA_F32, static_cast<int64_t>(L.d_in()),
                           da.get(), db.get(), L.bias_trainable ? dbias.get() : nullptr, nullptr));
  L.adapter.grad_a = detail::download_f32(da, L.d_out(), r);
  L.adapter.grad_b = detail::download_f32(db, L.d_in(), r);
  if (L.bias_trainable) L.grad_bias = detail::download_f32(dbias, 1, L.d_out());
  L.adapter.has_grad = true;
  return need_dx ? detail::download_f32(dx, s.m, L.d_in()) : HostMatrix();
}

// grads_of_adapter (lora.cpp:74-80): ContractError before backward.
inline std::pair<HostMatrix, HostMatrix> grads_of_adapter(const ModuLoraLayer& L) {
  if (!L.adapter.has_grad) throw ContractError("grads_of_adapter: called before backward()");
  return {L.adapter.grad_a, L.adapter.grad_b};
}

}  // namespace modulora_b200

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
struct IoError : Error {
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
    case MLRA_ERR_FORMAT: {
      uint64_t off = 0;
      const int k = mlra_last_format_error(&off);
      throw FormatError(k >= 0 ? static_cast<FormatError::Kind>(k) : FormatError::Kind::BadField,
                        static_cast<std::size_t>(off), m);
    }
    case MLRA_ERR_IO: throw IoError(m);
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
  void download(T* h, std::size_t count) const {
    if (count > n_) throw ContractError("DeviceBuffer: download past the end");
    if (count) cuda_check(cudaMemcpy(h, p_, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
  }

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

// bitpack.hpp:31 pack(): LSB-first bitstream, code i at bit i*bits (host side,
// for building plugin formats; RangeError on a code wider than `bits`).
inline PackedCodes pack(const std::vector<std::uint32_t>& codes, int bits) {
  if (bits < 1 || bits > 16) throw ConfigError("bitpack: unsupported bit width " + std::to_string(bits));
  PackedCodes p;
  p.bits = bits;
  p.count = codes.size();
  p.words.assign(mlra_packed_word_count(codes.size(), bits), 0u);
  for (std::size_t i = 0; i < codes.size(); ++i) {
    const std::uint32_t c = codes[i];
    if (c >> bits) throw RangeError("bitpack: code " + std::to_string(c) + " out of range");
    const std::uint64_t bit = static_cast<std::uint64_t>(i) * bits;
    const std::uint64_t v = static_cast<std::uint64_t>(c) << (bit & 31);
    p.words[bit >> 5] |= static_cast<std::uint32_t>(v);
    if ((bit & 31) + bits > 32) p.words[(bit >> 5) + 1] |= static_cast<std::uint32_t>(v >> 32);
  }
  return p;
}

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
  // Adopts a handle from another constructor of the C ABI (mlra_cb2_create,
  // mlra_qweight_create_opaque, mlra_checkpoint_upload).
  DeviceQuantizedMatrix(mlra_qweight* h, std::size_t rows, std::size_t cols)
      : h_(h), rows_(rows), cols_(cols) {}
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

// ----------------------------------------------------------------- quantize.hpp:59-75
// quantize_rtn / quantize_optq on the device (mlra_quantize_rtn / mlra_quantize_optq),
// bit-identical to the reference; host matrices in, the host QuantizedMatrix out.
namespace detail {
inline QuantizedMatrix download_q(std::size_t rows, std::size_t cols, int bits, std::size_t g,
                                  DeviceBuffer<std::uint32_t>& words, DeviceBuffer<float>& sc,
                                  DeviceBuffer<float>& z, std::size_t nw, std::size_t ng) {
  QuantizedMatrix q;
  q.rows = rows;
  q.cols = cols;
  q.bits = bits;
  q.group_size = g;
  q.codes.bits = bits;
  q.codes.count = rows * cols;
  q.codes.words.resize(nw);
  q.scales.resize(ng);
  q.zeros.resize(ng);
  cuda_check(cudaDeviceSynchronize(), "quantize");
  words.download(q.codes.words.data(), nw);
  sc.download(q.scales.data(), ng);
  z.download(q.zeros.data(), ng);
  return q;
}
}  // namespace detail

inline QuantizedMatrix quantize_rtn(const HostMatrix& w, int bits, std::size_t group_size = 0) {
  const std::size_t g = group_size ? group_size : w.cols;
  const std::size_t nw = w.rows && w.cols ? mlra_packed_word_count(w.rows * w.cols, bits) : 0;
  const std::size_t ng = g && w.cols % g == 0 ? w.rows * (w.cols / g) : 0;
  DeviceBuffer<double> dw(std::max<std::size_t>(w.data.size(), 1));
  if (!w.data.empty()) dw.upload(w.data.data());
  DeviceBuffer<std::uint32_t> words(std::max<std::size_t>(nw, 1));
  DeviceBuffer<float> sc(std::max<std::size_t>(ng, 1)), z(std::max<std::size_t>(ng, 1));
  check(mlra_quantize_rtn(dw.get(), MLRA_F64, static_cast<int64_t>(w.rows),
                          static_cast<int64_t>(w.cols), bits, static_cast<int64_t>(group_size),
                          words.get(), sc.get(), z.get(), nullptr));
  return detail::download_q(w.rows, w.cols, bits, g, words, sc, z, nw, ng);
}

inline QuantizedMatrix quantize_optq(const HostMatrix& w, const HostMatrix& calib, int bits,
                                     std::size_t group_size = 0, double damping = 0.01) {
  if (calib.cols != w.cols)
    throw DimensionError("optq: calibration must be [m x " + std::to_string(w.cols) + "]");
  const std::size_t g = group_size ? group_size : w.cols;
  const std::size_t nw = w.rows && w.cols ? mlra_packed_word_count(w.rows * w.cols, bits) : 0;
  const std::size_t ng = g && w.cols % g == 0 ? w.rows * (w.cols / g) : 0;
  DeviceBuffer<double> dw(std::max<std::size_t>(w.data.size(), 1)),
      dx(std::max<std::size_t>(calib.data.size(), 1));
  if (!w.data.empty()) dw.upload(w.data.data());
  if (!calib.data.empty()) dx.upload(calib.data.data());
  DeviceBuffer<std::uint32_t> words(std::max<std::size_t>(nw, 1));
  DeviceBuffer<float> sc(std::max<std::size_t>(ng, 1)), z(std::max<std::size_t>(ng, 1));
  check(mlra_quantize_optq(dw.get(), dx.get(), static_cast<int64_t>(w.rows),
                           static_cast<int64_t>(w.cols), static_cast<int64_t>(calib.rows), bits,
                           static_cast<int64_t>(group_size), damping, words.get(), sc.get(),
                           z.get(), nullptr));
  return detail::download_q(w.rows, w.cols, bits, g, words, sc, z, nw, ng);
}

// ----------------------------------------------------------------- quantize.hpp:91-106
// The black-box Quantizer plugin in device form (include/mlra.h mlra_hook):
// the reference's override point is Quantizer::matvec / matvec_transposed;
// here a plugin overrides materialize_tile(), the dequantization of one tile
// of Ŵ into device memory on a stream, and the library runs its own tcgen05
// GEMM over hook-materialized slabs under QuantizerMatvec.
class Quantizer {
 public:
  virtual ~Quantizer() = default;
  virtual std::string_view name() const = 0;
  virtual mlra_status materialize_tile(const mlra_qweight* q, int64_t row0, int64_t nrows,
                                       int64_t col0, int64_t ncols, void* out, mlra_dtype dtype,
                                       int64_t ld, cudaStream_t stream) const = 0;
  // The C-ABI hook (valid while this object lives).
  const mlra_hook* hook() const {
    name_ = std::string(name());
    hook_.name = name_.c_str();
    hook_.state = const_cast<Quantizer*>(this);
    hook_.materialize = [](void* st, const mlra_qweight* q, int64_t r0, int64_t nr, int64_t c0,
                           int64_t nc, void* out, mlra_dtype dt, int64_t ld,
                           void* stream) -> mlra_status {
      try {
        return static_cast<const Quantizer*>(st)->materialize_tile(
            q, r0, nr, c0, nc, out, dt, ld, static_cast<cudaStream_t>(stream));
      } catch (...) {
        return MLRA_ERR_CONTRACT;  // exceptions do not cross the C ABI
      }
    };
    return &hook_;
  }

 private:
  mutable mlra_hook hook_{};
  mutable std::string name_;
};

// The reference test plugin (test_lowprec.cpp:354-377): twice the default product.
class DoublingQuantizer final : public Quantizer {
 public:
  std::string_view name() const override { return "doubling"; }
  mlra_status materialize_tile(const mlra_qweight* q, int64_t r0, int64_t nr, int64_t c0,
                               int64_t nc, void* out, mlra_dtype dt, int64_t ld,
                               cudaStream_t st) const override;
};

// Built-in non-affine plugin "cb2" (mlra_cb2_create): 2 bits per weight as one
// u16 code per 8 entries (8-bit codebook index + 8 sign bits), f32 scale per
// (row, group). Returns the frozen matrix, dequantized only through its hook.
inline std::shared_ptr<const DeviceQuantizedMatrix> upload_cb2(
    std::size_t rows, std::size_t cols, std::size_t group, const std::vector<std::uint16_t>& codes,
    const std::vector<float>& codebook, const std::vector<float>& scales, cudaStream_t st = nullptr) {
  if (codes.size() != rows * (cols / 8) || codebook.size() != 256 * 8 ||
      (group && scales.size() != rows * (cols / group)))
    throw FormatError(FormatError::Kind::BadField, 0, "cb2: buffer sizes do not match the shape");
  mlra_qweight* h = nullptr;
  check(mlra_cb2_create(static_cast<int64_t>(rows), static_cast<int64_t>(cols),
                        static_cast<int64_t>(group), codes.data(), codebook.data(), scales.data(),
                        st, &h));
  return std::make_shared<const DeviceQuantizedMatrix>(h, rows, cols);
}

// Built-in plugin "lut" (mlra_lut_create): the reference's b-bit bitstream of
// level indices (b in {2, 3, 4}), a table of 2^b f32 levels (e.g. NF4) and an
// f32 scale per (row, group); Ŵ = RN_f32(s · levels[c]). An ordinary frozen
// matrix: materialize() and the fused GEMM decode the table on the device.
inline std::shared_ptr<const DeviceQuantizedMatrix> upload_lut(
    std::size_t rows, std::size_t cols, std::size_t group, const PackedCodes& codes,
    const std::vector<float>& levels, const std::vector<float>& scales, cudaStream_t st = nullptr) {
  if (codes.bits < 1 || codes.bits > 4 || levels.size() != (std::size_t{1} << codes.bits) ||
      !group || scales.size() != rows * (cols / group) || codes.count != rows * cols)
    throw FormatError(FormatError::Kind::BadField, 0, "lut: buffer sizes do not match the shape");
  mlra_qweight* h = nullptr;
  check(mlra_lut_create(static_cast<int64_t>(rows), static_cast<int64_t>(cols), codes.bits,
                        static_cast<int64_t>(group), codes.words.data(), codes.words.size(),
                        levels.data(), scales.data(), st, &h));
  return std::make_shared<const DeviceQuantizedMatrix>(h, rows, cols);
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
  std::shared_ptr<const Quantizer> matvec_hook;  // optional, QuantizerMatvec only
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
  check(mlra_lp_forward_ex(q, static_cast<mlra_strategy>(ctx.strategy),
                           ctx.matvec_hook ? ctx.matvec_hook->hook() : nullptr, dx.get(),
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
  check(mlra_lp_backward_ex(q, static_cast<mlra_strategy>(ctx.strategy),
                            ctx.matvec_hook ? ctx.matvec_hook->hook() : nullptr, dg.get(),
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
  std::shared_ptr<const Quantizer> matvec_hook;  // lora.hpp:47
  std::size_t d_in() const { return weights->cols(); }
  std::size_t d_out() const { return weights->rows(); }
};

// init_adapter (lora.cpp:14-32): A = 0, B = gaussian(d_in x r, Rng(seed), 0, 0.02) from the
// reference's own stream (mlra_gaussian_fill: bit-identical f64 values, stored as fp32);
// ConfigError on rank 0 / alpha <= 0.
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
  std::vector<double> b64(d_in * rank);
  mlra_gaussian_fill(seed, b64.data(), b64.size(), 0.0, kAdapterInitStd);
  for (std::size_t i = 0; i < hb.size(); ++i) hb[i] = static_cast<float>(b64[i]);
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
  c.hook = L.matvec_hook ? L.matvec_hook->hook() : nullptr;
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

inline mlra_status DoublingQuantizer::materialize_tile(const mlra_qweight* q, int64_t r0,
                                                     int64_t nr, int64_t c0, int64_t nc, void* out,
                                                     mlra_dtype dt, int64_t ld,
                                                     cudaStream_t st) const {
  // default dequantization, then x2 on the host side of a round trip: a plugin
  // may do anything; this one stays simple (exact: x2 is exact in bf16 / f32)
  if (mlra_status s = mlra_materialize_tile(q, r0, nr, c0, nc, out, dt, ld, st)) return s;
  const std::size_t es = dt == MLRA_F32 ? 4 : 2;
  std::vector<unsigned char> h(static_cast<std::size_t>(nr * ld) * es);
  if (cudaMemcpyAsync(h.data(), out, h.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return MLRA_ERR_CUDA;
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t j = 0; j < nc; ++j) {
      const std::size_t k = static_cast<std::size_t>(i * ld + j);
      if (dt == MLRA_F32) {
        float* f = reinterpret_cast<float*>(h.data()) + k;
        *f *= 2.0f;
      } else {
        __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(h.data()) + k;
        *b = __float2bfloat16_rn(2.0f * __bfloat162float(*b));
      }
    }
  if (cudaMemcpyAsync(out, h.data(), h.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return MLRA_ERR_CUDA;
  return MLRA_OK;
}

// ----------------------------------------------------------------- train.hpp:51-70
// AdamW (train.cpp:75-134) over device f64 parameters: masters and moments stay
// in HBM, one fused launch per step, bit-identical to the reference's f64
// arithmetic given the same gradients. NumericError (naming the parameter)
// on a non-finite gradient, with the earlier parameters updated.
class AdamW {
 public:
  AdamW(double beta1, double beta2, double eps, double weight_decay)
      : cfg_{beta1, beta2, eps, weight_decay} {}
  // params: device f64 [n] (flat bucket, updated in place); grads: device f32 or
  // f64 [n]; sizes/names: the parameter list laid out back to back.
  void step(double* params, const void* grads, mlra_dtype grad_dtype,
            const std::vector<std::size_t>& sizes, const std::vector<std::string>& names,
            std::size_t step_index, double lr, float* params_f32 = nullptr,
            cudaStream_t st = nullptr) {
    if (sizes.size() != names.size()) throw ContractError("adamw: params/names size mismatch");
    std::size_t n = 0;
    std::vector<int64_t> offs{0};
    for (std::size_t s : sizes) offs.push_back(static_cast<int64_t>(n += s));
    if (m_.size() == 0) {
      sizes_ = sizes;
      m_ = DeviceBuffer<double>(n);
      v_ = DeviceBuffer<double>(n);
      cuda_check(cudaMemsetAsync(m_.get(), 0, n * 8, st), "cudaMemsetAsync");
      cuda_check(cudaMemsetAsync(v_.get(), 0, n * 8, st), "cudaMemsetAsync");
    } else if (sizes != sizes_) {
      throw ContractError("adamw: parameter list changed between steps");
    }
    const mlra_status s = mlra_adamw_step(&cfg_, static_cast<int64_t>(step_index), lr,
                                          static_cast<int64_t>(sizes.size()), offs.data(), params,
                                          m_.get(), v_.get(), grads, grad_dtype, params_f32,
                                          nullptr, st);
    if (s == MLRA_ERR_NUMERIC) {
      const std::string m = mlra_last_error();
      const std::size_t i = std::stoul(m.substr(m.find('#') + 1));
      throw NumericError("adamw: non-finite gradient for parameter '" + names[i] + "' at step " +
                         std::to_string(step_index));
    }
    check(s);
  }

 private:
  mlra_adamw cfg_;
  DeviceBuffer<double> m_, v_;
  std::vector<std::size_t> sizes_;
};

// ----------------------------------------------------------------- data parallelism
// One sum all-reduce of the flat fp32 LoRA-gradient bucket per step (NCCL, loaded
// by libmlra at run time). Rank 0 calls unique_id() and shares the bytes.
class GradExchange {
 public:
  static std::vector<unsigned char> unique_id() {
    std::vector<unsigned char> id(128);
    check(mlra_dp_unique_id(id.data()));
    return id;
  }
  GradExchange(int rank, int world, const std::vector<unsigned char>& id) {
    if (id.size() != 128) throw ContractError("dp: unique id must be 128 bytes");
    check(mlra_dp_init(rank, world, id.data(), &h_));
  }
  ~GradExchange() { mlra_dp_destroy(h_); }
  GradExchange(const GradExchange&) = delete;
  GradExchange& operator=(const GradExchange&) = delete;
  void allreduce(float* bucket, std::size_t count, cudaStream_t st = nullptr) {
    check(mlra_allreduce_lora_grads(h_, bucket, count, st));
  }

 private:
  mlra_dp* h_ = nullptr;
};

// ----------------------------------------------------------------- checkpoint.hpp:36-67
// The .mlra format -> device: parse + validate like load_model (FormatError
// kinds/offsets, IoError), upload layers verbatim, save byte-identically.
class Checkpoint {
 public:
  explicit Checkpoint(const std::string& path) { check(mlra_checkpoint_load(path.c_str(), &h_)); }
  ~Checkpoint() { mlra_checkpoint_free(h_); }
  Checkpoint(const Checkpoint&) = delete;
  Checkpoint& operator=(const Checkpoint&) = delete;
  std::size_t size() const { return static_cast<std::size_t>(mlra_checkpoint_layer_count(h_)); }
  mlra_ckpt_layer layer(std::size_t i) const {
    mlra_ckpt_layer o{};
    check(mlra_checkpoint_layer(h_, static_cast<int64_t>(i), &o));
    return o;
  }
  std::uint64_t frozen_state_hash() const { return mlra_checkpoint_frozen_hash(h_); }
  std::uint64_t file_hash() const { return mlra_checkpoint_file_hash(h_); }
  std::shared_ptr<const DeviceQuantizedMatrix> upload(std::size_t i, cudaStream_t st = nullptr) const {
    const mlra_ckpt_layer L = layer(i);
    mlra_qweight* q = nullptr;
    check(mlra_checkpoint_upload(h_, static_cast<int64_t>(i), st, &q));
    return std::make_shared<const DeviceQuantizedMatrix>(q, static_cast<std::size_t>(L.rows),
                                                         static_cast<std::size_t>(L.cols));
  }
  void set_adapter(std::size_t i, const HostMatrix& a, const HostMatrix& b) {
    const mlra_ckpt_layer L = layer(i);
    if (a.rows != static_cast<std::size_t>(L.rows) || a.cols != static_cast<std::size_t>(L.rank) ||
        b.rows != static_cast<std::size_t>(L.cols) || b.cols != static_cast<std::size_t>(L.rank))
      throw DimensionError("checkpoint: adapter shape mismatch");
    check(mlra_checkpoint_set_adapter(h_, static_cast<int64_t>(i), a.data.data(), b.data.data()));
  }
  void save(const std::string& path) const { check(mlra_checkpoint_save(h_, path.c_str())); }

 private:
  mlra_checkpoint* h_ = nullptr;
};

}  // namespace modulora_b200

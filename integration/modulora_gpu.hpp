// modulora_gpu.hpp — the reference-side binding of libmlra (the drop-in a
// maintainer adds to the reference tree).
//
// Compiled AGAINST THE REFERENCE'S OWN HEADERS (modulora/autodiff.hpp,
// lowprec_linear.hpp, lora.hpp, errors.hpp) and linked with the reference's
// objects plus libmlra.so. It plugs the B200 path into the reference's tape at
// the two extension points the reference exposes:
//
//  * GpuLpLinearFunction — a CustomFunction (autodiff.hpp:77-89) replacing
//    LpLinearFunction (lowprec_linear.hpp:96-112, lowprec_linear.cpp:249-266):
//    forward = mlra_lp_forward_ex, backward = mlra_lp_backward_ex (Ŵ
//    re-dequantized inside the fused kernel, never cached; ctx.saved holds the
//    device weight handle only). layer_forward (lora.cpp:52-72) keeps its
//    seven records when built with gpu_base_layer_forward below; only the
//    register_custom line (lora.cpp:64-66) changes.
//  * GpuModuLoraFunction — the whole layer as ONE tape record whose inputs are
//    {x, A, B, bias}: forward = mlra_lora_forward (x·B and the LoRA term fused
//    into the base GEMM as an extra K block), backward = mlra_lora_backward
//    (dX, dA, dB, dbias), so grads_of_adapter (lora.cpp:74-80) sees the
//    device-computed adapter gradients through the tape's accumulate_grad.
//
// Host f64 DenseMatrix values cross the boundary as bf16 activations and fp32
// factors (the device arithmetic); libmlra status codes become
// the reference's exception types (errors.hpp:15-63). Header-only; needs
// <cuda_runtime.h> and include/mlra.h.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "mlra.h"
#include "modulora/autodiff.hpp"
#include "modulora/errors.hpp"
#include "modulora/lora.hpp"
#include "modulora/lowprec_linear.hpp"
#include "modulora/quantize.hpp"

namespace modulora::gpu {

// libmlra status -> the reference's exception taxonomy (include/mlra.h:41-52).
inline void check(mlra_status st) {
  if (st == MLRA_OK) return;
  const std::string m = mlra_last_error();
  switch (st) {
    case MLRA_ERR_DIMENSION: throw DimensionError(m);
    case MLRA_ERR_CONFIG: throw ConfigError(m);
    case MLRA_ERR_RANGE: throw RangeError(m);
    case MLRA_ERR_CONTRACT: throw ContractError(m);
    case MLRA_ERR_NUMERIC: throw NumericError(m);
    case MLRA_ERR_IO: throw IoError(m);
    case MLRA_ERR_FORMAT: {
      uint64_t off = 0;
      const int k = mlra_last_format_error(&off);
      throw FormatError(static_cast<FormatError::Kind>(k < 0 ? 3 : k), off, m);
    }
    default: throw Error("libmlra: " + m);  // CUDA / unsupported device
  }
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string("libmlra binding: ") + what + ": " +
                                    cudaGetErrorString(e));
}

// Device buffer owned by the binding (freed on destruction).
struct DeviceBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : bytes(n) {
    if (n) cuda_check(cudaMalloc(&p, n), "cudaMalloc");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// f64 -> RN-even bf16 bits (via the f32 rounding the device applies).
inline uint16_t to_bf16(double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return static_cast<uint16_t>((u >> 16) | 0x40);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

// A DenseMatrix to the device: bf16 (activations) or fp32 (factors, bias).
inline std::shared_ptr<DeviceBuffer> upload_bf16(const DenseMatrix& a) {
  std::vector<uint16_t> h(a.size());
  for (size_t i = 0; i < a.size(); ++i) h[i] = to_bf16(a.data()[i]);
  auto d = std::make_shared<DeviceBuffer>(h.size() * 2);
  if (!h.empty()) cuda_check(cudaMemcpy(d->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "H2D");
  return d;
}
inline std::shared_ptr<DeviceBuffer> upload_f32(const DenseMatrix& a) {
  std::vector<float> h(a.size());
  for (size_t i = 0; i < a.size(); ++i) h[i] = static_cast<float>(a.data()[i]);
  auto d = std::make_shared<DeviceBuffer>(h.size() * 4);
  if (!h.empty()) cuda_check(cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "H2D");
  return d;
}
inline DenseMatrix download_f32(const DeviceBuffer& d, size_t rows, size_t cols) {
  std::vector<float> h(rows * cols);
  if (!h.empty()) cuda_check(cudaMemcpy(h.data(), d.p, h.size() * 4, cudaMemcpyDeviceToHost), "D2H");
  return DenseMatrix(rows, cols, std::vector<double>(h.begin(), h.end()));
}

// One upload per frozen QuantizedMatrix (quantize.hpp:29-48), reference
// bitstream words verbatim (validated on the device exactly as
// QuantizedMatrix::validate, quantize.cpp:82-115).
struct DeviceWeights {
  mlra_qweight* h = nullptr;
  size_t rows = 0, cols = 0;
  explicit DeviceWeights(const QuantizedMatrix& q) : rows(q.rows), cols(q.cols) {
    check(mlra_qweight_create(static_cast<int64_t>(q.rows), static_cast<int64_t>(q.cols), q.bits,
                              static_cast<int64_t>(q.group_size), q.codes.words.data(),
                              q.codes.words.size(), q.codes.count, q.scales.data(),
                              q.zeros.data(), q.scales.size(), nullptr, &h));
  }
  DeviceWeights(const DeviceWeights&) = delete;
  DeviceWeights& operator=(const DeviceWeights&) = delete;
  ~DeviceWeights() { mlra_qweight_destroy(h); }
};

inline mlra_strategy to_c(MaterializationStrategy s) {
  switch (s) {
    case MaterializationStrategy::WeightMaterialize: return MLRA_WEIGHT;
    case MaterializationStrategy::RowMaterialize: return MLRA_ROW;
    default: return MLRA_MATVEC;
  }
}

// LpLinearFunction on the B200 (lowprec_linear.cpp:249-266 + lp_forward /
// lp_backward :150-247): exactly one input; the only gradient is dX.
class GpuLpLinearFunction final : public CustomFunction {
 public:
  GpuLpLinearFunction(std::shared_ptr<const DeviceWeights> w, MaterializationStrategy s)
      : w_(std::move(w)), s_(to_c(s)) {}
  std::string_view name() const override { return "lp_linear_gpu"; }
  DenseMatrix forward(FunctionContext& ctx, std::span<const DenseMatrix* const> in) override {
    if (in.size() != 1) throw ContractError("lp_linear: expected exactly one input");
    ctx.saved = w_;  // the packed-code handle only, never Ŵ
    return run(*in[0], false);
  }
  std::vector<std::optional<DenseMatrix>> backward(FunctionContext&, const DenseMatrix& g) override {
    std::vector<std::optional<DenseMatrix>> r;
    r.emplace_back(run(g, true));  // re-dequantized inside the fused kernel
    return r;
  }

 private:
  DenseMatrix run(const DenseMatrix& a, bool bwd) const {
    if (!w_) throw ContractError("lp_linear: missing quantized weights");
    const size_t in_cols = bwd ? w_->rows : w_->cols, out_cols = bwd ? w_->cols : w_->rows;
    if (a.cols() != in_cols)
      throw DimensionError(std::string(bwd ? "lp_backward: grad cols " : "lp_forward: input cols ") +
                           std::to_string(a.cols()) + " != weight " + (bwd ? "rows " : "cols ") +
                           std::to_string(in_cols));
    const size_t m = a.rows();
    if (m == 0) return DenseMatrix(0, out_cols);
    auto da = upload_bf16(a);
    DeviceBuffer out(m * out_cols * 4);
    const int64_t mi = static_cast<int64_t>(m);
    if (!bwd)
      check(mlra_lp_forward_ex(w_->h, s_, nullptr, da->p, static_cast<int64_t>(in_cols), mi, out.p,
                               MLRA_F32, static_cast<int64_t>(out_cols), nullptr));
    else
      check(mlra_lp_backward_ex(w_->h, s_, nullptr, da->p, static_cast<int64_t>(in_cols), mi,
                                out.p, MLRA_F32, static_cast<int64_t>(out_cols), nullptr));
    return download_f32(out, m, out_cols);
  }
  std::shared_ptr<const DeviceWeights> w_;
  mlra_strategy s_;
};

// layer_forward (lora.cpp:52-72) with the base on the B200: the same seven
// records, the lp_linear record backed by GpuLpLinearFunction.
inline Variable gpu_base_layer_forward(Tape& t, ModuLoraLayer& layer, const Variable& x,
                                       std::shared_ptr<const DeviceWeights> w) {
  if (x.cols() != layer.d_in())
    throw DimensionError("layer '" + layer.name + "': input cols " + std::to_string(x.cols()) +
                         " != d_in " + std::to_string(layer.d_in()));
  Variable base =
      register_custom(t, std::make_shared<GpuLpLinearFunction>(std::move(w), layer.strategy), {x});
  Variable xb = matmul(t, x, layer.adapter.b);
  Variable ab = matmul(t, xb, transpose(t, layer.adapter.a));
  Variable low_rank = scalar_mul(t, ab, layer.adapter.scaling());
  return bias_add(t, add(t, base, low_rank), layer.bias);
}

// The whole ModuLoRA layer as one record on the reference tape: inputs
// {x, A, B, bias}, one mlra_lora_forward / mlra_lora_backward each way.
class GpuModuLoraFunction final : public CustomFunction {
 public:
  GpuModuLoraFunction(std::shared_ptr<const DeviceWeights> w, MaterializationStrategy s,
                      size_t rank, double alpha)
      : w_(std::move(w)), s_(to_c(s)), rank_(rank), alpha_(alpha) {}
  std::string_view name() const override { return "modulora_layer_gpu"; }

  DenseMatrix forward(FunctionContext& ctx, std::span<const DenseMatrix* const> in) override {
    if (in.size() != 4) throw ContractError("modulora_layer_gpu: expected {x, A, B, bias}");
    const DenseMatrix &x = *in[0], &a = *in[1], &b = *in[2], &bias = *in[3];
    if (x.cols() != w_->cols)
      throw DimensionError("layer: input cols " + std::to_string(x.cols()) + " != d_in " +
                           std::to_string(w_->cols));
    auto st = std::make_shared<Saved>();
    st->m = x.rows();
    st->x = upload_bf16(x);
    st->a = upload_f32(a);
    st->b = upload_f32(b);
    st->bias = upload_f32(bias);
    st->xb = std::make_shared<DeviceBuffer>(st->m * rank_ * 4);
    DeviceBuffer y(st->m * w_->rows * 4);
    const mlra_lora L = lora(*st);
    if (st->m)
      check(mlra_lora_forward(&L, st->x->p, static_cast<int64_t>(w_->cols),
                              static_cast<int64_t>(st->m), y.p, MLRA_F32,
                              static_cast<int64_t>(w_->rows), st->xb->as<float>(), nullptr));
    ctx.saved = st;  // x and xb on the device; Ŵ is never saved
    return download_f32(y, st->m, w_->rows);
  }

  std::vector<std::optional<DenseMatrix>> backward(FunctionContext& ctx,
                                                   const DenseMatrix& g) override {
    auto st = std::any_cast<std::shared_ptr<Saved>>(ctx.saved);
    if (g.cols() != w_->rows || g.rows() != st->m)
      throw DimensionError("layer backward: grad shape mismatch");
    auto dg = upload_bf16(g);
    DeviceBuffer dx(st->m * w_->cols * 4), da(w_->rows * rank_ * 4), db(w_->cols * rank_ * 4),
        dbias(w_->rows * 4);
    const mlra_lora L = lora(*st);
    check(mlra_lora_backward(&L, st->x->p, static_cast<int64_t>(w_->cols), st->xb->as<float>(),
                             dg->p, static_cast<int64_t>(w_->rows), static_cast<int64_t>(st->m),
                             dx.p, MLRA_F32, static_cast<int64_t>(w_->cols), da.as<float>(),
                             db.as<float>(), dbias.as<float>(), nullptr));
    std::vector<std::optional<DenseMatrix>> r;
    r.emplace_back(download_f32(dx, st->m, w_->cols));
    r.emplace_back(download_f32(da, w_->rows, rank_));
    r.emplace_back(download_f32(db, w_->cols, rank_));
    DenseMatrix bsum = download_f32(dbias, 1, w_->rows);
    r.emplace_back(std::move(bsum));
    return r;
  }

 private:
  struct Saved {
    size_t m = 0;
    std::shared_ptr<DeviceBuffer> x, a, b, bias, xb;
  };
  mlra_lora lora(const Saved& st) const {
    mlra_lora L{};
    L.q = w_->h;
    L.strategy = s_;
    L.rank = static_cast<int64_t>(rank_);
    L.alpha = alpha_;
    L.a = st.a->as<float>();
    L.b = st.b->as<float>();
    L.bias = st.bias->as<float>();
    L.hook = nullptr;
    return L;
  }
  std::shared_ptr<const DeviceWeights> w_;
  mlra_strategy s_;
  size_t rank_;
  double alpha_;
};

// The whole layer on the B200 as one tape record (grads_of_adapter and the
// bias gradient arrive through the tape as for the CPU layer).
inline Variable gpu_layer_forward(Tape& t, ModuLoraLayer& layer, const Variable& x,
                                  std::shared_ptr<const DeviceWeights> w) {
  return register_custom(t,
                         std::make_shared<GpuModuLoraFunction>(std::move(w), layer.strategy,
                                                               layer.adapter.rank,
                                                               layer.adapter.alpha),
                         {x, layer.adapter.a, layer.adapter.b, layer.bias});
}

}  // namespace modulora::gpu

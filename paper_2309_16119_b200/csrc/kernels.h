// kernels.h — launchers of the non-GEMM kernels (materialize.cu, lora_thin.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mlra {

// Counts every kernel this library launches (mlra_kernel_launches()).
void note_launch();

cudaError_t launch_relayout(const uint32_t* src, int64_t rows, int64_t cols, int bits,
                            int64_t row_words, int64_t rows_pad, uint32_t* dst, cudaStream_t st);
cudaError_t launch_grid(const float* scales, const float* zeros, int64_t rows, int64_t ng,
                        int64_t rows_pad, int64_t ng_pad, int bits, float2* grid,
                        int* n_uncertified, cudaStream_t st);
cudaError_t launch_materialize(const QWeightDev& q, int64_t row0, int64_t nrows, void* out,
                               int64_t ld, bool f32, cudaStream_t st);

// out[m x r] = act[m x kd] · W[kd x r] (fp32); pad[t, j] = bf16(scale * out[t, j]).
cudaError_t launch_rowdot(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const float* W, int64_t r, float scale, float* out,
                          __nv_bfloat16* pad, int64_t ldp, cudaStream_t st);
// out[nd x r] += scale · actᵀ[nd x m] · V[m x r]; colsum[n] += Σ_t act[t, n] (optional).
cudaError_t launch_coldot(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const float* V, int64_t r, float scale, float* out, float* colsum,
                          cudaStream_t st);
cudaError_t launch_pad_bf16(const float* src, int64_t rows, int64_t cols, int64_t lds,
                            __nv_bfloat16* dst, int64_t rows_pad, int64_t ldd, cudaStream_t st);

}  // namespace mlra

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

// Skinny rank-r products on tensor cores (thin_mma.cu); r <= 64 per call. Factors are passed
// transposed and split into bf16 hi/lo planes [thin_rows(r) x ld] (launch_split_t).
int thin_rows(int64_t r, bool ones);
cudaError_t launch_split_t(const float* src, int64_t rows, int64_t r, int64_t lds, bool ones,
                           __nv_bfloat16* hi, __nv_bfloat16* lo, int64_t ldt, cudaStream_t st);
cudaError_t launch_scale_pad(const float* src, int64_t m, int64_t r, float scale,
                             __nv_bfloat16* pad, int64_t ldp, cudaStream_t st);
// out[m x r] += act[m x kd] · W      (W given as Wt hi/lo [rows x ldw])
cudaError_t launch_rowmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const __nv_bfloat16* wt_hi, const __nv_bfloat16* wt_lo, int64_t ldw,
                          float* out, int64_t ldo, int64_t r, cudaStream_t st);
// out[nd x r] += scale · actᵀ · V    (V given as Vt hi/lo [rows x ldv]); colsum[n] += Σ_t act
cudaError_t launch_colmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const __nv_bfloat16* vt_hi, const __nv_bfloat16* vt_lo, int64_t ldv,
                          float scale, float* out, int64_t ldo, int64_t r, float* colsum,
                          cudaStream_t st);
cudaError_t launch_pad_bf16(const float* src, int64_t rows, int64_t cols, int64_t lds,
                            __nv_bfloat16* dst, int64_t rows_pad, int64_t ldd, cudaStream_t st);

}  // namespace mlra

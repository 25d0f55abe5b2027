// kernels.h — launchers of the non-GEMM kernels (materialize.cu, lora_thin.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mlra {

// Counts every kernel this library launches (mlra_kernel_launches()).
void note_launch();

// Programmatic dependent launch for the layer-pass kernels (prep, skinny
// products, fused GEMMs): the kernel may start while its stream predecessor
// drains and synchronises with it through pdl_wait (ptx.cuh). MLRA_PDL=0
// launches them classically (A/B switch).
bool pdl_enabled();
// dev-only host profile of launches (MLRA_HOSTPROF, capi.cu)
struct HostLaunchTimer {
  void* impl;
  HostLaunchTimer();
  ~HostLaunchTimer();
};
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, bool pdl, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
  note_launch();
  HostLaunchTimer lt;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

cudaError_t launch_relayout(const uint32_t* src, int64_t rows, int64_t cols, int bits,
                            int64_t row_words, int64_t rows_pad, uint32_t* dst, cudaStream_t st);
cudaError_t launch_grid(const float* scales, const float* zeros, int64_t rows, int64_t ng,
                        int64_t rows_pad, int64_t ng_pad, int bits, float2* grid,
                        int* n_uncertified, cudaStream_t st);
cudaError_t launch_materialize(const QWeightDev& q, int64_t row0, int64_t nrows, void* out,
                               int64_t ld, bool f32, cudaStream_t st);
cudaError_t launch_materialize_tile(const QWeightDev& q, int64_t row0, int64_t nrows, int64_t col0,
                                    int64_t ncols, void* out, int64_t ld, bool f32,
                                    cudaStream_t st);
cudaError_t launch_cb2_materialize(const Cb2Dev& c, int64_t row0, int64_t nrows, int64_t col0,
                                   int64_t ncols, void* out, int64_t ld, bool f32,
                                   cudaStream_t st);

// RTN quantize (quantize.cu): w device f64/f32 [rows x cols] -> reference bitstream words
// [nwords] + f32 scales / zeros [rows x cols/group]
cudaError_t launch_quantize_rtn(const void* w, bool f64, int64_t rows, int64_t cols, int64_t group,
                                int bits, uint32_t* words, uint64_t nwords, float* scales,
                                float* zeros, cudaStream_t st);

// compute_grid (quantize.cpp:24-36) per (row, group) of a device f64 matrix
cudaError_t launch_rtn_grid(const double* w, int64_t rows, int64_t cols, int64_t group, int bits,
                            float* scales, float* zeros, cudaStream_t st);

// OPTQ (optq.cu): build_optq_workspace (quantize.cpp:186-211) — hessian / upper [n x n],
// scratch 2 n^2 doubles, bad[2] = first failing pivot of the two factorizations (init INT_MAX)
cudaError_t launch_optq_workspace(const double* calib, int64_t m, int64_t n, double damping,
                                  double* hessian, double* upper, double* scratch, int* bad,
                                  cudaStream_t st);
// the column sweep (quantize.cpp:231-252) + packing; e_scratch [rows x cols] f64,
// codes [rows x cols] u32
cudaError_t launch_optq_sweep(const double* w, const double* upper, int64_t rows, int64_t cols,
                              int64_t group, int bits, const float* scales, const float* zeros,
                              double* e_scratch, uint32_t* codes, uint32_t* words, uint64_t nwords,
                              cudaStream_t st);

// AdamW (optim.cu): host-evaluated constants of AdamW::step (train.cpp:99-101, :122-127).
struct AdamwConsts {
  double beta1, one_m_beta1, beta2, one_m_beta2, bc1, bc2, lr, eps, decay;
};
// Parameter segment offsets passed by value (kernel parameter space), so a step
// needs no host->device copy and can be captured in a CUDA graph.
constexpr int kAdamwMaxSegs = 1024;
struct AdamwSegs {
  int64_t off[kAdamwMaxSegs + 1];
};
// first_bad: device int (set to the first parameter with a non-finite gradient,
// any value >= nseg when none), or null for no check
cudaError_t launch_adamw(const void* grad, bool grad_f64, int64_t n, const AdamwSegs& offs, int nseg,
                         int* first_bad, double* p, double* m, double* v, float* p32,
                         const AdamwConsts& c, cudaStream_t st);

// Batched small jobs of one layer pass, one launch (thin_mma.cu k_prep).
struct PrepTask {
  enum Kind : int { kZeroF32 = 0, kZeroBf16 = 1, kSplitT = 2, kPadBf16 = 3 };
  int kind;
  int ones;            // kSplitT: append a ones row at index cols
  const float* src;
  void* dst;
  void* dst2;          // kSplitT: lo plane
  int64_t rows, cols;  // source extent (kSplitT: rows = source rows, cols = r)
  int64_t lds;         // source leading dimension
  int64_t rows_out;    // output rows
  int64_t ldd;         // output leading dimension
  float scale;         // kPadBf16
};
constexpr int kMaxPrep = 16;
struct PrepBatch {
  PrepTask t[kMaxPrep];
  int64_t offs[kMaxPrep + 1];
  int n = 0;
  void add(const PrepTask& k, int64_t count) {
    if (n == 0) offs[0] = 0;
    t[n] = k;
    offs[n + 1] = offs[n] + count;
    ++n;
  }
  void zero_f32(float* p, int64_t count) {
    add(PrepTask{PrepTask::kZeroF32, 0, nullptr, p, nullptr, 0, 0, 0, 0, 0, 0.f}, count);
  }
  void zero_bf16(void* p, int64_t count) {
    add(PrepTask{PrepTask::kZeroBf16, 0, nullptr, p, nullptr, 0, 0, 0, 0, 0, 0.f}, count);
  }
  // hi/lo bf16 planes [rows_t x ldt] of the transpose of src [rows x r] (ld lds)
  void split_t(const float* src, int64_t rows, int64_t r, int64_t lds, bool ones, void* hi,
               void* lo, int64_t rows_t, int64_t ldt) {
    add(PrepTask{PrepTask::kSplitT, ones ? 1 : 0, src, hi, lo, rows, r, lds, rows_t, ldt, 0.f},
        rows_t * ldt);
  }
  // dst [rows_out x ldd] = bf16(scale * src[rows x cols]) zero padded
  void pad(const float* src, int64_t rows, int64_t cols, int64_t lds, float scale, void* dst,
           int64_t rows_out, int64_t ldd) {
    add(PrepTask{PrepTask::kPadBf16, 0, src, dst, nullptr, rows, cols, lds, rows_out, ldd, scale},
        rows_out * ldd);
  }
};
// First block of each task in a k_prep launch (host-computed partition).
struct PrepBlocks {
  int first[kMaxPrep + 1];
};
cudaError_t launch_prep(const PrepBatch& b, cudaStream_t st);

// Block randomized Hadamard transform of bf16 activations (rht.cu).
cudaError_t launch_rht(const void* in, int64_t rows, int64_t cols, int64_t ld_in,
                       const float* signs, int inverse, int block, void* out, int64_t ld_out,
                       bool f32, cudaStream_t st);

// Skinny rank-r products on tensor cores (thin_mma.cu); r <= 64 per call. Factors are passed
// transposed and split into bf16 hi/lo planes [thin_rows(r) x ld] (PrepBatch::split_t).
int thin_rows(int64_t r, bool ones);
// Where a skinny product's finished tiles go (thin_mma.cu thin_flush). Outputs are
// stored, not accumulated: no zero-fill needed.
struct ThinOut {
  float* out = nullptr;            // [n_out x ldo] fp32: out[row, j] = scale · v (j < rc)
  int64_t ldo = 0;
  float scale = 1.0f;
  int rc = 0;                      // set by the launcher (= r of this call)
  float* colsum = nullptr;         // colmma: colsum[row] = v of the ones column (j == rc)
  __nv_bfloat16* pad = nullptr;    // rowmma: bf16(pad_scale · v) [n_out x ldp], cols [rc, pad_cols) = 0
  int64_t ldp = 0;
  int pad_cols = 0;
  float pad_scale = 1.0f;
  __nv_bfloat16* thi = nullptr;    // rowmma: transposed hi/lo planes [t_rows x ldt] (lo after hi)
  int64_t ldt = 0;
  int t_rows = 0;
  float* ws = nullptr;             // per-CTA partial slots (thin_ws_size floats)
  int64_t ws_floats = 0;           // capacity of ws (checked against the launch's grid)
  int* cnt = nullptr;              // per-tile contributor counters, zero before the first
                                   // launch; the finisher resets its tile's counter to 0
  unsigned long long* trace = nullptr;  // dev-only (-DMLRA_DEV_TRACE, MLRA_TRACE3): 8 globaltimer
                                        // stamps per CTA
};
// Workspace of one launch: ws floats and counters (ints).
void thin_ws_size(bool row, int64_t m, int64_t d, int64_t r, bool ones, int64_t* ws_floats,
                  int64_t* n_cnt);
// out[m x r] = act[m x kd] · W      (W given as Wt hi/lo [rows x ldw])
cudaError_t launch_rowmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const __nv_bfloat16* wt_hi, const __nv_bfloat16* wt_lo, int64_t ldw,
                          int64_t r, const ThinOut& o, cudaStream_t st);
// out[m x r] = act[m x kd] · F for an fp32 factor F [kd x r] (ld ldf), r <= 64, on
// the cluster kernel (k_rowmma_cl: factor split in-kernel, no counters); `post`
// (the pass's small jobs) runs inside the launch after its PDL wait.
bool thin_fused_ok(int64_t r, int64_t m);
cudaError_t launch_rowmma_fused(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                                const float* F, int64_t ldf, int64_t r, const ThinOut& o,
                                const PrepBatch& post, cudaStream_t st);
// out[nd x r] = scale · actᵀ · V    (V given as Vt hi/lo [rows x ldv]); colsum[n] = Σ_t act
cudaError_t launch_colmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const __nv_bfloat16* vt_hi, const __nv_bfloat16* vt_lo, int64_t ldv,
                          int64_t r, const ThinOut& o, cudaStream_t st);

}  // namespace mlra

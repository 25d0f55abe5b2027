/*
 * mlra.h — C ABI of the B200-native ModuLoRA linear layer (libmlra.so).
 *
 * Drop-in boundary for the reference's hot path. Every entry
 * point names the reference interface it replaces. Plain pointers and sizes
 * only: device pointers for activations/parameters, host pointers for the
 * one-time weight upload, a cudaStream_t passed as void*. All calls are
 * stream-ordered and asynchronous unless stated.
 *
 * Layouts (reference layout kept; lora.hpp:24-31):
 *   packed codes  — the reference's LSB-first u32 bitstream over the whole
 *                   row-major rows x cols matrix (bitpack.hpp:17-23)
 *   scales/zeros  — f32, rows x (cols/group), row-major by group (quantize.hpp:36-37)
 *   A             — f32 [d_out x r] row-major (the "up" factor, zero-init)
 *   B             — f32 [d_in  x r] row-major (the "down" factor, Gaussian-init)
 *   activations   — bf16 row-major, x: [m x d_in], y/dy: [m x d_out]
 *   gradients     — dA f32 [d_out x r], dB f32 [d_in x r], dbias f32 [d_out]
 *
 * Errors: exceptions cannot cross a C ABI, so each reference exception type
 * maps 1:1 onto a status code (errors.hpp:15-63) and the message is kept in a
 * thread-local string (mlra_last_error). There is no CPU fallback: on a
 * device that is not sm_100 every compute entry point returns
 * MLRA_ERR_UNSUPPORTED.
 */
#ifndef MLRA_H_
#define MLRA_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MLRA_API __attribute__((visibility("default")))
#else
#define MLRA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum mlra_status {
  MLRA_OK = 0,
  MLRA_ERR_DIMENSION = 2,   /* modulora::DimensionError  errors.hpp:20 */
  MLRA_ERR_CONFIG = 3,      /* modulora::ConfigError     errors.hpp:26 */
  MLRA_ERR_RANGE = 4,       /* modulora::RangeError      errors.hpp:32 */
  MLRA_ERR_CONTRACT = 5,    /* modulora::ContractError   errors.hpp:38 */
  MLRA_ERR_NUMERIC = 6,     /* modulora::NumericError    errors.hpp:44 */
  MLRA_ERR_FORMAT = 7,      /* modulora::FormatError{BadField} errors.hpp:55-63 */
  MLRA_ERR_CUDA = 8,        /* CUDA runtime failure (no reference equivalent) */
  MLRA_ERR_UNSUPPORTED = 9  /* not an sm_100 device / extension unavailable */
} mlra_status;

/* MaterializationStrategy (lowprec_linear.hpp:29-30), GPU meaning:
 *   MLRA_WEIGHT — materialize Ŵ (bf16) in HBM, then the tcgen05 GEMM (TMA operands)
 *   MLRA_ROW    — tile-level materialization: codes dequantized into shared memory
 *                 per GEMM tile; Ŵ never exists in HBM (the fused kernel)
 *   MLRA_MATVEC — the quantizer-hook path; the built-in affine plugin's device
 *                 hook is the same fused kernel */
typedef enum mlra_strategy { MLRA_WEIGHT = 0, MLRA_ROW = 1, MLRA_MATVEC = 2 } mlra_strategy;

typedef enum mlra_dtype { MLRA_F32 = 0, MLRA_BF16 = 1 } mlra_dtype;

/* Device-resident frozen QuantizedMatrix (quantize.hpp:29-48). Immutable and
 * shareable across streams once created. */
typedef struct mlra_qweight mlra_qweight;

/* One ModuLoraLayer (lora.hpp:40-51) as seen by the kernels. scaling() = alpha/rank
 * (lora.hpp:30). bias may be NULL (zero bias). */
typedef struct mlra_lora {
  const mlra_qweight* q;
  mlra_strategy strategy;
  int64_t rank;
  double alpha;
  const float* a;    /* device, [d_out x rank] */
  const float* b;    /* device, [d_in x rank]  */
  const float* bias; /* device, [d_out] or NULL */
} mlra_lora;

/* Last error message of this thread ("" if none). */
MLRA_API const char* mlra_last_error(void);
MLRA_API int mlra_abi_version(void);
/* Number of CUDA kernels this library has launched in this process. */
MLRA_API uint64_t mlra_kernel_launches(void);

/* MLRA_OK iff the current CUDA device is sm_100 (B200). */
MLRA_API mlra_status mlra_device_check(void);

/* packed_word_count (bitpack.cpp:64-66). */
MLRA_API uint64_t mlra_packed_word_count(uint64_t count, int bits);

/* Upload + validate a QuantizedMatrix from HOST memory.
 * Replaces QuantizedMatrix::validate (quantize.cpp:82-115) + bitpack
 * validate_metadata (bitpack.cpp:37-60) + the device upload of SURVEY §7.2:
 * verbatim when rows, cols are multiples of 256 (all LLaMA shapes), else a
 * device relayout to word-aligned padded rows. Also precomputes, per group,
 * whether the fp32-FMA dequant is exact (else the kernels use f64). */
MLRA_API mlra_status mlra_qweight_create(int64_t rows, int64_t cols, int bits, int64_t group_size,
                                const uint32_t* words, uint64_t word_count,
                                uint64_t code_count, const float* scales, const float* zeros,
                                uint64_t grid_count, void* stream, mlra_qweight** out);
MLRA_API void mlra_qweight_destroy(mlra_qweight* q);
MLRA_API mlra_status mlra_qweight_info(const mlra_qweight* q, int64_t* rows, int64_t* cols, int* bits,
                              int64_t* group_size, uint64_t* device_bytes,
                              int64_t* uncertified_groups);

/* dequantize_into (quantize.cpp:123-137): out[rows x cols] (leading dim ld) =
 * RN(double(s)·c + double(z)) as f32, or bf16 = RN(that f32). Bit-exact with
 * (float)modulora::dequantize(q). */
MLRA_API mlra_status mlra_materialize(const mlra_qweight* q, void* out, mlra_dtype dtype, int64_t ld,
                             void* stream);
/* dequantize_row_into (quantize.cpp:139-155) for rows [row0, row0+nrows):
 * RangeError when the range runs past q.rows. */
MLRA_API mlra_status mlra_materialize_rows(const mlra_qweight* q, int64_t row0, int64_t nrows, void* out,
                                  mlra_dtype dtype, int64_t ld, void* stream);

/* Bytes a strategy materializes in HBM per pass — what MemoryLedger::on_alloc
 * would be charged (lowprec_linear.cpp:17-37; bf16 = 2 B/entry on the GPU,
 * 0 for the fused strategies, like QuantizerMatvec :101-103). */
MLRA_API uint64_t mlra_ledger_bytes(const mlra_qweight* q, mlra_strategy strategy);

/* lp_forward (lowprec_linear.cpp:150-196): y[m x rows] = x[m x cols] · Ŵᵀ. */
MLRA_API mlra_status mlra_lp_forward(const mlra_qweight* q, mlra_strategy strategy, const void* x,
                            int64_t ldx, int64_t m, void* y, mlra_dtype y_dtype, int64_t ldy,
                            void* stream);
/* lp_backward (lowprec_linear.cpp:198-247): dx[m x cols] = g[m x rows] · Ŵ,
 * re-dequantizing Ŵ (never cached). */
MLRA_API mlra_status mlra_lp_backward(const mlra_qweight* q, mlra_strategy strategy, const void* g,
                             int64_t ldg, int64_t m, void* dx, mlra_dtype dx_dtype,
                             int64_t lddx, void* stream);

/* layer_forward (lora.cpp:52-72): y = x·Ŵᵀ + (alpha/r)·(x·B)·Aᵀ + bias.
 * xb: device f32 [m x rank], receives x·B (saved for the backward pass). */
MLRA_API mlra_status mlra_lora_forward(const mlra_lora* layer, const void* x, int64_t ldx, int64_t m,
                              void* y, mlra_dtype y_dtype, int64_t ldy, float* xb,
                              void* stream);
/* The tape replay of layer_forward's records (autodiff.cpp:101-193) for
 * upstream gradient dy:
 *   dA = s·dyᵀ·xb,  dB = s·xᵀ·(dy·A),  dbias = Σ_t dy (if dbias != NULL),
 *   dx = dy·Ŵ + s·(dy·A)·Bᵀ  (skipped when dx == NULL, as autodiff.cpp:136
 *   skips a frozen input). Gradients are written (not accumulated). */
MLRA_API mlra_status mlra_lora_backward(const mlra_lora* layer, const void* x, int64_t ldx,
                               const float* xb, const void* dy, int64_t lddy, int64_t m,
                               void* dx, mlra_dtype dx_dtype, int64_t lddx, float* da,
                               float* db, float* dbias, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MLRA_H_ */

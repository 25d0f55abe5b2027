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
 *
 * Streams and workspace: a layer pass enqueues its kernels on `stream` (the
 * backward also uses an internal side stream that is joined back into `stream`
 * before the call returns). Temporary device memory comes from a per-(device,
 * stream) arena kept by the library across calls (regrown on demand; the
 * stream-ordered pool under stream capture or for buffers > 64 MB), so calls
 * are capturable into CUDA graphs. The small-token GEMM schedules (split-K /
 * stream-K) need all CTAs of their grid resident at once: do not run two layer
 * passes concurrently on different streams of one device.
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
  MLRA_ERR_UNSUPPORTED = 9, /* not an sm_100 device / extension unavailable */
  MLRA_ERR_IO = 10          /* modulora::IoError         errors.hpp:50 */
} mlra_status;

/* MaterializationStrategy (lowprec_linear.hpp:29-30), GPU meaning:
 *   MLRA_WEIGHT — materialize Ŵ (bf16) in HBM, then the tcgen05 GEMM (TMA operands)
 *   MLRA_ROW    — tile-level materialization: codes dequantized into shared memory
 *                 per GEMM tile; Ŵ never exists in HBM (the fused kernel)
 *   MLRA_MATVEC — the quantizer-hook path; the built-in affine plugin's device
 *                 hook is the same fused kernel */
typedef enum mlra_strategy { MLRA_WEIGHT = 0, MLRA_ROW = 1, MLRA_MATVEC = 2 } mlra_strategy;

typedef enum mlra_dtype { MLRA_F32 = 0, MLRA_BF16 = 1, MLRA_F64 = 2 } mlra_dtype;

/* Device-resident frozen QuantizedMatrix (quantize.hpp:29-48). Immutable and
 * shareable across streams once created. */
typedef struct mlra_qweight mlra_qweight;

/* Device form of the black-box Quantizer plugin (quantize.hpp:91-106).
 *
 * The reference's per-plugin override point is the virtual
 * Quantizer::matvec / matvec_transposed pair (quantize.hpp:98-105), consulted
 * by lp_forward / lp_backward under QuantizerMatvec (lowprec_linear.cpp:
 * 174-182, 226-235) through LpLinearContext::matvec_hook
 * (lowprec_linear.hpp:85-91). A per-token f64 matvec is the wrong shape for a
 * GPU, so the device hook is the plugin's *dequantize* of one tile of Ŵ: the
 * library materializes Ŵ through the hook in bounded slabs (rows for the
 * forward, columns for dX) into a bf16 workspace and runs its TMA-fed tcgen05
 * GEMM over each slab. The hook sees only (q, tile) — it may decode any packed
 * format it owns (a non-affine codebook, a scaled copy of the affine codes…).
 *
 * materialize(): write Ŵ[row0:row0+nrows, col0:col0+ncols] (dtype, leading
 * dimension ld, row-major) to device memory `out`, stream-ordered on `stream`
 * (a cudaStream_t). col0 and ncols are multiples of 8 except at the last
 * column. Return MLRA_OK or an error status (the message via the hook's own
 * mlra_last_error-style channel is the plugin's business). */
typedef struct mlra_hook {
  const char* name; /* Quantizer::name() (quantize.hpp:94) */
  void* state;
  mlra_status (*materialize)(void* state, const mlra_qweight* q, int64_t row0, int64_t nrows,
                             int64_t col0, int64_t ncols, void* out, mlra_dtype dtype,
                             int64_t ld, void* stream);
} mlra_hook;

/* One ModuLoraLayer (lora.hpp:40-51) as seen by the kernels. scaling() = alpha/rank
 * (lora.hpp:30). bias may be NULL (zero bias). hook: the layer's optional
 * Quantizer plugin (ModuLoraLayer::matvec_hook, lora.hpp:47; consulted only
 * under MLRA_MATVEC, like lowprec_linear.cpp:174-182), NULL for none. */
typedef struct mlra_lora {
  const mlra_qweight* q;
  mlra_strategy strategy;
  int64_t rank;
  double alpha;
  const float* a;    /* device, [d_out x rank] */
  const float* b;    /* device, [d_in x rank]  */
  const float* bias; /* device, [d_out] or NULL */
  const mlra_hook* hook; /* optional matvec hook (ABI >= 2) */
} mlra_lora;

/* Last error message of this thread ("" if none). */
MLRA_API const char* mlra_last_error(void);
MLRA_API int mlra_abi_version(void);
/* FormatError::Kind of this thread's last MLRA_ERR_FORMAT (errors.hpp:55-63:
 * 0 BadMagic, 1 BadVersion, 2 Truncated, 3 BadField) and its byte offset;
 * -1 when the last error carried no kind. */
MLRA_API int mlra_last_format_error(uint64_t* offset);
/* Number of CUDA kernels this library has launched in this process. */
MLRA_API uint64_t mlra_kernel_launches(void);

/* MLRA_OK iff the current CUDA device is sm_100 (B200). */
MLRA_API mlra_status mlra_device_check(void);

/* The reference's seeded generator (rng.hpp:15-57) on the host: mix_seed, and
 * DenseMatrix::gaussian's row-major fill out[i] = mean + stddev·g_i
 * (matrix.cpp:62-67) from Rng(seed) — bit-identical to the reference, so
 * init_adapter (lora.cpp:14-32: B = gaussian(d_in x r, Rng(seed), 0, 0.02))
 * and seeded inputs match it exactly. */
MLRA_API uint64_t mlra_mix_seed(uint64_t seed, uint64_t salt);
MLRA_API void mlra_gaussian_fill(uint64_t seed, double* out, uint64_t n, double mean,
                                 double stddev);

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

/* A quantized matrix whose packed format only its plugin understands (a
 * non-affine codebook): rows x cols with nominal `bits` per
 * entry, every dequantization (all strategies, mlra_materialize*) goes through
 * hook->materialize. The hook struct is copied; hook->state must outlive q. */
MLRA_API mlra_status mlra_qweight_create_opaque(int64_t rows, int64_t cols, int bits,
                                                const mlra_hook* hook, mlra_qweight** out);

/* Built-in non-affine plugin "cb2": a QuIP#-style 2-bit vector codebook.
 * Every 8 consecutive entries of a row share one u16 code: bits 0-7 index a
 * 256 x 8 f32 codebook of magnitudes, bit 8+j negates entry j. Per-(row,
 * group) f32 scale s (group along cols, a multiple of 8 dividing cols):
 *   Ŵ[i, 8u+j] = RN_f32(s[i, (8u+j)/g] · (±cb[idx][j]))
 * codes: host u16 [rows x cols/8]; codebook: host f32 [256 x 8]; scales: host
 * f32 [rows x cols/group] (> 0). Uploads everything and returns an opaque
 * qweight whose hook is the library's cb2 materialize kernel. */
MLRA_API mlra_status mlra_cb2_create(int64_t rows, int64_t cols, int64_t group_size,
                                     const uint16_t* codes, const float* codebook,
                                     const float* scales, void* stream, mlra_qweight** out);

/* Built-in plugin "e8p": QuIP#'s E8P lattice codebook (2 bits/weight) in the
 * cb2 stream format — one u16 per 8 consecutive row entries: bits 0-7 index
 * the 256-pattern abs table (mlra_e8p_abs_table), bits 8-14 negate entries
 * 0-6, entry 7's sign makes the negation count congruent to the pattern's
 * coordinate sum (mod 2: the point lies in E8's half-integer coset), bit 15
 * shifts every entry by +1/4 (set) or -1/4 — and one f32 scale per (row,
 * group). Ŵ = RN_f32(s · value) with value = sign·|a| + shift (exact in bf16).
 * Decoded inside the fused GEMM (Q ring) for whole 256-multiples, through its
 * hook otherwise. Reference: none (the interface must host
 * such plugins; the decode law is pinned by oracle/mlra_oracle.c). */
MLRA_API mlra_status mlra_e8p_create(int64_t rows, int64_t cols, int64_t group_size,
                                     const uint16_t* codes, const float* scales, void* stream,
                                     mlra_qweight** out);
/* The E8P abs-pattern table (256 x 8 f32, row-major) and its 256 odd bits
 * (8 words); returns 256. Either pointer may be NULL. */
MLRA_API int mlra_e8p_abs_table(float* abs_out, uint32_t* odd_out);

/* Block randomized Hadamard transform of bf16 activations [rows x cols] (QuIP#'s
 * incoherence processing): per block of `block` columns
 * (a power of two in [64, 1024] dividing cols), inverse = 0: out = H·diag(s)·in
 * / sqrt(block); inverse = 1: out = diag(s)·H·in / sqrt(block) (H symmetric, so
 * the two are each other's inverse). signs: device f32 [cols] of +-1. out is
 * bf16 or f32 with leading dimension ld_out. A layer quantized in the rotated
 * basis W~ = U W V^T runs y = U^T(W~(V x)), dx = V^T(W~^T(U dy)). */
MLRA_API mlra_status mlra_rht(const void* in, int64_t rows, int64_t cols, int64_t ld_in,
                              const float* signs, int inverse, int block, void* out,
                              int64_t ld_out, mlra_dtype out_dtype, void* stream);

/* Built-in "lut" plugin (non-uniform levels, e.g. QLoRA's NF4; a plugin behind
 * the reference's Quantizer interface, quantize.hpp:91-106, like cb2): codes
 * in the reference's b-bit bitstream (bitpack.cpp:25-35; words / word_count as
 * mlra_qweight_create), a table of 2^bits finite f32 levels and one f32 scale
 * (> 0) per (row, group):  Ŵ[i, j] = RN_f32(s[i, j/g] · levels[c[i, j]]).
 * bits in {2, 3, 4}; group_size % 8 == 0. The result is an ordinary
 * (non-opaque) qweight: materialize() runs the lut kernel, and the fused GEMM
 * decodes the table in its dequant warps when the group tiles the Q ring
 * (32, 64 or a multiple of 128), else Ŵ goes through HBM. */
MLRA_API mlra_status mlra_lut_create(int64_t rows, int64_t cols, int bits, int64_t group_size,
                                     const uint32_t* words, uint64_t word_count,
                                     const float* levels, const float* scales, void* stream,
                                     mlra_qweight** out);

/* RtnQuantizer::quantize (quantize.hpp:108-113; quantize.cpp:24-44, 163-184)
 * on the device: w is a DEVICE matrix [rows x cols] of dtype MLRA_F64 or
 * MLRA_F32 (widened exactly); group_size 0 selects per-row grids
 * (quantize.cpp:78-80). Writes, on `stream`, the reference's QuantizedMatrix
 * layout to device buffers: words [mlra_packed_word_count(rows*cols, bits)]
 * (LSB-first bitstream over the whole row-major matrix), scales / zeros
 * [rows x cols/group]. Bit-identical to quantize_rtn((double)w).
 * Errors: DimensionError (empty), ConfigError (bits / group). */
MLRA_API mlra_status mlra_quantize_rtn(const void* w, mlra_dtype dtype, int64_t rows, int64_t cols,
                                       int bits, int64_t group_size, uint32_t* words,
                                       float* scales, float* zeros, void* stream);

/* build_optq_workspace (quantize.hpp:65-71; quantize.cpp:186-211) on the
 * device: calib DEVICE f64 [m x dim] -> hessian = XᵀX + damping·mean(diag)·I
 * and upper = the upper Cholesky factor of its inverse (linalg.cpp:68-71),
 * both DEVICE f64 [dim x dim], bit-identical to the reference. Synchronous.
 * Errors: DimensionError (empty calibration), ConfigError (damping < 0 or
 * NaN), NumericError ("Hessian not invertible after damping"). */
MLRA_API mlra_status mlra_optq_workspace(const double* calib, int64_t m, int64_t dim,
                                         double damping, double* hessian, double* upper,
                                         void* stream);

/* OptqQuantizer::quantize (quantize.hpp:73-75, 115-125; quantize.cpp:213-255)
 * on the device: w DEVICE f64 [rows x cols], calib DEVICE f64 [m x cols];
 * writes the reference's QuantizedMatrix layout to DEVICE words / scales /
 * zeros exactly as mlra_quantize_rtn (same grids: computed from the original
 * weights), with the calibration-aware column sweep's codes. Bit-identical to
 * quantize_optq. Synchronous. Errors as quantize_rtn, then as
 * mlra_optq_workspace. */
MLRA_API mlra_status mlra_quantize_optq(const double* w, const double* calib, int64_t rows,
                                        int64_t cols, int64_t m, int bits, int64_t group_size,
                                        double damping, uint32_t* words, float* scales,
                                        float* zeros, void* stream);

/* The hook an opaque qweight carries (NULL for the affine built-in format). */
MLRA_API const mlra_hook* mlra_qweight_hook(const mlra_qweight* q);

/* dequantize_into (quantize.cpp:123-137): out[rows x cols] (leading dim ld) =
 * RN(double(s)·c + double(z)) as f32, or bf16 = RN(that f32). Bit-exact with
 * (float)modulora::dequantize(q). */
MLRA_API mlra_status mlra_materialize(const mlra_qweight* q, void* out, mlra_dtype dtype, int64_t ld,
                             void* stream);
/* dequantize_row_into (quantize.cpp:139-155) for rows [row0, row0+nrows):
 * RangeError when the range runs past q.rows. */
MLRA_API mlra_status mlra_materialize_rows(const mlra_qweight* q, int64_t row0, int64_t nrows, void* out,
                                  mlra_dtype dtype, int64_t ld, void* stream);

/* One tile Ŵ[row0:row0+nrows, col0:col0+ncols] (col0 a multiple of 8) —
 * the device hook's unit of work. Affine qweights decode it with the K1
 * kernel (bit-exact like mlra_materialize); opaque ones call their hook. */
MLRA_API mlra_status mlra_materialize_tile(const mlra_qweight* q, int64_t row0, int64_t nrows,
                                           int64_t col0, int64_t ncols, void* out,
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

/* lp_forward / lp_backward with LpLinearContext::matvec_hook
 * (lowprec_linear.hpp:85-91): under MLRA_MATVEC a non-NULL hook replaces the
 * built-in dequantization (slab materialization through the hook + GEMM);
 * the other strategies ignore it, as the reference's do. */
MLRA_API mlra_status mlra_lp_forward_ex(const mlra_qweight* q, mlra_strategy strategy,
                                        const mlra_hook* hook, const void* x, int64_t ldx,
                                        int64_t m, void* y, mlra_dtype y_dtype, int64_t ldy,
                                        void* stream);
MLRA_API mlra_status mlra_lp_backward_ex(const mlra_qweight* q, mlra_strategy strategy,
                                         const mlra_hook* hook, const void* g, int64_t ldg,
                                         int64_t m, void* dx, mlra_dtype dx_dtype, int64_t lddx,
                                         void* stream);

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

/* AdamW with decoupled weight decay (train.hpp:51-70, AdamW::AdamW). */
typedef struct mlra_adamw {
  double beta1, beta2, eps, weight_decay;
} mlra_adamw;

/* AdamW::step (train.cpp:81-134) over n_params parameters stored back to back
 * in one flat device bucket: parameter i is elements [offsets[i], offsets[i+1])
 * (offsets: HOST array of n_params + 1, offsets[0] = 0, n_params <= 1024). params, m, v: device
 * f64 (masters and moments; m, v zero before the first step — "allocated on
 * first use"); grad: device, dtype MLRA_F32 (the layer kernels' gradients) or
 * MLRA_F64; params_f32: optional device f32 working copy written with the new
 * values (the factors the GEMMs read). step_index is the reference's
 * zero-based step (t = step_index + 1). Bit-identical to the reference f64
 * arithmetic given the same gradients.
 * Non-finite gradients (train.cpp:113-117): parameters before the first one
 * holding a non-finite gradient are updated, it and the rest are not. With
 * first_bad == NULL the call synchronizes on `stream` and returns
 * MLRA_ERR_NUMERIC naming that parameter; otherwise it stays asynchronous and
 * writes the index (a value >= n_params when all are finite) to the device int
 * *first_bad. Capturable in a CUDA graph in that form (no host copies). */
MLRA_API mlra_status mlra_adamw_step(const mlra_adamw* opt, int64_t step_index, double lr,
                                     int64_t n_params, const int64_t* offsets, double* params,
                                     double* m, double* v, const void* grad,
                                     mlra_dtype grad_dtype, float* params_f32, int* first_bad,
                                     void* stream);

/* ------------------------------------------------------------------------
 * Data-parallel exchange: tokens sharded across ranks, frozen
 * weights replicated; the only per-step exchange is a sum all-reduce of the
 * flat fp32 LoRA-gradient bucket ({dA, dB[, dbias]} per layer, the parameter
 * order of ToyModel::trainable_params, model.cpp:170-184), NCCL over NVLink /
 * NVSwitch. NCCL is loaded at run time (dlopen libnccl.so.2); without it these
 * return MLRA_ERR_UNSUPPORTED. The reference itself has no distribution
 * (SPEC.md:453). */
typedef struct mlra_dp mlra_dp;
/* Rank 0 creates the 128-byte id and shares it out of band (file, socket). */
MLRA_API mlra_status mlra_dp_unique_id(void* id_out);
/* One communicator per process (one process per GPU; the current device). */
MLRA_API mlra_status mlra_dp_init(int rank, int world, const void* id, mlra_dp** out);
/* In-place sum all-reduce of `count` fp32 gradients on `stream`. */
MLRA_API mlra_status mlra_allreduce_lora_grads(mlra_dp* dp, float* bucket, uint64_t count,
                                               void* stream);
MLRA_API void mlra_dp_destroy(mlra_dp* dp);

/* ------------------------------------------------------------------------
 * On-disk checkpoint -> device. The reference's binary .mlra
 * format (checkpoint.hpp:4-24, little-endian): parsed and validated with the
 * reference's rules and error taxonomy (checkpoint.cpp:141-306: FormatError
 * BadMagic / BadVersion / Truncated / BadField with the byte offset, IoError),
 * each layer's packed words then uploaded verbatim to HBM (they are already
 * the device layout at LLaMA shapes). The config JSON is carried as opaque
 * bytes (model assembly from it is outside the hot path). Saving re-encodes
 * byte-identically (checkpoint.cpp:93-130), with adapters optionally replaced
 * (the finetune flow rewrites only the adapter section). */
typedef struct mlra_checkpoint mlra_checkpoint;

/* One layer record + its adapter (pointers into the checkpoint, valid until it
 * is freed or the adapter is replaced). */
typedef struct mlra_ckpt_layer {
  const char* name;
  int64_t rows, cols;
  int bits;
  int64_t group_size;
  const uint32_t* words;
  uint64_t word_count;
  const float* scales; /* rows * (cols/group) */
  const float* zeros;
  const float* bias;   /* rows */
  int64_t rank;        /* 0 when the layer has no adapter record */
  float alpha;
  const double* a;     /* rows x rank */
  const double* b;     /* cols x rank */
  uint64_t record_offset, record_size;   /* layer record bytes (inspect_layout) */
  uint64_t adapter_offset, adapter_size; /* adapter record bytes */
} mlra_ckpt_layer;

/* load_model's parse (checkpoint.cpp:141-306) of `path`. */
MLRA_API mlra_status mlra_checkpoint_load(const char* path, mlra_checkpoint** out);
MLRA_API void mlra_checkpoint_free(mlra_checkpoint* c);
MLRA_API int64_t mlra_checkpoint_layer_count(const mlra_checkpoint* c);
MLRA_API mlra_status mlra_checkpoint_layer(const mlra_checkpoint* c, int64_t i,
                                           mlra_ckpt_layer* out);
/* The ModelConfig JSON bytes (NUL-terminated copy) and format version. */
MLRA_API const char* mlra_checkpoint_config_json(const mlra_checkpoint* c, int* version);
/* ToyModel::frozen_state_hash (model.cpp:203-211; hash_quantized
 * quantize.cpp:383-391) over the layer records, and fnv1a64_file
 * (hash.cpp:11-20) of the bytes save() would write. */
MLRA_API uint64_t mlra_checkpoint_frozen_hash(const mlra_checkpoint* c);
MLRA_API uint64_t mlra_checkpoint_file_hash(const mlra_checkpoint* c);
/* Device upload of layer i's QuantizedMatrix (mlra_qweight_create, verbatim). */
MLRA_API mlra_status mlra_checkpoint_upload(const mlra_checkpoint* c, int64_t i, void* stream,
                                            mlra_qweight** out);
/* Replace layer i's adapter factors (host f64, rows x rank and cols x rank). */
MLRA_API mlra_status mlra_checkpoint_set_adapter(mlra_checkpoint* c, int64_t i, const double* a,
                                                 const double* b);
/* The adapter section in file order (inspect_layout's adapter list,
 * checkpoint.cpp:294-296): the record's layer name, offset and size. */
MLRA_API int64_t mlra_checkpoint_adapter_count(const mlra_checkpoint* c);
MLRA_API mlra_status mlra_checkpoint_adapter(const mlra_checkpoint* c, int64_t i,
                                             const char** layer_name, uint64_t* offset,
                                             uint64_t* size);
/* load_model's assemble_model checks (model.cpp:472-531) -> MLRA_ERR_CONFIG: one
 * adapter per layer, unique layer names, the parity transformer's layer names
 * (parity_transformer != 0) or chained dims, adapter i naming layer i, rank >= 1
 * and alpha > 0, bias length d_out. */
MLRA_API mlra_status mlra_checkpoint_assemble_check(const mlra_checkpoint* c,
                                                    int parity_transformer);
/* save_model's encoding (checkpoint.cpp:93-130, 307-314) to `path`. */
MLRA_API mlra_status mlra_checkpoint_save(const mlra_checkpoint* c, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* MLRA_H_ */

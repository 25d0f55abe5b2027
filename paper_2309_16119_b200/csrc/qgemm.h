// qgemm.h — host-side interface of the fused dequant tcgen05 GEMM (qgemm.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mlra {

struct GemmMaps {
  CUtensorMap act;       // activations [tokens x K_red] bf16, box 64 x 256, SW128
  CUtensorMap act_lora;  // LoRA activations [tokens x 64*nlb] bf16, box 64 x 256
  CUtensorMap w;         // materialized W bf16 (strategy weight): box 64x128 (K-major) or 64x64 (MN)
  CUtensorMap w_lora;    // adapter factor padded [m_total x 64*nlb] bf16, box 64 x 128
  CUtensorMap codes;     // packed codes as u8 [rows_pad x row_bytes], box 16*bits x 128
  CUtensorMap grid;      // signed grid as f32 [rows_pad x 2*ng_pad], box 2*max(2,128/g) x 128
};

struct GemmArgs {
  int64_t m_total;   // weight-side extent, multiple of 128
  int64_t m_valid;   // weight-side extent actually stored
  int n_kb_main;     // 64-wide reduction blocks over the quantized operand (even)
  int n_kb_lora;     // extra 64-wide LoRA blocks (ceil(r/64)), 0 = none
  int lora_k16_last; // useful 16-wide MMA steps in the last LoRA block
  int64_t tokens;    // m
  int bn;            // 1-CTA kernel: tokens per tile (128 or 256)
  void* out;         // [tokens x ldo], f32 or bf16
  int64_t ldo;
  const float* bias; // [m_valid] or nullptr
  int out_pairs;     // bf16 out with even ldo and 4-byte aligned base: paired-row stores
  const void* cb2_codebook;  // non-null: fused cb2 plugin decode (bf16 codebook, uint4[256])
  int e8p;                   // with cb2_codebook: the e8p plugin's tables and decode
  const float* lut;          // non-null: fused lut plugin decode (16 f32 levels)
  // Q ring (fused path with TMA-fed codes); q_stages == 0 selects the LDG path
  int q_stages;
  int q_stage_bytes;
  int q_codes_bytes;
  int q_grid_bytes;
  int q_group_shift; // log2(group) when group < 128, else -1
  int q_group_div128; // group / 128 when group >= 128
  uint32_t q_group_magic; // ceil(2^32 / (group/128)) when group/128 > 1, else 0
  unsigned long long* trace;  // dev-only: per-CTA MMA-thread wait cycles (MLRA_TRACE), else null
  unsigned long long* trace2; // dev-only: per-CTA globaltimer timeline, 8 slots (MLRA_TRACE2)
  // Stream-K / split-K (pair kernel only): 0 = whole tiles strided over the
  // grid; else the tile x k-block space is cut into sk_pairs contiguous ranges
  // (split > 0: S equal cuts per tile). Pair q's range start is a closed form
  // of (q, sk_pairs, split, tiles, k-blocks) evaluated by the kernel once
  // (sk_cut in qgemm2_kernel.cuh; the host planner uses the same formula), so
  // the launch carries no per-pair tables (kernel parameters stay small).
  int sk_pairs;
  int split;             // > 0: split-K mode, S pairs per tile (pair q = tile*S + s)
  int tok256;            // split-K with 256-token pair tiles (one accumulator)
  int no_pdl;            // host only: launch without programmatic dependent launch
  int sk_owner4;         // dev A/B (MLRA_SK_OWNER4=1): stream-K owner fix-up by the 4
                         // epilogue warps instead of all 16 (set by qgemm2_launch)
  float* sk_ws;          // [sk_pairs x 2 CTAs x 512 tokens x 128 rows] fp32 partials
  unsigned* sk_flags;    // [sk_pairs x 2], zeroed before the launch
};

// true when the fused path can stream codes/grids through the TMA Q ring
bool qgemm_q_tma_ok(const QWeightDev& q);
int qgemm_max_q_stages(int q_stage_bytes, int extra_smem = 0);

// mn = false: forward (Ŵ K-major on the weight side); true: dX (Ŵᵀ, MN-major).
cudaError_t qgemm_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                         bool w_tma, bool mn, bool out_f32, cudaStream_t stream);
// CTA-pair variant (qgemm2.cu): 256 weight rows x 512 tokens per pair tile.
// Same maps, except the activation boxes are 64 x 128 (each CTA stages half).
cudaError_t qgemm2_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                          bool w_tma, bool mn, bool out_f32, cudaStream_t stream);
// Plans the pair kernel's schedule: sets p.sk_pairs (0 = whole tiles) and the
// per-pair cut tables. The caller provides sk_ws / sk_flags when sk_pairs > 0.
void qgemm2_plan(GemmArgs& p);
// Kernel choice by cost model (qgemm2.cu): 2 = the pair kernel with its planned
// schedule, 1 = the 1-CTA kernel with 256-token tiles, 3 = 1-CTA with 128.
int qgemm_choose(const GemmArgs& p);
constexpr int kMaxSkPairs = 128;
constexpr int kCb2SmemBytes = 256 * 16;  // the cb2 codebook staged in shared memory
constexpr int kE8pSmemBytes = 2 * 256 * 16 + 128;  // e8p (|a| +- 1/4) tables + odd bits (padded)
constexpr int kLutSmemBytes = 64;         // the lut plugin's 16 levels in shared memory
constexpr int64_t kSkSlotFloats = 2LL * 512 * 128;  // per pair

}  // namespace mlra

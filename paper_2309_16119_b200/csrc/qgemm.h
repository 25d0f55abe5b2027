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
};

struct GemmArgs {
  int64_t m_total;   // weight-side extent, multiple of 128 (grid.x = m_total/128)
  int64_t m_valid;   // weight-side extent actually stored
  int n_kb_main;     // 64-wide reduction blocks over the quantized operand
  int n_kb_lora;     // extra 64-wide LoRA blocks (ceil(r/64)), 0 = none
  int lora_k16_last; // useful 16-wide MMA steps in the last LoRA block
  int64_t tokens;    // m
  void* out;         // [tokens x ldo], f32 or bf16
  int64_t ldo;
  const float* bias; // [m_valid] or nullptr
};

int qgemm_tile_m();
int qgemm_tile_n();
int qgemm_tile_k();

// mn = false: forward (Ŵ K-major on the weight side); true: dX (Ŵᵀ, MN-major).
cudaError_t qgemm_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                         bool w_tma, bool mn, bool out_f32, cudaStream_t stream);

}  // namespace mlra

// qgemm.cu — K2/K3: the fused dequant-GEMM on tcgen05 tensor cores.
//
// One kernel serves both products of the ModuLoRA linear:
//   forward  (K2): Y[t, n]  = Σ_k X[t,k]·Ŵ[n,k]  + Σ_j (s·XB)[t,j]·A[n,j] + bias[n]
//                  replaces lp_forward (lowprec_linear.cpp:150-196) plus the adapter
//                  records of layer_forward (lora.cpp:68-71);
//   backward (K3): dX[t, k] = Σ_n dY[t,n]·Ŵ[n,k] + Σ_j (s·dYA)[t,j]·B[k,j]
//                  replaces lp_backward (lowprec_linear.cpp:198-247) plus the
//                  matmul backward rule for x (autodiff.cpp:150-152).
// The LoRA term rides as extra K blocks ("[X, s·XB]·[Ŵ, A]ᵀ").
//
// Tile = 128 weight-side rows (MMA M; the dequantized operand) x 256 tokens
// (MMA N; activations via TMA) x 64 K per pipeline stage. The weight side is
// produced per stage either by 8 dequant warps straight from the packed codes
// (strategy row/matvec: the full-precision W never exists in HBM) or by TMA
// from a materialized bf16 W (strategy weight). Accumulator: 128 lanes x 256
// f32 columns of TMEM. Epilogue: TMEM -> registers -> (+bias) -> global, with
// lane = weight-side index so stores are coalesced along the output row.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer + TMEM owner,
// w2-3 idle, w4-11 dequant producers, w4-7 then run the epilogue.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "qgemm.h"

namespace mlra {

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int W_TILE = BM * BK * 2;  // 16 KB
constexpr int T_TILE = BN * BK * 2;  // 32 KB
constexpr int DQ_WARP0 = 4;
constexpr int NUM_DQ_WARPS = 8;
constexpr int NUM_DQ_THREADS = NUM_DQ_WARPS * 32;
constexpr int NUM_THREADS = (DQ_WARP0 + NUM_DQ_WARPS) * 32;
constexpr int UNITS_PER_THREAD = (BM * BK / 8) / NUM_DQ_THREADS;  // 4
constexpr uint32_t TMEM_COLS = 256;
constexpr size_t SMEM_BYTES = 1024 + STAGES * (W_TILE + T_TILE) + 256;

struct UnitRegs {
  uint64_t v[UNITS_PER_THREAD];
  float2 g[UNITS_PER_THREAD];
};

// Unit u (0..1023) of a stage -> (weight row, unit index along that row) and
// the byte offset of its 16-byte chunk inside the SW128 stage tile.
//  K-major (forward):  tile = 128 rows x 64 k; unit = (r = u/8, k8 = u%8);
//     canonical K-major SW128: row r at r*128, chunk k8 at (k8 ^ r%8)*16.
//  MN-major (dX):      tile = 64 reduction rows (n) x 128 output cols (k);
//     unit = (n = u/16, k8 = u%16); chunk c = k8/8 of 64 columns at c*8192,
//     row n at n*128, 16-byte column group (k8%8 ^ n%8).
template <bool MN>
__device__ __forceinline__ void unit_coords(int u, int m_tile, int kb, int64_t& wrow,
                                            int64_t& wunit, uint32_t& soff) {
  if constexpr (!MN) {
    const int r = u >> 3, k8 = u & 7;
    wrow = static_cast<int64_t>(m_tile) * BM + r;
    wunit = static_cast<int64_t>(kb) * (BK / 8) + k8;
    soff = r * 128 + ((k8 ^ (r & 7)) << 4);
  } else {
    const int n = u >> 4, k8 = u & 15;
    wrow = static_cast<int64_t>(kb) * BK + n;
    wunit = static_cast<int64_t>(m_tile) * (BM / 8) + k8;
    soff = (k8 >> 3) * 8192 + n * 128 + (((k8 & 7) ^ (n & 7)) << 4);
  }
}

template <int BITS, bool MN>
__device__ __forceinline__ void dq_load(const QWeightDev& q, int m_tile, int kb, int tid,
                                        bool fast_group, UnitRegs& ur) {
#pragma unroll
  for (int i = 0; i < UNITS_PER_THREAD; ++i) {
    int64_t wrow, wunit;
    uint32_t soff;
    unit_coords<MN>(i * NUM_DQ_THREADS + tid, m_tile, kb, wrow, wunit, soff);
    ur.v[i] = load_unit<BITS>(q.words + wrow * q.row_words, wunit);
    if (fast_group) ur.g[i] = __ldg(q.grid + wrow * q.ng_pad + (wunit * 8) / q.group);
  }
}

template <int BITS, bool MN>
__device__ __forceinline__ void dq_store(const QWeightDev& q, int m_tile, int kb, int tid,
                                         bool fast_group, const UnitRegs& ur, uint8_t* stile) {
#pragma unroll
  for (int i = 0; i < UNITS_PER_THREAD; ++i) {
    int64_t wrow, wunit;
    uint32_t soff;
    unit_coords<MN>(i * NUM_DQ_THREADS + tid, m_tile, kb, wrow, wunit, soff);
    uint4 o;
    if (fast_group)
      o = deq8_bf16<BITS>(ur.v[i], ur.g[i]);
    else
      o = deq8_bf16_general<BITS>(ur.v[i], q.grid + wrow * q.ng_pad, wunit * 8, q.group);
    *reinterpret_cast<uint4*>(stile + soff) = o;
  }
}

template <int BITS, bool W_TMA, bool MN, bool OUT_F32>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    qgemm_kernel(const __grid_constant__ CUtensorMap tm_act,
                 const __grid_constant__ CUtensorMap tm_act_lora,
                 const __grid_constant__ CUtensorMap tm_w,
                 const __grid_constant__ CUtensorMap tm_w_lora, const QWeightDev q,
                 const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sW = smem;
  uint8_t* sT = smem + STAGES * W_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sT + STAGES * T_TILE);
  uint64_t* empty = full + STAGES;
  uint64_t* accum_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x;
  const int n_tile = blockIdx.y;
  const int n_kb_main = p.n_kb_main;
  const int n_kb = p.n_kb_main + p.n_kb_lora;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_act);
    if (p.n_kb_lora) {
      tma_prefetch_desc(&tm_act_lora);
      tma_prefetch_desc(&tm_w_lora);
    }
    if (W_TMA) tma_prefetch_desc(&tm_w);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1 + NUM_DQ_WARPS);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accum_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int kb = 0; kb < n_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        const bool lora = kb >= n_kb_main;
        const bool w_tma = lora || W_TMA;
        mbar_arrive_expect_tx(&full[s], T_TILE + (w_tma ? W_TILE : 0));
        uint8_t* st = sT + s * T_TILE;
        uint8_t* sw = sW + s * W_TILE;
        if (!lora) {
          tma_load_2d(st, &tm_act, &full[s], kb * BK, n_tile * BN);
          if (W_TMA) {
            if (!MN) {
              tma_load_2d(sw, &tm_w, &full[s], kb * BK, m_tile * BM);
            } else {
              tma_load_2d(sw, &tm_w, &full[s], m_tile * BM, kb * BK);
              tma_load_2d(sw + 8192, &tm_w, &full[s], m_tile * BM + 64, kb * BK);
            }
          }
        } else {
          const int lk = (kb - n_kb_main) * BK;
          tma_load_2d(st, &tm_act_lora, &full[s], lk, n_tile * BN);
          tma_load_2d(sw, &tm_w_lora, &full[s], lk, m_tile * BM);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_main = idesc_bf16(BM, BN, MN ? 1u : 0u, 0u);
      constexpr uint32_t idesc_kmaj = idesc_bf16(BM, BN, 0u, 0u);
      for (int kb = 0; kb < n_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const bool lora = kb >= n_kb_main;
        const int nk16 = (lora && kb == n_kb - 1) ? p.lora_k16_last : BK / 16;
        const uint32_t sw = smem_u32(sW + s * W_TILE);
        const uint32_t st = smem_u32(sT + s * T_TILE);
        for (int k = 0; k < nk16; ++k) {
          uint64_t adesc;
          uint32_t idesc;
          if (MN && !lora) {
            adesc = sdesc_sw128(sw + k * 2048, 8192, 1024);
            idesc = idesc_main;
          } else {
            adesc = sdesc_sw128(sw + k * 32, 16, 1024);
            idesc = idesc_kmaj;
          }
          const uint64_t bdesc = sdesc_sw128(st + k * 32, 16, 1024);
          tc_mma_f16(tmem_base, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(accum_full);
    }
  } else if (warp >= DQ_WARP0) {
    // ------------------------------------------------------------ dequant producers
    const int tid = threadIdx.x - DQ_WARP0 * 32;
    if constexpr (!W_TMA) {
      const bool fast_group = (q.group % 8) == 0;
      UnitRegs cur, nxt;
      if (n_kb_main > 0) dq_load<BITS, MN>(q, m_tile, 0, tid, fast_group, cur);
      for (int kb = 0; kb < n_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        const bool main = kb < n_kb_main;
        if (kb + 1 < n_kb_main) dq_load<BITS, MN>(q, m_tile, kb + 1, tid, fast_group, nxt);
        mbar_wait(&empty[s], ph ^ 1);
        if (main) {
          dq_store<BITS, MN>(q, m_tile, kb, tid, fast_group, cur, sW + s * W_TILE);
          fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
        cur = nxt;
      }
    } else {
      for (int kb = 0; kb < n_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    }

    if (warp < DQ_WARP0 + 4) {
      // ---------------------------------------------------------- epilogue
      mbar_wait(accum_full, 0);
      tc_fence_after();
      const int qd = warp & 3;  // TMEM lane quadrant this warp may access
      const int64_t wrow = static_cast<int64_t>(m_tile) * BM + qd * 32 + lane;
      const bool row_ok = wrow < p.m_valid;
      const float bias = (p.bias != nullptr && row_ok) ? p.bias[wrow] : 0.0f;
      const int64_t t0 = static_cast<int64_t>(n_tile) * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(qd * 32) << 16) + c * 32, r);
        tc_wait_ld();
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int64_t t = t0 + c * 32 + j;
            if (t < p.tokens) {
              const float v = __uint_as_float(r[j]) + bias;
              if constexpr (OUT_F32) {
                reinterpret_cast<float*>(p.out)[t * p.ldo + wrow] = v;
              } else {
                reinterpret_cast<__nv_bfloat16*>(p.out)[t * p.ldo + wrow] =
                    __float2bfloat16_rn(v);
              }
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, TMEM_COLS);
}

template <int BITS, bool W_TMA, bool MN, bool OUT_F32>
cudaError_t launch_t(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                     cudaStream_t stream) {
  auto kern = qgemm_kernel<BITS, W_TMA, MN, OUT_F32>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  dim3 grid(static_cast<unsigned>(p.m_total / BM),
            static_cast<unsigned>((p.tokens + BN - 1) / BN));
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(maps.act, maps.act_lora, maps.w, maps.w_lora,
                                                  q, p);
  return cudaGetLastError();
}

template <int BITS>
cudaError_t launch_bits(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool w_tma,
                        bool mn, bool out_f32, cudaStream_t stream) {
  if (w_tma) {
    if (mn) return out_f32 ? launch_t<BITS, true, true, true>(maps, q, p, stream)
                           : launch_t<BITS, true, true, false>(maps, q, p, stream);
    return out_f32 ? launch_t<BITS, true, false, true>(maps, q, p, stream)
                   : launch_t<BITS, true, false, false>(maps, q, p, stream);
  }
  if (mn) return out_f32 ? launch_t<BITS, false, true, true>(maps, q, p, stream)
                         : launch_t<BITS, false, true, false>(maps, q, p, stream);
  return out_f32 ? launch_t<BITS, false, false, true>(maps, q, p, stream)
                 : launch_t<BITS, false, false, false>(maps, q, p, stream);
}

}  // namespace

int qgemm_tile_m() { return BM; }
int qgemm_tile_n() { return BN; }
int qgemm_tile_k() { return BK; }

cudaError_t qgemm_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                         bool w_tma, bool mn, bool out_f32, cudaStream_t stream) {
  if (p.tokens <= 0 || p.m_total <= 0) return cudaSuccess;
  if (w_tma) return launch_bits<4>(maps, q, p, true, mn, out_f32, stream);  // bits unused
  switch (q.bits) {
    case 2: return launch_bits<2>(maps, q, p, false, mn, out_f32, stream);
    case 3: return launch_bits<3>(maps, q, p, false, mn, out_f32, stream);
    case 4: return launch_bits<4>(maps, q, p, false, mn, out_f32, stream);
    case 8: return launch_bits<8>(maps, q, p, false, mn, out_f32, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mlra

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
// (MMA N; activations via TMA) x 64 K per pipeline stage. Persistent CTAs
// (one per SM) walk the tile list; two TMEM accumulators (2 x 256 f32
// columns) let the epilogue of tile i overlap the mainloop of tile i+1.
//
// Weight-side operand, per strategy:
//  * row/matvec (fused): packed codes + grids arrive by TMA in their own ring
//    ("Q ring", 128 codes x 128 rows per stage = two K blocks), and 8 dequant
//    warps expand them to bf16 straight into the SW128 operand tile — the
//    full-precision Ŵ never exists in HBM (PAPER.md:116-126 at tile level).
//  * weight: Ŵ (bf16) materialized in HBM by K1, loaded by TMA.
//
// Warp roles (512 threads): w0 operand TMA, w1 MMA issuer + TMEM owner,
// w2 Q-ring TMA, w3 idle, w4-7 epilogue (TMEM -> regs -> +bias -> global),
// w8-15 dequant producers.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "ptx.cuh"
#include "kernels.h"
#include "qgemm.h"
#include "qgemm_dev.cuh"

namespace mlra {

namespace {

using namespace qg;

#ifndef MLRA_NSPLIT
#define MLRA_NSPLIT 2
#endif

// TBN = tokens per tile (MMA N): 256, or 128 for small token counts, where
// 256-token tiles leave most SMs idle (cfg1: 64 vs 128 CTAs at m=512). Each
// dequantized weight tile then feeds half the MMA work, so TBN=128 only pays
// below ~1.5 waves of 256-token tiles (cost model: qgemm_choose, qgemm2.cu).
template <int BITS, bool W_TMA, bool MN, bool OUT_F32, bool QTMA, int TBN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    qgemm_kernel(const __grid_constant__ CUtensorMap tm_act,
                 const __grid_constant__ CUtensorMap tm_act_lora,
                 const __grid_constant__ CUtensorMap tm_w,
                 const __grid_constant__ CUtensorMap tm_w_lora,
                 const __grid_constant__ CUtensorMap tm_codes,
                 const __grid_constant__ CUtensorMap tm_grid, const QWeightDev q,
                 const GemmArgs p) {
  constexpr int BN = TBN;
  constexpr int T_TILE = BN * BK * 2;
  constexpr int STAGES = qgemm1_stages(TBN);
  constexpr uint32_t TMEM_COLS = 2 * BN;  // two accumulators (a power of 2 >= 32)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sW = smem;
  uint8_t* sT = sW + STAGES * W_TILE;
  uint8_t* sQ = sT + STAGES * T_TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sQ + p.q_stages * p.q_stage_bytes);
  uint64_t* empty = full + STAGES;
  uint64_t* qfull = empty + STAGES;
  uint64_t* qempty = qfull + MAX_QS;
  uint64_t* tfull = qempty + MAX_QS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // dev-only (MLRA_TRACE2): per CTA [0] total cycles, [1] MMA wait on full,
  // [2..4] / [5..7] dequant group 0 / 1: wait qfull, wait empty, compute+arrive
#ifdef MLRA_DEV_TRACE  // dev-only instrumentation (MLRA_TRACE2), compiled in with -DMLRA_DEV_TRACE
  unsigned long long* tl = p.trace2 ? p.trace2 + 8 * blockIdx.x : nullptr;
#else
  constexpr unsigned long long* tl = nullptr;
#endif
  const long long t_entry = clock64();
  const int n_kb_main = p.n_kb_main;
  const int n_kb = p.n_kb_main + p.n_kb_lora;
  const TileIter it{static_cast<int>(p.m_total / BM), static_cast<int>((p.tokens + BN - 1) / BN)};
  const int n_tiles = it.m_tiles * it.n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_act);
    if (p.n_kb_lora) {
      tma_prefetch_desc(&tm_act_lora);
      tma_prefetch_desc(&tm_w_lora);
    }
    if (W_TMA) tma_prefetch_desc(&tm_w);
    if (QTMA) {
      tma_prefetch_desc(&tm_codes);
      tma_prefetch_desc(&tm_grid);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1 + NUM_DQ_WARPS / 2);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < MAX_QS; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], NUM_DQ_WARPS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
  pdl_trigger();
  pdl_wait();  // every operand may come from earlier kernels
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ operand TMA
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        it.coords(tile, m_tile, n_tile);
        for (int kb = 0; kb < n_kb; ++kb) {
          mbar_wait_backoff<PROD_NS>(&empty[s], ph ^ 1);
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
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // The token tile is issued as NSPLIT independent MMAs per k16 step (column
      // halves of the accumulator, adjacent in TMEM so the epilogue is unchanged):
      // back-to-back MMAs into one accumulator serialise on it, so with a single
      // chain the 1-CTA kernel ran at ~250 cycles per MMA whatever N was.
      constexpr int NSPLIT = MLRA_NSPLIT;
      constexpr int NH = BN / NSPLIT;
      constexpr uint32_t idesc_main = idesc_bf16(BM, NH, MN ? 1u : 0u, 0u);
      constexpr uint32_t idesc_kmaj = idesc_bf16(BM, NH, 0u, 0u);
      int s = 0;
      uint32_t ph = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t aph = (local >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < n_kb; ++kb) {
          const long long f0 = tl ? clock64() : 0;
          mbar_wait(&full[s], ph);
          if (tl) tl[1] += clock64() - f0;
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
#pragma unroll
            for (int h = 0; h < NSPLIT; ++h) {
              const uint64_t bdesc = sdesc_sw128(st + h * NH * 128 + k * 32, 16, 1024);
              tc_mma_f16(tmem_d + h * NH, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          tc_commit(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ Q-ring TMA
    if (QTMA && !W_TMA && lane == 0) {
      const uint32_t qbytes = p.q_codes_bytes + p.q_grid_bytes;
      int qs = 0;
      uint32_t qph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        it.coords(tile, m_tile, n_tile);
        for (int pr = 0; pr < n_kb_main / 2; ++pr) {
          mbar_wait_backoff<PROD_NS>(&qempty[qs], qph ^ 1);
          mbar_arrive_expect_tx(&qfull[qs], qbytes);
          uint8_t* dst = sQ + qs * p.q_stage_bytes;
          // grid boxes start on an even group: TMA box starts must be 16-byte aligned
          if (!MN) {  // rows = weight rows of the tile, bytes = codes [pr*128, pr*128+128)
            tma_load_2d(dst, &tm_codes, &qfull[qs], pr * 16 * BITS, m_tile * BM);
            tma_load_2d(dst + p.q_codes_bytes, &tm_grid, &qfull[qs],
                        2 * (pair_group(pr, p) & ~1), m_tile * BM);
          } else {    // rows = weight rows [pr*128, +128), bytes = codes of tile columns
            tma_load_2d(dst, &tm_codes, &qfull[qs], m_tile * 16 * BITS, pr * 128);
            tma_load_2d(dst + p.q_codes_bytes, &tm_grid, &qfull[qs],
                        2 * (pair_group(m_tile, p) & ~1), pr * 128);
          }
          if (++qs == p.q_stages) {
            qs = 0;
            qph ^= 1;
          }
        }
      }
    }
  } else if (warp >= EPI_WARP0 && warp < DQ_WARP0) {
    // ------------------------------------------------------------ epilogue
    const int qd = warp & 3;  // TMEM lane quadrant this warp may access
    int local = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++local) {
      int m_tile, n_tile;
      it.coords(tile, m_tile, n_tile);
      const int acc = local & 1;
      const uint32_t aph = (local >> 1) & 1;
      mbar_wait_backoff<EPI_NS>(&tfull[acc], aph);
      tc_fence_after();
      const int64_t wrow = static_cast<int64_t>(m_tile) * BM + qd * 32 + lane;
      const bool row_ok = wrow < p.m_valid;
      const float bias = (p.bias != nullptr && row_ok) ? p.bias[wrow] : 0.0f;
      const int64_t t0 = static_cast<int64_t>(n_tile) * BN;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  } else if (warp >= DQ_WARP0) {
    // ------------------------------------------------------------ dequant producers
    // Two groups of 4 warps; group g owns the pipeline stages with (s & 1) == g,
    // so each stage waits on 4 warps and the groups run a stage apart.
    const int grp = (warp - DQ_WARP0) >> 2;
    const int gtid = threadIdx.x - (DQ_WARP0 + 4 * grp) * 32;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    if constexpr (W_TMA) {
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int kb = 0; kb < n_kb; ++kb) {
          if ((s & 1) == grp) {
            mbar_wait(&empty[s], ph ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    } else if constexpr (QTMA) {
      // Per-thread constants. Unit u = i*128 + gtid (i < 8) of a 1024-unit stage:
      //   K-major: row r = i*16 + gtid/8 (Q row r), unit k8 = gtid%8 (+8 for odd kb)
      //   MN:      row n = i*8 + gtid/16 (Q row n, +64 for odd kb), unit k8 = gtid%16
      constexpr int UPT = UNITS_PER_GROUP_THREAD;
      uint32_t soff[UPT];
#pragma unroll
      for (int i = 0; i < UPT; ++i) soff[i] = unit_soff<MN>(i * 128 + gtid);
      const int k8 = MN ? (gtid & 15) : (gtid & 7);
      const int row0 = MN ? (gtid >> 4) : (gtid >> 3);
      constexpr int ROW_STEP = MN ? 8 : 16;
      const int gshift = p.q_group_shift;  // log2(group) when group < 128, else -1
      const int gbox = p.q_grid_bytes / BM;  // grid bytes per Q row
      const uint32_t sQ32 = smem_u32(sQ), sW32 = smem_u32(sW);
      int qs = 0;
      uint32_t qph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        it.coords(tile, m_tile, n_tile);
        // g >= 128: one group per 128-code block; which half of the 2-group box
        const int gpar_mn = pair_group(m_tile, p) & 1;
        for (int kb = 0; kb < n_kb; ++kb) {
          const bool main = kb < n_kb_main;
          const int kp = kb & 1;
          if ((s & 1) == grp) {
            const long long c0 = tl ? clock64() : 0;
            if (main) mbar_wait(&qfull[qs], qph);
            const long long c1 = tl ? clock64() : 0;
            mbar_wait(&empty[s], ph ^ 1);
            const long long c2 = tl ? clock64() : 0;
            if (main) {
              const uint32_t qc = sQ32 + qs * p.q_stage_bytes;
              const uint32_t qg = qc + p.q_codes_bytes;
              const uint32_t st = sW32 + s * W_TILE;
              const int unit = MN ? k8 : (k8 + 8 * kp);
              const int code = unit * 8;  // first code of the unit within the 128-code block
              const int gsub = gshift >= 0 ? (code >> gshift)
                                           : (MN ? gpar_mn : (pair_group(kb >> 1, p) & 1));
              const int rbase = MN ? (row0 + 64 * kp) : row0;
              dequant_units<BITS, UPT, ROW_STEP>(qc, qg, st, soff, unit, gsub, rbase, gbox);
              fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&full[s]);
              if (main) mbar_arrive(&qempty[qs]);
            }
            if (tl && gtid == 0) {  // dev-only: group leader's wait/compute cycles
              const long long c3 = clock64();
              atomicAdd(reinterpret_cast<unsigned long long*>(tl + 2 + 3 * grp), c1 - c0);
              atomicAdd(reinterpret_cast<unsigned long long*>(tl + 3 + 3 * grp), c2 - c1);
              atomicAdd(reinterpret_cast<unsigned long long*>(tl + 4 + 3 * grp), c3 - c2);
            }
          }
          if (main && kp == 1) {
            if (++qs == p.q_stages) {
              qs = 0;
              qph ^= 1;
            }
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    } else {
      // generic LDG path (odd group sizes / 8-bit codes)
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m_tile, n_tile;
        it.coords(tile, m_tile, n_tile);
        for (int kb = 0; kb < n_kb; ++kb) {
          if ((s & 1) == grp) {
            mbar_wait(&empty[s], ph ^ 1);
            if (kb < n_kb_main) {
              uint8_t* stile = sW + s * W_TILE;
#pragma unroll 2
              for (int i = 0; i < UNITS_PER_GROUP_THREAD; ++i) {
                const int u = i * 128 + gtid;
                int64_t wrow, wunit;
                if constexpr (!MN) {
                  wrow = static_cast<int64_t>(m_tile) * BM + (u >> 3);
                  wunit = static_cast<int64_t>(kb) * (BK / 8) + (u & 7);
                } else {
                  wrow = static_cast<int64_t>(kb) * BK + (u >> 4);
                  wunit = static_cast<int64_t>(m_tile) * (BM / 8) + (u & 15);
                }
                const uint64_t v = load_unit<BITS>(q.words + wrow * q.row_words, wunit);
                *reinterpret_cast<uint4*>(stile + unit_soff<MN>(u)) =
                    deq8_bf16_general<BITS>(v, q.grid + wrow * q.ng_pad, wunit * 8, q.group);
              }
              fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (tl && threadIdx.x == 0) tl[0] = clock64() - t_entry;
  if (warp == 1) tmem_dealloc(tmem_base, TMEM_COLS);
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <int BITS, bool W_TMA, bool MN, bool OUT_F32, bool QTMA, int TBN>
cudaError_t launch_t(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                     cudaStream_t stream) {
  auto kern = qgemm_kernel<BITS, W_TMA, MN, OUT_F32, QTMA, TBN>;
  const int smem = qgemm1_smem_fixed(TBN) + p.q_stages * p.q_stage_bytes;
  static int smem_set = 0;  // per instantiation: the opt-in only ever grows
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  const int64_t tiles = (p.m_total / BM) * ((p.tokens + TBN - 1) / TBN);
  const int grid = static_cast<int>(tiles < num_sms() ? tiles : num_sms());
  return launch_pdl(kern, dim3(grid), dim3(NUM_THREADS), smem, stream, p.no_pdl == 0, maps.act, maps.act_lora,
                    maps.w, maps.w_lora, maps.codes, maps.grid, q, p);
}

template <int BITS, bool W_TMA, bool QTMA, int TBN>
cudaError_t launch_mo(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool mn,
                      bool out_f32, cudaStream_t st) {
  if (mn) return out_f32 ? launch_t<BITS, W_TMA, true, true, QTMA, TBN>(maps, q, p, st)
                         : launch_t<BITS, W_TMA, true, false, QTMA, TBN>(maps, q, p, st);
  return out_f32 ? launch_t<BITS, W_TMA, false, true, QTMA, TBN>(maps, q, p, st)
                 : launch_t<BITS, W_TMA, false, false, QTMA, TBN>(maps, q, p, st);
}

template <int TBN>
cudaError_t launch_bits(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool w_tma,
                        bool mn, bool out_f32, cudaStream_t stream) {
  if (w_tma) return launch_mo<4, true, false, TBN>(maps, q, p, mn, out_f32, stream);
  const bool qtma = p.q_stages > 0;
  switch (q.bits) {
    case 2: return qtma ? launch_mo<2, false, true, TBN>(maps, q, p, mn, out_f32, stream)
                        : launch_mo<2, false, false, TBN>(maps, q, p, mn, out_f32, stream);
    case 3: return qtma ? launch_mo<3, false, true, TBN>(maps, q, p, mn, out_f32, stream)
                        : launch_mo<3, false, false, TBN>(maps, q, p, mn, out_f32, stream);
    case 4: return qtma ? launch_mo<4, false, true, TBN>(maps, q, p, mn, out_f32, stream)
                        : launch_mo<4, false, false, TBN>(maps, q, p, mn, out_f32, stream);
    case 8: return launch_mo<8, false, false, TBN>(maps, q, p, mn, out_f32, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

bool qgemm_q_tma_ok(const QWeightDev& q) {
  const int64_t g = q.group;
  const bool g_ok = (g == 32 || g == 64 || g % 128 == 0);
  return (q.bits == 2 || q.bits == 3 || q.bits == 4) && g_ok;
}

int qgemm_max_q_stages(int q_stage_bytes, int extra_smem) {
  int qs = (SMEM_LIMIT - SMEM_FIXED - extra_smem) / q_stage_bytes;
  return qs > MAX_QS ? MAX_QS : qs;
}

cudaError_t qgemm_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                         bool w_tma, bool mn, bool out_f32, cudaStream_t stream) {
  if (p.tokens <= 0 || p.m_total <= 0) return cudaSuccess;
  if (p.bn == 128) return launch_bits<128>(maps, q, p, w_tma, mn, out_f32, stream);
  if (p.bn == 256) return launch_bits<256>(maps, q, p, w_tma, mn, out_f32, stream);
  return cudaErrorInvalidValue;
}

}  // namespace mlra

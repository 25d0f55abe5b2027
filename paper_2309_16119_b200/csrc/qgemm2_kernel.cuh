// qgemm2_kernel.cuh — K2/K3 on CTA pairs: cta_group::2 tcgen05 with two accumulators.
//
// Same products as qgemm.cu (forward Y = X·Ŵᵀ + LoRA, dX = dY·Ŵ + LoRA;
// lowprec_linear.cpp:150-247, lora.cpp:68-71, autodiff.cpp:150-152), but each
// pair tile is 256 weight-side rows (128 per CTA, each CTA dequantizes only its
// own half) x 512 tokens (two N=256 accumulators of 256 TMEM columns each; each
// CTA stages 128 tokens of every 256-token half). Every dequantized weight
// element now feeds 512 tokens of MMA instead of 256, and every activation tile
// read from L2 feeds 256 weight rows instead of 128 — halving both the
// dequant-issue and the L2-traffic cost per FLOP relative to the 1-CTA kernel.
//
// Pair protocol (the leader is cluster rank 0):
//  * operand TMA: each CTA loads its own halves with cta_group::2 TMA whose
//    completion counts on the LEADER's full barrier; only the leader arms it
//    (expect_tx = both CTAs' bytes);
//  * dequant warps of both CTAs arrive (remote, release.cluster) on the
//    leader's full barrier after fence.proxy.async;
//  * the leader's single MMA thread issues tcgen05.mma.cta_group::2 (M=256,
//    N=256) for both accumulators and commits empty/tfull to both CTAs
//    (multicast);
//  * each CTA's epilogue drains its own 128 TMEM lanes, then arrives (remote)
//    on the leader's tempty before the next tile may overwrite TMEM.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "ptx.cuh"
#include "qgemm.h"
#include "qgemm_dev.cuh"


namespace mlra {

// The pair kernel's four families (forward / dX x whole tiles / stream-K and
// split-K), one translation unit each (qgemm2_f0.cu .. qgemm2_d1.cu).
cudaError_t qgemm2_launch_f0(const GemmMaps&, const QWeightDev&, const GemmArgs&, bool, bool, cudaStream_t);
cudaError_t qgemm2_launch_f1(const GemmMaps&, const QWeightDev&, const GemmArgs&, bool, bool, cudaStream_t);
cudaError_t qgemm2_launch_d0(const GemmMaps&, const QWeightDev&, const GemmArgs&, bool, bool, cudaStream_t);
cudaError_t qgemm2_launch_d1(const GemmMaps&, const QWeightDev&, const GemmArgs&, bool, bool, cudaStream_t);

namespace {

using namespace qg;

// Dev-only instrumentation (MLRA_TRACE / MLRA_TRACE2 at run time) is compiled in
// only with -DMLRA_DEV_TRACE (make EXTRA=-DMLRA_DEV_TRACE): the production
// kernel carries none of its registers or branches.
#ifdef MLRA_DEV_TRACE
constexpr bool kDevTrace = true;
#else
constexpr bool kDevTrace = false;
#endif
constexpr uint32_t TMEM_COLS = 512;  // two N=256 accumulators
constexpr int kFixChunkBytes = 32 * 128 * 4;  // one stream-K partial chunk: 32 tokens x 128 rows
constexpr int kFixSlots = STAGES * (W_TILE + T_TILE) / kFixChunkBytes;  // staged in the idle ring
constexpr int kSplitMaxS = 8;  // split-K ways: (S - 1) partial slabs of one chunk fit the ring
static_assert(kSplitMaxS - 1 <= kFixSlots, "split-K fix-up ring");
constexpr int HB = 128;            // tokens per CTA per accumulator (MMA N=256 split in two)
constexpr int HB_TILE = HB * BK * 2;  // 16 KB
constexpr int PAIR_ROWS = 2 * BM;  // 256 weight-side rows per pair tile
constexpr int PAIR_TOK = 2 * 2 * HB;  // 512 tokens per pair tile
static_assert(2 * HB_TILE == T_TILE, "stage layout shared with the 1-CTA kernel");
static_assert(kSkSlotFloats == 2LL * PAIR_TOK * BM, "stream-K slot = both CTAs' accumulators");

// Work schedule shared by every warp role: a sequence of segments (tile,
// k-blocks [kb0, kb1)) for this pair.
//  * whole tiles (sk_pairs == 0): tiles cid, cid + ncl, ... each [0, n_kb);
//  * stream-K: the tile-major space of n_tiles * n_kb k-blocks is cut into
//    sk_pairs contiguous ranges, so every pair gets the same MMA work however
//    the tile count divides the SM count. Cuts land on even k-block offsets
//    inside a tile (a Q-ring stage holds two k-blocks). A segment that starts
//    at k-block 0 but ends early OWNS its tile: it adds the fp32 partials of
//    the following pairs' first segments (in pair order — deterministic) and
//    stores the result. A pair's first segment may start mid-tile: it writes
//    its accumulators as a partial and publishes a flag. Owners process their
//    part last in their range, so the partials they need are normally ready.
// Start (tile, k-block) of pair q's range (q = sk_pairs: the end of the space).
// Same formula as the host planner (qgemm2.cu set_split / stream-K cuts): cuts
// land on even k-block offsets (a Q-ring stage holds two k-blocks).
__device__ __forceinline__ void sk_cut(const GemmArgs& p, int n_kb, int n_tiles, int q, int& t,
                                       int& kb) {
  if (p.split > 0) {
    const int S = p.split;
    t = q / S;
    int b = n_kb * (q - t * S) / S;
    if (b & 1) ++b;
    kb = b;
  } else {
    const long long total = static_cast<long long>(n_tiles) * n_kb;
    long long b = total * q / p.sk_pairs;
    if ((b % n_kb) & 1) ++b;
    t = static_cast<int>(b / n_kb);
    kb = static_cast<int>(b % n_kb);
  }
}

template <bool SK>
struct SegSched {
  int t, kb, t_end, kb_end, n_kb, n_tiles, stride;
  static constexpr bool sk = SK;
  __device__ void init(const GemmArgs& p, int cid, int ncl, int tiles, int nkb) {
    n_kb = nkb;
    n_tiles = tiles;
    if (sk) {
      // called by full, converged warps: the REDUX broadcast puts the cuts in
      // uniform registers, keeping the MMA issuer's loop (and its smem
      // descriptors) on the uniform datapath instead of an R2UR waterfall
      int t0, k0, t1, k1;
      sk_cut(p, nkb, tiles, cid, t0, k0);
      sk_cut(p, nkb, tiles, cid + 1, t1, k1);
      t = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(t0)));
      kb = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(k0)));
      t_end = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(t1)));
      kb_end = static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(k1)));
    } else {
      t = cid;
      stride = ncl;
    }
  }
  __device__ bool next(int& tile, int& kb0, int& kb1) {
    if (!sk) {
      if (t >= n_tiles) return false;
      tile = t;
      kb0 = 0;
      kb1 = n_kb;
      t += stride;
      return true;
    }
    if (t > t_end || (t == t_end && kb >= kb_end)) return false;
    tile = t;
    kb0 = kb;
    kb1 = t == t_end ? kb_end : n_kb;
    ++t;
    kb = 0;
    return true;
  }
  // number of segments next() will yield
  __device__ int count() const {
    if (!sk) return t < n_tiles ? (n_tiles - 1 - t) / stride + 1 : 0;
    if (t > t_end || (t == t_end && kb >= kb_end)) return 0;
    return t_end - t + (kb_end > 0 ? 1 : 0);
  }
  // pairs (cid, q_end) whose ranges start inside `tile` (the owner's contributors)
  __device__ int contrib_end(const GemmArgs& p, int cid, int tile) const {
    int q = cid + 1;
    while (q < p.sk_pairs) {
      int tq, kq;
      sk_cut(p, n_kb, n_tiles, q, tq, kq);
      if (tq != tile) break;
      ++q;
    }
    return q;
  }
};

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void epi_bar_sync() {  // the 4 epilogue warps only
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// One drained chunk (32 tokens x this thread's weight row) -> output (+bias).
// bf16 output, paired rows: lanes 2i / 2i+1 swap half their tokens with one
// shfl.xor so each stores a 32-bit word (rows 2i, 2i+1) for one token; the
// pointer advances by ldo words. Needs even ldo and a 4-byte aligned output
// (p.out_pairs) and every row of the warp valid (`pairs`, warp-uniform);
// otherwise the scalar path.
template <bool OUT_F32>
__device__ __forceinline__ void epi_store(const GemmArgs& p, const uint32_t (&r)[32], int64_t t0,
                                          int64_t wrow, bool row_ok, float bias, float bias_nb,
                                          bool pairs, bool odd) {
  if constexpr (!OUT_F32) {
    if (pairs && t0 + 32 <= p.tokens) {
      const float b_lo = odd ? bias_nb : bias, b_hi = odd ? bias : bias_nb;
      uint32_t* o = reinterpret_cast<uint32_t*>(
          reinterpret_cast<__nv_bfloat16*>(p.out) + (t0 + odd) * p.ldo + (wrow & ~1ll));
      const int64_t step = p.ldo;  // two tokens = ldo 32-bit words
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float ev = __uint_as_float(r[2 * k]), ov = __uint_as_float(r[2 * k + 1]);
        const float mine = odd ? ov : ev;
        const float other = __shfl_xor_sync(0xffffffffu, odd ? ev : ov, 1);
        const float lo = odd ? other : mine, hi = odd ? mine : other;
        *o = pack_bf16x2(lo + b_lo, hi + b_hi);
        o += step;
      }
      return;
    }
  }
  if (!row_ok) return;
  if (t0 + 32 <= p.tokens) {
    if constexpr (OUT_F32) {
      float* o = reinterpret_cast<float*>(p.out) + t0 * p.ldo + wrow;
#pragma unroll
      for (int j = 0; j < 32; ++j, o += p.ldo) *o = __uint_as_float(r[j]) + bias;
    } else {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + t0 * p.ldo + wrow;
#pragma unroll
      for (int j = 0; j < 32; ++j, o += p.ldo) *o = __float2bfloat16_rn(__uint_as_float(r[j]) + bias);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (t0 + j < p.tokens) {
        const float v = __uint_as_float(r[j]) + bias;
        if constexpr (OUT_F32)
          reinterpret_cast<float*>(p.out)[(t0 + j) * p.ldo + wrow] = v;
        else
          reinterpret_cast<__nv_bfloat16*>(p.out)[(t0 + j) * p.ldo + wrow] = __float2bfloat16_rn(v);
      }
    }
  }
}

// Split-K fix-up (p.split = S > 0: every pair runs one (tile, k-range) unit),
// run by all 16 warps of the CTA once its MMAs are complete. The S pairs of a
// tile each own 16/S of its 16 token chunks (32 tokens x 128 rows). Warp w
// reads TMEM lane quadrant w & 3 and takes chunks w >> 2, +4, ...:
//  1. non-owned chunks -> this pair's fp32 partial slots (coalesced rows);
//  2. publish (one release after a CTA barrier), acquire the tile's other pairs;
//  3. one thread stages every (owned chunk, other pair) 16 KB slab into the
//     idle operand ring with cp.async.bulk (all in flight at once, rounds only
//     when they exceed the ring), and each owned chunk is summed in pair order
//     (deterministic: identical bits for identical inputs) with the TMEM
//     accumulator and stored.
template <bool OUT_F32>
__device__ __forceinline__ void split_fixup(const GemmArgs& p, int cid, uint32_t rank, int m_pairs,
                                            uint32_t tmem_base, uint64_t* tfull, uint64_t* fixb,
                                            uint8_t* smem, unsigned long long* tl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qd = warp & 3, wg = warp >> 2;
  mbar_wait_backoff<EPI_NS>(tfull, 0);
  tc_fence_after();
  if (tl && threadIdx.x == 0) tl[2] = gtime();
  const int S = p.split;
  const int tile = cid / S, q0 = tile * S, sidx = cid - q0;
  const int mp = tile % m_pairs, np = tile / m_pairs;
  const int nch = p.tok256 ? 8 : 16;  // 32-token chunks per tile
  const int tok_tile = 32 * nch;
  const int c0 = nch * sidx / S, c1 = nch * (sidx + 1) / S;
  const int r_in = qd * 32 + lane;
  const int64_t wrow = static_cast<int64_t>(mp) * PAIR_ROWS + rank * BM + r_in;
  const bool row_ok = wrow < p.m_valid;
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16);
  auto slot_of = [&](int q, int cc) {  // [512 tokens][128 rows] fp32 per CTA
    return p.sk_ws + (2 * static_cast<int64_t>(q) + rank) * (PAIR_TOK * BM) +
           static_cast<int64_t>(cc * 32) * BM;
  };
  // 1. partials of the chunks other pairs own
  for (int cc = wg; cc < nch; cc += 4) {
    if (cc >= c0 && cc < c1) continue;
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + cc * 32, r);
    tc_wait_ld();
    if (row_ok) {
      float* d = slot_of(cid, cc) + r_in;
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j * BM] = __uint_as_float(r[j]);
    }
  }
  // 2. publish: the CTA barrier orders every thread's partial stores before one
  // thread's gpu-scope release (cumulative); it acquires the other pairs' flags
  __syncthreads();
  if (tl && threadIdx.x == 0) tl[5] = gtime();
  if (threadIdx.x == 0) {
    st_release_gpu(&p.sk_flags[2 * cid + rank], 1u);
    for (int q = q0; q < q0 + S; ++q)
      if (q != cid)
        while (ld_acquire_gpu(&p.sk_flags[2 * q + rank]) == 0) __nanosleep(32);
    fence_proxy_async_global();  // acquired partials (generic writes) -> async-proxy reads
    if (tl) tl[3] = gtime();
  }
  const float bias = (p.bias != nullptr && row_ok) ? p.bias[wrow] : 0.0f;
  const float bias_nb = __shfl_xor_sync(0xffffffffu, bias, 1);
  const bool odd = lane & 1;
  const bool pairs = p.out_pairs && __all_sync(0xffffffffu, (wrow | 1) < p.m_valid);
  const int nq = S - 1, nc = c1 - c0;
  // owned chunks staged per round (S <= kSplitMaxS); S == 1: whole tiles, no partials
  const int per_round = nq > 0 ? kFixSlots / nq : nc;
  const uint32_t ring = smem_u32(smem);
  int round = 0;
  for (int b0 = 0; b0 < nc; b0 += per_round, ++round) {
    const int nb = nc - b0 < per_round ? nc - b0 : per_round;
    __syncthreads();  // the ring is free (round 0: every MMA has completed; else: consumed)
    if (threadIdx.x == 0) {
      for (int i = 0; i < nb; ++i)
        for (int k = 0; k < nq; ++k) {
          const int q = q0 + k + (k >= sidx ? 1 : 0), slot = i * nq + k;
          mbar_arrive_expect_tx(&fixb[slot], kFixChunkBytes);
          bulk_g2s(ring + slot * kFixChunkBytes, slot_of(q, c0 + b0 + i), kFixChunkBytes,
                   &fixb[slot]);
        }
    }
    for (int i = wg; i < nb; i += 4) {
      const int cc = c0 + b0 + i;
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + cc * 32, r);
      tc_wait_ld();
      float acc[32];
      for (int qi = 0; qi < S; ++qi) {  // pair order
        if (qi == sidx) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            acc[j] = qi == 0 ? __uint_as_float(r[j]) : acc[j] + __uint_as_float(r[j]);
        } else {
          const int slot = i * nq + qi - (qi > sidx ? 1 : 0);
          mbar_wait(&fixb[slot], static_cast<uint32_t>(round & 1));
          if (tl && round == 0 && i == 0 && lane == 0 && warp == 0) tl[7] = gtime();
          const float* src = reinterpret_cast<const float*>(smem + slot * kFixChunkBytes) + r_in;
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] = qi == 0 ? src[j * BM] : acc[j] + src[j * BM];
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(acc[j]);
      epi_store<OUT_F32>(p, r, static_cast<int64_t>(np) * tok_tile + cc * 32, wrow, row_ok, bias,
                         bias_nb, pairs, odd);
    }
  }
  if (tl) {
    __syncthreads();
    if (threadIdx.x == 0) tl[4] = gtime();
  }
}

// Stream-K owner fix-up of the pair's LAST segment (tile, k-blocks [0, kb_end)),
// run by all 16 warps once every MMA of the CTA has completed (the 4 epilogue
// warps alone took ~12 us after the last MMA at 1024 tokens, profiles/r03x).
// Contributors (pairs cid+1 .. cid+nc) each published the fp32 partial of the
// tile's remaining k-blocks. One thread acquires their flags and stages the
// (chunk, contributor) 16 KB slabs into the idle operand ring in rounds of
// kFixSlots / nc chunks; warp w (TMEM lane quadrant w & 3) takes chunks
// w >> 2, +4, ... of each round and sums own + partials in pair order — the
// same order as the 4-warp path, so the bits are unchanged.
template <bool OUT_F32>
__device__ __forceinline__ void sk_owner_fixup(const GemmArgs& p, int cid, uint32_t rank,
                                               int m_pairs, int tile, int nc, uint32_t tfull_par,
                                               uint32_t tmem_base, uint64_t* tfull, uint64_t* fixb,
                                               uint8_t* smem, unsigned long long* tl) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qd = warp & 3, wg = warp >> 2;
  mbar_wait_backoff<EPI_NS>(tfull, tfull_par);
  tc_fence_after();
  if (tl && threadIdx.x == 0) tl[2] = gtime();
  const int mp = tile % m_pairs, np = tile / m_pairs;
  const int r_in = qd * 32 + lane;
  const int64_t wrow = static_cast<int64_t>(mp) * PAIR_ROWS + rank * BM + r_in;
  const bool row_ok = wrow < p.m_valid;
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16);
  auto slot_of = [&](int q, int cc) {  // [512 tokens][128 rows] fp32 per CTA
    return p.sk_ws + (2 * static_cast<int64_t>(q) + rank) * (PAIR_TOK * BM) +
           static_cast<int64_t>(cc * 32) * BM;
  };
  if (threadIdx.x == 0) {
    for (int q = cid + 1; q <= cid + nc; ++q)
      while (ld_acquire_gpu(&p.sk_flags[2 * q + rank]) == 0) __nanosleep(64);
    fence_proxy_async_global();  // acquired partials (generic writes) -> async-proxy reads
    if (tl) tl[3] = gtime();
  }
  const float bias = (p.bias != nullptr && row_ok) ? p.bias[wrow] : 0.0f;
  const float bias_nb = __shfl_xor_sync(0xffffffffu, bias, 1);
  const bool odd = lane & 1;
  const bool pairs = p.out_pairs && __all_sync(0xffffffffu, (wrow | 1) < p.m_valid);
  const int per_round = kFixSlots / nc;
  const uint32_t ring = smem_u32(smem);
  int round = 0;
  for (int b0 = 0; b0 < 16; b0 += per_round, ++round) {
    const int nb = 16 - b0 < per_round ? 16 - b0 : per_round;
    __syncthreads();  // the ring is free (round 0: every MMA has completed; else: consumed)
    if (threadIdx.x == 0) {
      for (int i = 0; i < nb; ++i)
        for (int k = 0; k < nc; ++k) {
          const int slot = i * nc + k;
          mbar_arrive_expect_tx(&fixb[slot], kFixChunkBytes);
          bulk_g2s(ring + slot * kFixChunkBytes, slot_of(cid + 1 + k, b0 + i), kFixChunkBytes,
                   &fixb[slot]);
        }
    }
    for (int i = wg; i < nb; i += 4) {
      const int cc = b0 + i;
      uint32_t r[32];
      tmem_ld_32x32b_x32(taddr + cc * 32, r);
      tc_wait_ld();
      for (int k = 0; k < nc; ++k) {  // pair order: deterministic sums
        const int slot = i * nc + k;
        mbar_wait(&fixb[slot], static_cast<uint32_t>(round & 1));
        const float* src = reinterpret_cast<const float*>(smem + slot * kFixChunkBytes) + r_in;
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(__uint_as_float(r[j]) + src[j * BM]);
      }
      epi_store<OUT_F32>(p, r, static_cast<int64_t>(np) * PAIR_TOK + cc * 32, wrow, row_ok, bias,
                         bias_nb, pairs, odd);
    }
  }
  if (tl) {
    __syncthreads();
    if (threadIdx.x == 0) tl[4] = gtime();
  }
}

template <int BITS, bool W_TMA, bool MN, bool OUT_F32, bool QTMA, bool SK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    qgemm2_kernel(const __grid_constant__ CUtensorMap tm_act,
                  const __grid_constant__ CUtensorMap tm_act_lora,
                  const __grid_constant__ CUtensorMap tm_w,
                  const __grid_constant__ CUtensorMap tm_w_lora,
                  const __grid_constant__ CUtensorMap tm_codes,
                  const __grid_constant__ CUtensorMap tm_grid, const QWeightDev q,
                  const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sW = smem;
  uint8_t* sT = sW + STAGES * W_TILE;
  uint8_t* sQ = sT + STAGES * T_TILE;
  constexpr bool CB2 = BITS == kCb2Bits;
  constexpr bool E8P = BITS == kE8pBits;
  constexpr bool LUT = is_lut<BITS>();
  constexpr int QB = q_geom_bits<BITS>();  // packed-stream geometry
  uint8_t* sCb = sQ + p.q_stages * p.q_stage_bytes;  // cb2 codebook / lut levels
  uint64_t* full = reinterpret_cast<uint64_t*>(
      sCb + (CB2 ? kCb2SmemBytes : (E8P ? kE8pSmemBytes : (LUT ? kLutSmemBytes : 0))));
  uint64_t* empty = full + STAGES;
  uint64_t* qfull = empty + STAGES;
  uint64_t* qempty = qfull + MAX_QS;
  uint64_t* tfull = qempty + MAX_QS;
  uint64_t* tempty = tfull + 1;    // accumulator 0 (tokens 0..255 of the pair tile) drained
  uint64_t* tempty1 = tempty + 1;  // accumulator 1 drained
  uint64_t* fixb = tempty1 + 1;    // stream-K owner fix-up: staged partial chunks landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixb + kFixSlots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  // dev-only timeline (MLRA_TRACE2): globaltimer ns per CTA at entry, MMA done,
  // each epilogue tile's tfull, contributor flags seen, epilogue done
  unsigned long long* tl = (kDevTrace && p.trace2) ? p.trace2 + 8 * blockIdx.x : nullptr;
  if (tl && threadIdx.x == 0) tl[0] = gtime();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int n_kb_main = p.n_kb_main;
  const int n_kb = p.n_kb_main + p.n_kb_lora;
  const int m_pairs = static_cast<int>(p.m_total / PAIR_ROWS);
  // split-K plans may use 256-token pair tiles (one accumulator, half the
  // partial volume per split; p.tok256)
  const bool one_acc = SK && p.tok256;
  const int tok_tile = one_acc ? PAIR_TOK / 2 : PAIR_TOK;
  const int n_pairs = static_cast<int>((p.tokens + tok_tile - 1) / tok_tile);
  const int n_tiles = m_pairs * n_pairs;
  SegSched<SK> sched;
  sched.init(p, cid, ncl, n_tiles, n_kb);
  // warp-uniform schedule summary for the MMA issuer (REDUX -> uniform registers)
  const int mma_nseg =
      static_cast<int>(__reduce_min_sync(0xffffffffu, static_cast<unsigned>(sched.count())));
  const int mma_kb_first = static_cast<int>(
      __reduce_min_sync(0xffffffffu, static_cast<unsigned>(sched.sk ? sched.kb : 0)));
  const int mma_kb_last = static_cast<int>(
      __reduce_min_sync(0xffffffffu, static_cast<unsigned>(sched.sk ? sched.kb_end : 0)));
  // stream-K: a last segment [0, kb_end) of tile t_end owns that tile and adds
  // the partials of pairs cid+1 .. cid+own_nc; all 16 warps run its fix-up
  // (sk_owner_fixup) unless the ring cannot stage one chunk of every partial
  const bool own_last = SK && p.split == 0 && !p.sk_owner4 && sched.kb_end > 0 &&
                        (sched.t_end != sched.t || sched.kb == 0);
  auto own_count = [&]() {  // contributors of the last segment's tile (0: 4-warp path)
    const int nc = sched.contrib_end(p, cid, sched.t_end) - cid - 1;
    return nc <= kFixSlots ? nc : 0;
  };

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
      mbar_init(&full[s], 1 + 2 * (NUM_DQ_WARPS / 2));  // leader's is the live one
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < MAX_QS; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], NUM_DQ_WARPS);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * 4);
    mbar_init(tempty1, 2 * 4);
    for (int i = 0; i < kFixSlots; ++i) mbar_init(&fixb[i], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, TMEM_COLS);
  pdl_trigger();
  pdl_wait();  // every operand (activations, LoRA planes, flags) may come from earlier kernels
  if constexpr (E8P) {  // the e8p decode table (dequant_units_e8p), from the (|a| +- 1/4) rows
    if (threadIdx.x < 256) {  // |a| = (|a| + 1/4) - 1/4, bf16-exact; odd bit -> sign bit of entry 0
      const uint4* src = reinterpret_cast<const uint4*>(p.cb2_codebook);
      const uint4 pr = __ldg(src + threadIdx.x);
      const uint32_t odd = (__ldg(reinterpret_cast<const uint32_t*>(src + 512) + (threadIdx.x >> 5)) >>
                            (threadIdx.x & 31)) & 1u;
      const uint32_t pw[4] = {pr.x, pr.y, pr.z, pr.w};
      uint32_t aw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        aw[q] = pack_bf16x2(__uint_as_float(pw[q] << 16) - 0.25f,
                            __uint_as_float(pw[q] & 0xFFFF0000u) - 0.25f);
      reinterpret_cast<uint4*>(sCb)[threadIdx.x] = make_uint4(aw[0] | (odd << 15), aw[1], aw[2], aw[3]);
    }
  }
  if constexpr (CB2) {  // stage the 4 KB codebook (read by this CTA's dequant warps)
    if (threadIdx.x < kCb2SmemBytes / 16)
      reinterpret_cast<uint4*>(sCb)[threadIdx.x] =
          __ldg(reinterpret_cast<const uint4*>(p.cb2_codebook) + threadIdx.x);
  }
  if constexpr (LUT) {
    if (threadIdx.x < kLutSmemBytes / 4)
      reinterpret_cast<float*>(sCb)[threadIdx.x] = __ldg(p.lut + threadIdx.x);
  }
  tc_fence_before();
  cluster_sync();  // barrier inits visible to the peer before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ operand TMA (both CTAs)
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      SegSched<SK> sc = sched;
      int tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        const int mp = tile % m_pairs, np = tile / m_pairs;
        const int cb = mp * 2 + static_cast<int>(rank);  // this CTA's 128-row block
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_backoff<PROD_NS>(&empty[s], ph ^ 1);
          const bool lora = kb >= n_kb_main;
          const bool w_tma = lora || W_TMA;
          if (leader)
            mbar_arrive_expect_tx(&full[s],
                                  2 * ((one_acc ? HB_TILE : T_TILE) + (w_tma ? W_TILE : 0)));
          uint8_t* st = sT + s * T_TILE;
          uint8_t* sw = sW + s * W_TILE;
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            if (a == 1 && one_acc) break;
            const int tok = np * tok_tile + a * 2 * HB + static_cast<int>(rank) * HB;
            if (!lora)
              tma_load_2d_2sm(st + a * HB_TILE, &tm_act, &full[s], kb * BK, tok);
            else
              tma_load_2d_2sm(st + a * HB_TILE, &tm_act_lora, &full[s], (kb - n_kb_main) * BK, tok);
          }
          if (lora) {
            tma_load_2d_2sm(sw, &tm_w_lora, &full[s], (kb - n_kb_main) * BK, cb * BM);
          } else if (W_TMA) {
            if (!MN) {
              tma_load_2d_2sm(sw, &tm_w, &full[s], kb * BK, cb * BM);
            } else {
              tma_load_2d_2sm(sw, &tm_w, &full[s], cb * BM, kb * BK);
              tma_load_2d_2sm(sw + 8192, &tm_w, &full[s], cb * BM + 64, kb * BK);
            }
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    // Segment bounds come from values broadcast in the preamble (mma_nseg,
    // mma_kb_first, mma_kb_last) and the segment index, so the loop, the stage
    // counter and the smem descriptors stay on the uniform datapath.
    if (leader && lane == 0) {
      constexpr uint32_t idesc_main = idesc_bf16(2 * BM, 2 * HB, MN ? 1u : 0u, 0u);
      constexpr uint32_t idesc_kmaj = idesc_bf16(2 * BM, 2 * HB, 0u, 0u);
      int s = 0;
      uint32_t ph = 0;
      unsigned long long t_full = 0, t_tempty = 0;
      const unsigned long long t_start = (kDevTrace && p.trace) ? clock64() : 0;
      // k16 MMAs of stage s (k-block kb) into accumulators [a0, a1]; per k16 the
      // accumulators are issued back to back so they share the A (weight) read
      auto issue = [&](int s_, int kb, int kb0, int a0, int a1) {
        const bool lora = kb >= n_kb_main;
        const int nk16 = (lora && kb == n_kb - 1) ? p.lora_k16_last : BK / 16;
        const uint32_t sw = smem_u32(sW + s_ * W_TILE);
        const uint32_t st = smem_u32(sT + s_ * T_TILE);
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
          for (int a = a0; a <= a1; ++a) {
            const uint64_t bdesc = sdesc_sw128(st + a * HB_TILE + k * 32, 16, 1024);
            tc_mma_f16_2sm(tmem_base + a * (2 * HB), adesc, bdesc, idesc,
                           (kb == kb0 && k == 0) ? 0u : 1u);
          }
        }
      };
      for (int sg = 0; sg < mma_nseg; ++sg) {
        const int kb0 = sg == 0 ? mma_kb_first : 0;
        const int kb1 = (sg == mma_nseg - 1 && mma_kb_last > 0) ? mma_kb_last : n_kb;
        // The epilogue drains accumulator 0 first and releases it early
        // (tempty): the first `pre` k-blocks' accumulator-0 MMAs of this tile
        // run while accumulator 1 is still being drained; their stages are
        // released once accumulator 1's MMAs for them follow (tempty1).
        if (one_acc) {  // (split-K only) one 256-token accumulator per tile
          mbar_wait_acq_cluster(tempty, (sg & 1) ^ 1);
          tc_fence_after();
          for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait_acq_cluster(&full[s], ph);
            tc_fence_after();
            issue(s, kb, kb0, 0, 0);
            tc_commit_2sm_mc(&empty[s], 0x3);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
          tc_commit_2sm_mc(tfull, 0x3);
          continue;
        }
        const int pre = kb1 - kb0 < STAGES ? kb1 - kb0 : STAGES;
        const unsigned long long tw0 = (kDevTrace && p.trace) ? clock64() : 0;
        mbar_wait_acq_cluster(tempty, (sg & 1) ^ 1);
        if (kDevTrace && p.trace) t_tempty += clock64() - tw0;
        tc_fence_after();
        int s0 = s;
        uint32_t ph0 = ph;
        for (int i = 0; i < pre; ++i) {
          const unsigned long long tf0 = (kDevTrace && p.trace) ? clock64() : 0;
          mbar_wait_acq_cluster(&full[s], ph);
          if (kDevTrace && p.trace) t_full += clock64() - tf0;
          tc_fence_after();
          issue(s, kb0 + i, kb0, 0, 0);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        const unsigned long long tw1 = (kDevTrace && p.trace) ? clock64() : 0;
        mbar_wait_acq_cluster(tempty1, (sg & 1) ^ 1);
        if (kDevTrace && p.trace) t_tempty += clock64() - tw1;
        tc_fence_after();
        for (int i = 0; i < pre; ++i) {
          issue(s0, kb0 + i, kb0, 1, 1);
          tc_commit_2sm_mc(&empty[s0], 0x3);
          if (++s0 == STAGES) {
            s0 = 0;
            ph0 ^= 1;
          }
        }
        (void)ph0;
        for (int kb = kb0 + pre; kb < kb1; ++kb) {
          const unsigned long long tf0 = (kDevTrace && p.trace) ? clock64() : 0;
          mbar_wait_acq_cluster(&full[s], ph);
          if (kDevTrace && p.trace) t_full += clock64() - tf0;
          tc_fence_after();
          issue(s, kb, kb0, 0, 1);
          tc_commit_2sm_mc(&empty[s], 0x3);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit_2sm_mc(tfull, 0x3);
      }
      if (tl) tl[1] = gtime();
      if (kDevTrace && p.trace) {  // dev-only instrumentation (MLRA_TRACE)
        p.trace[4 * cid + 0] = clock64() - t_start;
        p.trace[4 * cid + 1] = t_full;
        p.trace[4 * cid + 2] = t_tempty;
        p.trace[4 * cid + 3] = static_cast<unsigned long long>(mma_nseg);
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ Q-ring TMA (both CTAs, local)
    if (QTMA && !W_TMA && lane == 0) {
      const uint32_t qbytes = p.q_codes_bytes + p.q_grid_bytes;
      int qs = 0;
      uint32_t qph = 0;
      SegSched<SK> sc = sched;
      int tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        const int mp = tile % m_pairs;
        const int cb = mp * 2 + static_cast<int>(rank);
        const int pr_end = (kb1 < n_kb_main ? kb1 : n_kb_main) / 2;
        for (int pr = kb0 / 2; pr < pr_end; ++pr) {
          mbar_wait_backoff<PROD_NS>(&qempty[qs], qph ^ 1);
          mbar_arrive_expect_tx(&qfull[qs], qbytes);
          uint8_t* dst = sQ + qs * p.q_stage_bytes;
          if (!MN) {
            tma_load_2d(dst, &tm_codes, &qfull[qs], pr * 16 * QB, cb * BM);
            tma_load_2d(dst + p.q_codes_bytes, &tm_grid, &qfull[qs],
                        2 * (pair_group(pr, p) & ~1), cb * BM);
          } else {
            tma_load_2d(dst, &tm_codes, &qfull[qs], cb * 16 * QB, pr * 128);
            tma_load_2d(dst + p.q_codes_bytes, &tm_grid, &qfull[qs],
                        2 * (pair_group(cb, p) & ~1), pr * 128);
          }
          if (++qs == p.q_stages) {
            qs = 0;
            qph ^= 1;
          }
        }
      }
    }
  } else if (warp >= EPI_WARP0 && warp < DQ_WARP0) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int qd = warp & 3;
    const uint32_t tempty_leader = mapa(smem_u32(tempty), 0);
    const uint32_t tempty1_leader = mapa(smem_u32(tempty1), 0);
    int local = 0;
    SegSched<SK> sc = sched;
    int tile, kb0, kb1;
    // split-K: every warp of the CTA runs the fix-up after its role (below)
    for (; !(SK && p.split > 0) && sc.next(tile, kb0, kb1); ++local) {
      if (own_last && sc.count() == 0 && own_count() > 0) break;  // -> sk_owner_fixup
      const int mp = tile % m_pairs, np = tile / m_pairs;
      // stream-K roles: a segment starting mid-tile writes a partial; one that
      // starts at k-block 0 but ends early adds pairs [cid+1, q_end)'s partials
      const bool contrib = SK && kb0 != 0;
      constexpr bool split = false;  // split-K runs in split_fixup (all warps)
      const int q_end = (SK && !split && !contrib && kb1 != n_kb) ? sc.contrib_end(p, cid, tile)
                                                            : cid + 1;
      const int r_in = qd * 32 + lane;
      mbar_wait_backoff<EPI_NS>(tfull, local & 1);
      tc_fence_after();
      if (tl && qd == 0 && lane == 0) tl[2] = gtime();
      const int64_t wrow = static_cast<int64_t>(mp) * PAIR_ROWS + rank * BM + r_in;
      const bool row_ok = wrow < p.m_valid;
      const float bias = (p.bias != nullptr && row_ok) ? p.bias[wrow] : 0.0f;
      for (int q = cid + 1; q < q_end; ++q)
        while (ld_acquire_gpu(&p.sk_flags[2 * q + rank]) == 0) __nanosleep(128);
      if (tl && qd == 0 && lane == 0) tl[3] = gtime();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(qd * 32) << 16);
      const int64_t tbase = static_cast<int64_t>(np) * PAIR_TOK;
      const float bias_nb = __shfl_xor_sync(0xffffffffu, bias, 1);
      const bool odd = lane & 1;
      const bool pairs = p.out_pairs && __all_sync(0xffffffffu, (wrow | 1) < p.m_valid);
      auto store_chunk = [&](const uint32_t(&r)[32], int cc) {
        epi_store<OUT_F32>(p, r, tbase + cc * 32, wrow, row_ok, bias, bias_nb, pairs, odd);
      };
      // stream-K partial slots of this CTA's rows: [512 tokens][128 rows] fp32
      auto slot_of = [&](int q, int cc) {
        return p.sk_ws + (2 * static_cast<int64_t>(q) + rank) * (PAIR_TOK * BM) +
               static_cast<int64_t>(cc * 32) * BM + r_in;
      };
      // Drains the 16 chunks of 32 TMEM columns = tokens [np*512 + 32cc, +32)
      // (acc0 then acc1). TMEM loads are double-buffered so their latency hides
      // under the previous chunk's stores; TMEM is released right after the last
      // load completes.
      auto drain = [&](auto&& handle) {
        uint32_t ra[32], rb[32];
        tmem_ld_32x32b_x32(taddr, ra);
        tc_wait_ld();
#pragma unroll 1
        for (int cc = 0; cc < 16; cc += 2) {
          tmem_ld_32x32b_x32(taddr + (cc + 1) * 32, rb);
          handle(ra, cc);
          tc_wait_ld();
          if (cc + 1 == 7) {
            tc_fence_before();  // accumulator 0 (chunks 0..7) fully read
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty_leader);
          }
          if (cc + 2 < 16) {
            tmem_ld_32x32b_x32(taddr + (cc + 2) * 32, ra);
          } else {
            tc_fence_before();  // all TMEM reads of this tile are complete
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty1_leader);
          }
          handle(rb, cc + 1);
          if (cc + 2 < 16) tc_wait_ld();
        }
      };
      if (contrib) {
        drain([&](uint32_t(&r)[32], int cc) {
          if (!row_ok) return;
          float* d = slot_of(cid, cc);
#pragma unroll
          for (int j = 0; j < 32; ++j) d[j * BM] = __uint_as_float(r[j]);
        });
        __threadfence();  // publish this CTA's partial to the tile's owner
        epi_bar_sync();
        if (qd == 0 && lane == 0) st_release_gpu(&p.sk_flags[2 * cid + rank], 1u);
      } else if (q_end > cid + 1 && q_end - cid - 1 <= kFixSlots && sc.count() == 0) {
        // Stream-K owner of its range's last segment: the operand ring is idle
        // (every MMA of this CTA has completed), so the contributors' partial
        // chunks (16 KB each: 32 tokens x 128 rows fp32, contiguous) are staged
        // into it by bulk copies, D chunks ahead of the drain, and added from
        // shared memory in pair order. (Loading them straight from L2 in the
        // drain cost one L2 round trip per (chunk, contributor): ~35 us of fix-up
        // per launch at cfg1, scripts/timeline.py.)
        const int nc = q_end - cid - 1;
        const int depth = kFixSlots / nc < 16 ? kFixSlots / nc : 16;
        const bool issuer = qd == 0 && lane == 0;
        const uint32_t ring = smem_u32(smem);
        auto issue = [&](int cc) {
          for (int i = 0; i < nc; ++i) {
            const int jb = cc * nc + i, slot = jb % kFixSlots;
            mbar_arrive_expect_tx(&fixb[slot], kFixChunkBytes);
            bulk_g2s(ring + slot * kFixChunkBytes, slot_of(cid + 1 + i, cc) - r_in,
                     kFixChunkBytes, &fixb[slot]);
          }
        };
        if (issuer) {
          fence_proxy_async_global();  // acquired partials (generic writes) -> async-proxy reads
          for (int cc = 0; cc < depth; ++cc) issue(cc);
        }
        drain([&](uint32_t(&r)[32], int cc) {
          for (int i = 0; i < nc; ++i) {  // pair order: deterministic sums
            const int jb = cc * nc + i, slot = jb % kFixSlots;
            mbar_wait(&fixb[slot], static_cast<uint32_t>(jb / kFixSlots) & 1u);
            const float* src = reinterpret_cast<const float*>(smem + slot * kFixChunkBytes) + r_in;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              r[j] = __float_as_uint(__uint_as_float(r[j]) + src[j * BM]);
          }
          store_chunk(r, cc);
          epi_bar_sync();  // every epilogue thread is done with chunk cc's slots
          if (issuer && cc + depth < 16) issue(cc + depth);
        });
      } else if (q_end > cid + 1) {
        drain([&](uint32_t(&r)[32], int cc) {
          if (!row_ok) return;
          for (int q = cid + 1; q < q_end; ++q) {  // pair order: deterministic sums
            const float* src = slot_of(q, cc);
#pragma unroll
            for (int j = 0; j < 32; ++j)
              r[j] = __float_as_uint(__uint_as_float(r[j]) + src[j * BM]);
          }
          store_chunk(r, cc);
        });
      } else {
        drain([&](uint32_t(&r)[32], int cc) { store_chunk(r, cc); });
      }
      if (tl && qd == 0 && lane == 0) tl[4] = gtime();
    }
  } else if (warp >= DQ_WARP0) {
    // ------------------------------------------------------------ dequant producers (both CTAs)
    const int grp = (warp - DQ_WARP0) >> 2;
    const int gtid = threadIdx.x - (DQ_WARP0 + 4 * grp) * 32;  // 0..127
    const uint32_t full_leader0 = mapa(smem_u32(full), 0);
    int s = 0;
    uint32_t ph = 0;
    if constexpr (W_TMA) {
      SegSched<SK> sc = sched;
      int tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        (void)tile;
        for (int kb = kb0; kb < kb1; ++kb) {
          if ((s & 1) == grp) {
            mbar_wait(&empty[s], ph ^ 1);
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(full_leader0 + 8 * s);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    } else if constexpr (QTMA) {
      constexpr int UPT = UNITS_PER_GROUP_THREAD;
      uint32_t soff[UPT];
#pragma unroll
      for (int i = 0; i < UPT; ++i) soff[i] = unit_soff<MN>(i * 128 + gtid);
      const int k8 = MN ? (gtid & 15) : (gtid & 7);
      const int row0 = MN ? (gtid >> 4) : (gtid >> 3);
      constexpr int ROW_STEP = MN ? 8 : 16;
      const int gshift = p.q_group_shift;
      const int gbox = p.q_grid_bytes / BM;
      const uint32_t sQ32 = smem_u32(sQ), sW32 = smem_u32(sW);
      int qs = 0;
      uint32_t qph = 0;
      SegSched<SK> sc = sched;
      int tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        const int mp = tile % m_pairs;
        const int cb = mp * 2 + static_cast<int>(rank);
        const int gpar_mn = pair_group(cb, p) & 1;
        for (int kb = kb0; kb < kb1; ++kb) {
          const bool main = kb < n_kb_main;
          const int kp = kb & 1;
          if ((s & 1) == grp) {
            if (main) mbar_wait(&qfull[qs], qph);
            mbar_wait(&empty[s], ph ^ 1);
            if (main) {
              const uint32_t qc = sQ32 + qs * p.q_stage_bytes;
              const uint32_t qg = qc + p.q_codes_bytes;
              const uint32_t st = sW32 + s * W_TILE;
              const int unit = MN ? k8 : (k8 + 8 * kp);
              const int code = unit * 8;
              const int gsub = gshift >= 0 ? (code >> gshift)
                                           : (MN ? gpar_mn : (pair_group(kb >> 1, p) & 1));
              const int rbase = MN ? (row0 + 64 * kp) : row0;
              if constexpr (CB2)
                dequant_units_cb2<UPT, ROW_STEP>(qc, qg, st, soff, unit, gsub, rbase, gbox,
                                                 smem_u32(sCb));
              else if constexpr (E8P)
                dequant_units_e8p<UPT, ROW_STEP>(qc, qg, st, soff, unit, gsub, rbase, gbox,
                                                 smem_u32(sCb));
              else if constexpr (LUT)
                dequant_units_lut<QB, UPT, ROW_STEP>(qc, qg, st, soff, unit, gsub, rbase, gbox,
                                                     smem_u32(sCb));
              else
                dequant_units<BITS, UPT, ROW_STEP>(qc, qg, st, soff, unit, gsub, rbase, gbox);
              fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) {
              mbar_arrive_cluster(full_leader0 + 8 * s);
              if (main) mbar_arrive(&qempty[qs]);
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
      SegSched<SK> sc = sched;
      int tile, kb0, kb1;
      while (sc.next(tile, kb0, kb1)) {
        const int mp = tile % m_pairs;
        const int cb = mp * 2 + static_cast<int>(rank);
        for (int kb = kb0; kb < kb1; ++kb) {
          if ((s & 1) == grp) {
            mbar_wait(&empty[s], ph ^ 1);
            if (kb < n_kb_main) {
              uint8_t* stile = sW + s * W_TILE;
#pragma unroll 2
              for (int i = 0; i < UNITS_PER_GROUP_THREAD; ++i) {
                const int u = i * 128 + gtid;
                int64_t wrow, wunit;
                if constexpr (!MN) {
                  wrow = static_cast<int64_t>(cb) * BM + (u >> 3);
                  wunit = static_cast<int64_t>(kb) * (BK / 8) + (u & 7);
                } else {
                  wrow = static_cast<int64_t>(kb) * BK + (u >> 4);
                  wunit = static_cast<int64_t>(cb) * (BM / 8) + (u & 15);
                }
                if constexpr (!CB2 && !E8P && !LUT) {  // (the plugin decodes always run on the Q ring)
                  const uint64_t v = load_unit<BITS>(q.words + wrow * q.row_words, wunit);
                  *reinterpret_cast<uint4*>(stile + unit_soff<MN>(u)) =
                      deq8_bf16_general<BITS>(v, q.grid + wrow * q.ng_pad, wunit * 8, q.group);
                }
              }
              fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(full_leader0 + 8 * s);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  }

  if constexpr (SK) {
    if (p.split > 0) {
      __syncwarp();
      split_fixup<OUT_F32>(p, cid, rank, m_pairs, tmem_base, tfull, fixb, smem, tl);
    } else if (own_last) {
      __syncwarp();
      const int own_nc = own_count();
      if (own_nc > 0)
        sk_owner_fixup<OUT_F32>(p, cid, rank, m_pairs, sched.t_end, own_nc,
                                static_cast<uint32_t>(sched.count() - 1) & 1u, tmem_base, tfull,
                                fixb, smem, tl);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) tmem_dealloc2(tmem_base, TMEM_COLS);
}

inline int sm_total() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

template <int BITS, bool W_TMA, bool MN, bool OUT_F32, bool QTMA, bool SK>
cudaError_t launch2_t(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                      cudaStream_t stream) {
  auto kern = qgemm2_kernel<BITS, W_TMA, MN, OUT_F32, QTMA, SK>;
  const int smem = SMEM_FIXED + p.q_stages * p.q_stage_bytes +
                   (BITS == kCb2Bits ? kCb2SmemBytes
                                     : (BITS == kE8pBits ? kE8pSmemBytes
                                                         : (is_lut<BITS>() ? kLutSmemBytes : 0)));
  static int smem_set = 0;  // per instantiation: the opt-in only ever grows
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  const int64_t tiles = (p.m_total / PAIR_ROWS) * ((p.tokens + PAIR_TOK - 1) / PAIR_TOK);
  const int64_t pairs = p.sk_pairs ? p.sk_pairs : (tiles < sm_total() / 2 ? tiles : sm_total() / 2);
  return launch_pdl(kern, dim3(static_cast<unsigned>(2 * pairs)), dim3(NUM_THREADS), smem, stream,
                    p.no_pdl == 0,
                    maps.act, maps.act_lora, maps.w, maps.w_lora, maps.codes, maps.grid, q, p);
}

template <bool MN, bool SK, int BITS, bool W_TMA, bool QTMA>
cudaError_t launch2_o(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool out_f32,
                      cudaStream_t st) {
  return out_f32 ? launch2_t<BITS, W_TMA, MN, true, QTMA, SK>(maps, q, p, st)
                 : launch2_t<BITS, W_TMA, MN, false, QTMA, SK>(maps, q, p, st);
}

// One (direction, schedule) family of the pair kernel: instantiated by exactly
// one of qgemm2_{f,d}{0,1}.cu, so the families compile in parallel.
template <bool MN, bool SK>
cudaError_t dispatch2(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool w_tma,
                      bool out_f32, cudaStream_t stream) {
  if (w_tma) return launch2_o<MN, SK, 4, true, false>(maps, q, p, out_f32, stream);
  const bool qtma = p.q_stages > 0;
  if (p.cb2_codebook != nullptr && p.e8p) {
    if (!qtma) return cudaErrorInvalidValue;  // the fused e8p decode needs the Q ring
    return launch2_o<MN, SK, kE8pBits, false, true>(maps, q, p, out_f32, stream);
  }
  if (p.cb2_codebook != nullptr) {
    if (!qtma) return cudaErrorInvalidValue;  // the fused cb2 decode needs the Q ring
    return launch2_o<MN, SK, kCb2Bits, false, true>(maps, q, p, out_f32, stream);
  }
  if (p.lut != nullptr) {
    if (!qtma) return cudaErrorInvalidValue;  // so does the lut decode
    switch (q.bits) {
      case 2: return launch2_o<MN, SK, kLutTag + 2, false, true>(maps, q, p, out_f32, stream);
      case 3: return launch2_o<MN, SK, kLutTag + 3, false, true>(maps, q, p, out_f32, stream);
      case 4: return launch2_o<MN, SK, kLutTag + 4, false, true>(maps, q, p, out_f32, stream);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (q.bits) {
    case 2: return qtma ? launch2_o<MN, SK, 2, false, true>(maps, q, p, out_f32, stream)
                        : launch2_o<MN, SK, 2, false, false>(maps, q, p, out_f32, stream);
    case 3: return qtma ? launch2_o<MN, SK, 3, false, true>(maps, q, p, out_f32, stream)
                        : launch2_o<MN, SK, 3, false, false>(maps, q, p, out_f32, stream);
    case 4: return qtma ? launch2_o<MN, SK, 4, false, true>(maps, q, p, out_f32, stream)
                        : launch2_o<MN, SK, 4, false, false>(maps, q, p, out_f32, stream);
    case 8: return launch2_o<MN, SK, 8, false, false>(maps, q, p, out_f32, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

}  // namespace mlra

// thin_mma.cu — K4/K5/K6 on tensor cores: the skinny rank-r adapter products.
//
//  k_rowmma (K4, K5a): out[t, j] = Σ_k act[t,k]·W[k,j]   (m x r; reduction over d)
//     XB  = X·B   — matmul(t, x, B)               lora.cpp:68
//     dYA = dY·A  — d(xb) = dab·A                  autodiff.cpp:150-152 on lora.cpp:69
//  k_colmma (K5b, K6): out[n, j] += s·Σ_t act[t,n]·V[t,j]  (d x r; reduction over tokens)
//     dA = s·dYᵀ·XB   — d(Aᵀ) = xbᵀ·dab, transposed   autodiff.cpp:153-155, :315-320
//     dB = s·Xᵀ·dYA   — dB = xᵀ·d(xb)                  autodiff.cpp:153-155
//     dbias = Σ_t dY  — bias_add backward (a ones column of V)  autodiff.cpp:183-191
//
// These are HBM-bound (r flop/B): each CTA streams 64 x 64 activation chunks
// through a TMA ring and runs bf16 mma.sync m16n8k16 against the rank-r factor. The fp32 factor is split into bf16 hi + lo parts (two MMAs),
// so the product keeps ~16 mantissa bits (fp32-grade
// intermediates); activations are exact bf16.
//
// Deterministic reduction: a CTA leaving an output tile writes its fp32 partial
// to its own slot; the last contributor of the tile (per-tile counter) sums the
// contributors' slots in CTA order and stores the result. No atomics touch the
// outputs, so XB, dYA, dA, dB and dbias are bitwise reproducible run to run, as
// the reference's fixed-order loops are (matrix.cpp:81-97, test_train.cpp:328-387),
// and the outputs need no zero-fill. The finisher also writes the derived
// operands the next kernels consume (bf16(s·XB) / bf16(s·dYA) padded extra-K
// operands of the GEMM, the transposed hi/lo planes of dYA for dB), so a layer
// pass needs no conversion launch between the skinny product and the GEMM.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"
#include "ptx.cuh"

namespace mlra {

namespace {

constexpr int TILE = 64;      // rows (tokens or n) per unit, and reduction chunk
#ifdef MLRA_DEV_TRACE
constexpr bool kThinTrace = true;
#else
constexpr bool kThinTrace = false;
#endif
// dev timeline (MLRA_TRACE3): per CTA [0] entry, [1] first unit landed (k_rowmma_cl: PDL
// wait passed), [2] last unit's MMAs done (k_rowmma_cl: main loop done), [3] exit,
// [4] 1 if this CTA finished a tile, [5] finisher start
__device__ __forceinline__ void thin_stamp(const ThinOut& o, int k) {
  if (kThinTrace && o.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    o.trace[8 * blockIdx.x + k] = t;
  }
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Work decomposition (both kernels): the (output tile x reduction chunk) space
// is flattened tile-major into U units of TM x 64 activations and cut into
// gridDim.x equal contiguous ranges — one resident wave, every CTA streaming
// the same number of chunks through one continuous pipeline. A CTA flushes its
// fp32 partials to its slot whenever its range leaves an output tile; the
// tile's last contributor finishes it (thin_flush).
//
// Operand staging is TMA (cp.async.bulk.tensor, SWIZZLE_128B): one elected
// thread issues the activation chunk and the hi+lo factor chunk per unit into
// an NS-deep ring signalled by mbarrier complete_tx, so the warps spend their
// issue slots on ldmatrix + mma only. Reads use the 128-B swizzle: 16-B chunk
// c of row r sits at r*128 + ((c ^ (r & 7)) << 4).

#ifndef MLRA_THIN_NS
#define MLRA_THIN_NS 3
#endif
constexpr int TNS = MLRA_THIN_NS;  // TMA ring depth (units in flight per CTA)

#ifndef MLRA_THIN_WARPS
#define MLRA_THIN_WARPS 8
#endif
constexpr int TW = MLRA_THIN_WARPS;   // warps per CTA; each owns 16 output rows of a unit
constexpr int TM = 16 * TW;           // output-tile rows per unit (tokens or n)
constexpr int TTHREADS = 32 * TW;

template <int NT, int NS = TNS>
struct ThinSmem {
  static constexpr int ROWS = 8 * NT;
  static constexpr int ACT = TM * 128;          // TM x 64 bf16
  static constexpr int FAC = 2 * ROWS * 128;    // hi + lo planes, 64 columns
  static constexpr int STAGE = ACT + FAC;       // multiple of 1024 when NT is even
  static constexpr int STAGE_AL = (STAGE + 1023) / 1024 * 1024;
  static constexpr int BYTES = 1024 + NS * STAGE_AL + 8 * NS;  // + alignment slack + barriers
};

__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + row * 128 + ((chunk ^ (row & 7)) << 4);
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// CTA whose contiguous unit range [u0(c), u0(c+1)) contains unit u, for
// u0(c) = floor(c·U/G): the largest c with c·U/G < u + 1.
__device__ __forceinline__ int cta_of_unit(int64_t u, int64_t units, int64_t G) {
  return static_cast<int>(((u + 1) * G - 1) / units);
}
__device__ __forceinline__ int first_tile_of(int c, int64_t units, int64_t G, int chunks) {
  return static_cast<int>(c * units / G) / chunks;
}

// The finished value of 4 consecutive columns [j, j+4) of output row `row`:
// out = scale·v, colsum (the ones column), the GEMM's padded bf16(pad_scale·v)
// operand and the transposed hi/lo planes (zero beyond n_out up to ldt).
__device__ __forceinline__ void thin_store4(const ThinOut& o, int64_t row, int j,
                                            const float (&vv)[4], int64_t n_out, bool vec_out,
                                            bool vec_pad) {
  if (row < n_out) {
    if (vec_out && j + 4 <= o.rc) {
      *reinterpret_cast<float4*>(o.out + row * o.ldo + j) =
          make_float4(o.scale * vv[0], o.scale * vv[1], o.scale * vv[2], o.scale * vv[3]);
    } else {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        if (j + kk < o.rc) o.out[row * o.ldo + j + kk] = o.scale * vv[kk];
    }
    if (o.colsum && j <= o.rc && o.rc < j + 4) o.colsum[row] = vv[o.rc - j];
    if (o.pad) {  // bf16(pad_scale · v), zero beyond rc (the padded extra-K operand)
      __nv_bfloat16 h[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        h[kk] = __float2bfloat16_rn(j + kk < o.rc ? o.pad_scale * vv[kk] : 0.0f);
      if (vec_pad && j + 4 <= o.pad_cols) {
        *reinterpret_cast<uint2*>(o.pad + row * o.ldp + j) = *reinterpret_cast<const uint2*>(h);
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (j + kk < o.pad_cols) o.pad[row * o.ldp + j + kk] = h[kk];
      }
    }
  }
  if (o.thi && row < o.ldt) {  // transposed hi/lo planes [t_rows x ldt] (zero padded)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      if (j + kk < o.t_rows) {
        const float tv = (row < n_out && j + kk < o.rc) ? vv[kk] : 0.0f;
        const __nv_bfloat16 h = __float2bfloat16_rn(tv);
        o.thi[static_cast<int64_t>(j + kk) * o.ldt + row] = h;
        o.thi[static_cast<int64_t>(o.t_rows + j + kk) * o.ldt + row] =
            __float2bfloat16_rn(tv - __bfloat162float(h));
      }
    }
  }
}

// Zero pad columns [ROWS, pad_cols) of rows [row0, row0 + nrows) (8-B stores).
template <int ROWS>
__device__ __forceinline__ void thin_pad_zero(const ThinOut& o, int64_t row0, int nrows,
                                              int64_t n_out, bool vec_pad) {
  if (!o.pad || o.pad_cols <= ROWS) return;
  const int pc4 = (o.pad_cols - ROWS) / 4;
  for (int idx = threadIdx.x; idx < nrows * pc4; idx += TTHREADS) {
    const int tr = idx / pc4, j = ROWS + 4 * (idx - tr * pc4);
    const int64_t row = row0 + tr;
    if (row < n_out) {
      if (vec_pad)
        *reinterpret_cast<uint2*>(o.pad + row * o.ldp + j) = make_uint2(0u, 0u);
      else
        for (int kk = 0; kk < 4; ++kk) o.pad[row * o.ldp + j + kk] = __float2bfloat16_rn(0.0f);
    }
  }
}

// Flush of one output tile (all threads of the CTA, uniform): the fragment
// partials go to this CTA's slot (slot 0 when `tile` is the first tile of its
// range, else slot 1; row-major [TM rows][ROWS cols], the output's own order);
// when every contributor has written (counter), the last one sums the slots in
// CTA order and stores.
// Lock-free on purpose: no CTA ever waits for another (a spin-waiting
// reduction deadlocks when two such grids are co-scheduled on different
// streams and each holds the SMs the other's unscheduled CTAs need); the
// launcher caps the contributors per tile instead (kMinUnitsPerCta).
template <int NT>
__device__ void thin_flush(float (&acc)[NT][4], int tile, int chunks, int units,
                           const ThinOut& o, int64_t n_out) {
  constexpr int ROWS = 8 * NT;
  constexpr int SLOT = TM * ROWS;
  __shared__ int s_last;
  const int G = gridDim.x, c = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int which = tile == first_tile_of(c, units, G, chunks) ? 0 : 1;
  float* slot = o.ws + (static_cast<int64_t>(c) * 2 + which) * SLOT;
  const int ra = warp * 16 + g;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int j = n * 8 + 2 * tq;
    *reinterpret_cast<float2*>(slot + ra * ROWS + j) = make_float2(acc[n][0], acc[n][1]);
    *reinterpret_cast<float2*>(slot + (ra + 8) * ROWS + j) = make_float2(acc[n][2], acc[n][3]);
    acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  }
  const int c_lo = cta_of_unit(static_cast<int64_t>(tile) * chunks, units, G);
  const int c_hi = cta_of_unit(static_cast<int64_t>(tile + 1) * chunks - 1, units, G);
  // bar.sync orders the CTA's slot stores before thread 0's acq_rel atomic (a
  // cumulative gpu-scope release); the finisher's thread 0 acquires every other
  // contributor's release through the same counter and the second bar.sync
  // passes that on to its threads, whose L2 (.cg) loads then see the slots.
  // (A per-thread __threadfence() here is a fence.sc per thread: measured
  // ~3x slower for the whole kernel.)
  __syncthreads();
  if (c_lo != c_hi) {
    if (threadIdx.x == 0) {
      const int old = atom_add_acq_rel_gpu(o.cnt + tile, 1);
      s_last = old == c_hi - c_lo;
      if (s_last) o.cnt[tile] = 0;  // self-resetting for the next launch on this stream
    }
    __syncthreads();
    if (!s_last) return;
  }
  thin_stamp(o, 5);
  if (kThinTrace && o.trace && threadIdx.x == 0) o.trace[8 * blockIdx.x + 4] = 1;
  // Finisher: v(row, j) = Σ_{q = c_lo..c_hi} slot_q(row, j), in CTA order. Every
  // contributor after c_lo starts its range inside this tile, so its slot is 0;
  // c_lo's is 0 only when the tile is its first. The finisher is the launch's
  // tail, so it is built for memory-level parallelism and coalescing: each
  // thread owns PER float4s = 4 consecutive columns of one row, keeps QB·PER
  // loads in flight, and stores row-major (16-B fp32 / 8-B bf16 stores; measured:
  // scattered 4-B stores made the tail ~10 us of a 28 us launch).
  constexpr int C4 = ROWS / 4;                  // float4s per slot row
  constexpr int PER = SLOT / (4 * TTHREADS);    // float4 positions per thread (= NT)
  static_assert(SLOT % (4 * TTHREADS) == 0, "slot must tile the CTA in float4s");
  constexpr int QB = 8 / PER > 0 ? 8 / PER : 1;
  const float* s0 = o.ws + (static_cast<int64_t>(c_lo) * 2 +
                            (tile == first_tile_of(c_lo, units, G, chunks) ? 0 : 1)) * SLOT;
  float4 acc4[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k)
    acc4[k] = __ldcg(reinterpret_cast<const float4*>(s0) + threadIdx.x + k * TTHREADS);
  for (int q0 = c_lo + 1; q0 <= c_hi; q0 += QB) {
    float4 buf[QB][PER];
#pragma unroll
    for (int i = 0; i < QB; ++i) {
      if (q0 + i <= c_hi) {
        const float4* p = reinterpret_cast<const float4*>(o.ws + static_cast<int64_t>(q0 + i) * 2 * SLOT);
#pragma unroll
        for (int k = 0; k < PER; ++k) buf[i][k] = __ldcg(p + threadIdx.x + k * TTHREADS);
      }
    }
#pragma unroll
    for (int i = 0; i < QB; ++i) {
      if (q0 + i <= c_hi) {
#pragma unroll
        for (int k = 0; k < PER; ++k) {
          acc4[k].x += buf[i][k].x;
          acc4[k].y += buf[i][k].y;
          acc4[k].z += buf[i][k].z;
          acc4[k].w += buf[i][k].w;
        }
      }
    }
  }
  const bool vec_out = (o.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(o.out) & 15) == 0;
  const bool vec_pad = o.pad && (o.ldp & 3) == 0 && (reinterpret_cast<uintptr_t>(o.pad) & 7) == 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int p4 = threadIdx.x + k * TTHREADS;
    const int tr = p4 / C4, j = 4 * (p4 - tr * C4);
    const float vv[4] = {acc4[k].x, acc4[k].y, acc4[k].z, acc4[k].w};
    thin_store4(o, static_cast<int64_t>(tile) * TM + tr, j, vv, n_out, vec_out, vec_pad);
  }
  thin_pad_zero<ROWS>(o, static_cast<int64_t>(tile) * TM, TM, n_out, vec_pad);
  __syncthreads();  // the slot is rewritten by this CTA's next flush
}

// out[t, j] (+)= Σ_k act[t, k] · Wt[j, k]   (Wt = W transposed, hi/lo bf16 planes)
template <int NT>
__global__ void __launch_bounds__(TTHREADS, 3)
    k_rowmma(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap fac_map,
             int64_t m, int kchunks, int units, const ThinOut o) {
  using L = ThinSmem<NT>;
  constexpr int ROWS = L::ROWS;
  extern __shared__ __align__(16) unsigned char thin_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(thin_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + TNS * L::STAGE_AL);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  thin_stamp(o, 0);
  const int u0 = static_cast<int>(static_cast<int64_t>(blockIdx.x) * units / gridDim.x);
  const int u1 = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * units / gridDim.x);
  auto issue = [&](int u, int slot) {
    const int tile = u / kchunks, ch = u - tile * kchunks;
    unsigned char* st = sm + slot * L::STAGE_AL;
    mbar_arrive_expect_tx(&full[slot], L::STAGE);
    tma_load_2d(st, &act_map, &full[slot], ch * TILE, tile * TM);
    tma_load_2d(st + L::ACT, &fac_map, &full[slot], ch * TILE, 0);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < TNS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    tma_prefetch_desc(&act_map);
    tma_prefetch_desc(&fac_map);
  }
  pdl_trigger();
  pdl_wait();  // activations / factor planes / counters come from earlier kernels
  if (threadIdx.x == 0) {
    for (int c = 0; c < TNS - 1; ++c)
      if (u0 + c < u1) issue(u0 + c, c);
  }
  __syncthreads();
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  const int arow = warp * 16 + (lane & 15);
  for (int u = u0; u < u1; ++u) {
    const int i = u - u0, b = i % TNS;
    if (threadIdx.x == 0 && u + TNS - 1 < u1) {
      fence_proxy_async_smem();  // the slot's last generic reads (iteration i-1) before TMA
      issue(u + TNS - 1, (i + TNS - 1) % TNS);
    }
    mbar_wait(&full[b], static_cast<uint32_t>((i / TNS) & 1));
    if (i == 0) thin_stamp(o, 1);
    if (u + 1 == u1) thin_stamp(o, 2);
    const uint32_t abase = smem_u32(sm + b * L::STAGE_AL);
    const uint32_t fbase = abase + L::ACT;
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      uint32_t a[4];
      ldsm_x4(swz(abase, arow, k16 * 2 + (lane >> 4)), a);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int rh = n * 8 + g, rl = rh + ROWS;
        const uint32_t h0 = lds_u32(swz(fbase, rh, k16 * 2) + 4 * tq);
        const uint32_t h1 = lds_u32(swz(fbase, rh, k16 * 2 + 1) + 4 * tq);
        const uint32_t l0 = lds_u32(swz(fbase, rl, k16 * 2) + 4 * tq);
        const uint32_t l1 = lds_u32(swz(fbase, rl, k16 * 2 + 1) + 4 * tq);
        mma_bf16(acc[n], a, h0, h1);
        mma_bf16(acc[n], a, l0, l1);
      }
    }
    __syncthreads();
    const int tile = u / kchunks;
    if (u + 1 == u1 || (u + 1) / kchunks != tile)  // leaving this token tile
      thin_flush<NT>(acc, tile, kchunks, units, o, m);
  }
  thin_stamp(o, 3);
}

// Row products on clusters: out[t, j] = Σ_k act[t,k]·F[k,j] for an fp32 factor
// F [kd x r] (B for x·B, A for dY·A). The CL CTAs of a cluster split one
// 128-token tile's reduction (kd / 64 chunks) into equal contiguous ranges and
// reduce their fp32 partials through distributed shared memory: CTA s sums rows
// [s·TM/CL, (s+1)·TM/CL) of the tile over the cluster's slabs in rank order
// (deterministic) and finishes them (thin_store4). No global partial slots,
// counters or finisher round trips, and no CTA waits for one outside its own
// co-scheduled cluster. CL = 8 when the token tiles x 8 fill the SMs, else 16.
//
// The factor is converted in the kernel: each unit's 64 x r fp32 chunk is
// loaded (L2-resident: every tile's CTAs read the same F) one unit ahead and
// split into the bf16 hi/lo planes of the stage, so no prep launch stands
// between the previous kernel and this one. `post` carries the pass's other
// small jobs (the GEMM's padded LoRA operand, its stream-K flags), run by the
// whole grid after the PDL wait while the first activation tiles load.
#ifndef MLRA_THIN_CL_NS
#define MLRA_THIN_CL_NS 3
#endif
constexpr int kClNS = MLRA_THIN_CL_NS;  // TMA ring depth of the cluster kernel

__device__ __forceinline__ void run_prep_task(const PrepTask& k, uint32_t j) {
  const uint32_t ldd = static_cast<uint32_t>(k.ldd);
  switch (k.kind) {
    case PrepTask::kZeroF32:
      reinterpret_cast<float*>(k.dst)[j] = 0.0f;
      break;
    case PrepTask::kZeroBf16:
      reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = __float2bfloat16_rn(0.0f);
      break;
    case PrepTask::kSplitT: {  // hi/lo planes [rows_out x ldd] of src^T (cols = r)
      const uint32_t row = j / ldd, col = j - row * ldd;
      float v = 0.0f;
      if (col < k.rows) {
        if (row < k.cols)
          v = k.src[static_cast<int64_t>(col) * k.lds + row];
        else if (row == k.cols && k.ones)
          v = 1.0f;
      }
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = h;
      reinterpret_cast<__nv_bfloat16*>(k.dst2)[j] = __float2bfloat16_rn(v - __bfloat162float(h));
      break;
    }
    case PrepTask::kPadBf16: {  // dst [rows_out x ldd] = bf16(scale * src) zero-padded
      const uint32_t row = j / ldd, col = j - row * ldd;
      const float v = (row < k.rows && col < k.cols)
                          ? k.scale * k.src[static_cast<int64_t>(row) * k.lds + col]
                          : 0.0f;
      reinterpret_cast<__nv_bfloat16*>(k.dst)[j] = __float2bfloat16_rn(v);
      break;
    }
  }
}

// A task's index space [0, count) strided over the caller's threads (first j0,
// stride). kPadBf16 with 16-B aligned rows runs 8 outputs per step (one 16-B
// store; the zero padding columns need no load), so a padded LoRA factor of
// 11008 rows x 64 columns is ~3 vector steps per thread of a 128-CTA launch
// instead of ~21 load-latency-bound scalar steps (~10 us inside the fused row
// product at 1024 tokens). Same values as run_prep_task, element for element.
__device__ __forceinline__ void run_prep_span(const PrepTask& k, uint32_t count, uint32_t j0,
                                              uint32_t stride) {
  if (k.kind == PrepTask::kPadBf16 && (k.ldd & 7) == 0 &&
      (reinterpret_cast<uintptr_t>(k.dst) & 15) == 0) {
    const uint32_t upr = static_cast<uint32_t>(k.ldd) >> 3, units = count >> 3;
    for (uint32_t u = j0; u < units; u += stride) {
      const uint32_t row = u / upr, c0 = (u - row * upr) * 8;
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      if (row < k.rows && c0 < k.cols) {
        const float* src = k.src + static_cast<int64_t>(row) * k.lds + c0;
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = c0 + i < k.cols ? k.scale * src[i] : 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __nv_bfloat16 lo = __float2bfloat16_rn(v[2 * i]);
          const __nv_bfloat16 hi = __float2bfloat16_rn(v[2 * i + 1]);
          w[i] = static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&lo)) |
                 (static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&hi)) << 16);
        }
      }
      *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(k.dst) + static_cast<size_t>(u) * 8) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
  for (uint32_t j = j0; j < count; j += stride) run_prep_task(k, j);
}

// One unit's factor chunk: rows k of F [kd x ldf] (fp32) -> the stage's bf16
// hi / lo planes [ROWS][64] (SWIZZLE_128B layout, as the TMA path stores them).
// Task (j, kq): the 8 values F[64 ch + 8 kq + i][j] — one 16-B swizzle chunk of
// row j in each plane, stored with one 16-B st.shared per plane. Consecutive
// threads take consecutive j, so each scalar load instruction of a warp reads
// consecutive floats of one F row.
template <int NT>
struct FacRegs {
  static constexpr int ROWS = 8 * NT;
  static constexpr int TASKS = 8 * ROWS;                          // (j, k-octet) pairs
  static constexpr int PER = (TASKS + TTHREADS - 1) / TTHREADS;   // per thread
  float v[PER][8];
  __device__ __forceinline__ void load(const float* F, int64_t ldf, int64_t kd, int rc, int ch,
                                       bool /*vec*/) {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int t = threadIdx.x + p * TTHREADS;
      const int j = t % ROWS, kq = t / ROWS;
      const int64_t k0 = static_cast<int64_t>(ch) * 64 + kq * 8;
      const bool ok = t < TASKS && j < rc;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[p][i] = (ok && k0 + i < kd) ? __ldg(F + (k0 + i) * ldf + j) : 0.0f;
    }
  }
  __device__ __forceinline__ void store(uint32_t fbase) const {
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int t = threadIdx.x + p * TTHREADS;
      if (t >= TASKS) break;
      const int j = t % ROWS, kq = t / ROWS;
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(v[p][2 * i]);
        const __nv_bfloat16 h1 = __float2bfloat16_rn(v[p][2 * i + 1]);
        const __nv_bfloat16 l0 = __float2bfloat16_rn(v[p][2 * i] - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(v[p][2 * i + 1] - __bfloat162float(h1));
        hi[i] = static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&h0)) |
                (static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&h1)) << 16);
        lo[i] = static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&l0)) |
                (static_cast<uint32_t>(*reinterpret_cast<const unsigned short*>(&l1)) << 16);
      }
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(swz(fbase, j, kq)), "r"(hi[0]),
                   "r"(hi[1]), "r"(hi[2]), "r"(hi[3]));
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(swz(fbase, ROWS + j, kq)),
                   "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]));
    }
  }
};

template <int NT, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(TTHREADS, 3)
    k_rowmma_cl(const __grid_constant__ CUtensorMap act_map, const float* F, int64_t ldf,
                int64_t kd, int64_t m, int kchunks, const ThinOut o, const PrepBatch post) {
  using L = ThinSmem<NT, kClNS>;
  constexpr int ROWS = L::ROWS;
  constexpr int RP = TM / CL;  // output rows finished per CTA
  static_assert(TM % CL == 0, "cluster rows");
  static_assert(TM * ROWS * 4 <= kClNS * L::STAGE_AL, "partial slab fits the ring");
  extern __shared__ __align__(16) unsigned char thin_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(thin_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kClNS * L::STAGE_AL);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int s = static_cast<int>(cluster_ctarank());
  const int tile = blockIdx.x / CL;
  const int c0 = kchunks * s / CL, c1 = kchunks * (s + 1) / CL;
  const bool vecf = (ldf & 3) == 0 && (reinterpret_cast<uintptr_t>(F) & 15) == 0;
  auto issue = [&](int ch, int slot) {
    mbar_arrive_expect_tx(&full[slot], L::ACT);
    tma_load_2d(sm + slot * L::STAGE_AL, &act_map, &full[slot], ch * TILE, tile * TM);
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < kClNS; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
    tma_prefetch_desc(&act_map);
  }
  thin_stamp(o, 0);
  pdl_trigger();
  pdl_wait();  // activations and the factor may come from earlier kernels
  thin_stamp(o, 1);
  if (threadIdx.x == 0) {
    for (int b = 0; b < kClNS - 1; ++b)
      if (c0 + b < c1) issue(c0 + b, b);
  }
  FacRegs<NT> fr;
  if (c0 < c1) {
    fr.load(F, ldf, kd, o.rc, c0, vecf);
    fr.store(smem_u32(sm) + L::ACT);
  }
  // the pass's small jobs, spread over the grid, while the first tiles load
  if (post.n > 0) {
    const uint32_t gt = blockIdx.x * TTHREADS + threadIdx.x, gs = gridDim.x * TTHREADS;
    for (int t = 0; t < post.n; ++t) {
      const uint32_t cnt = static_cast<uint32_t>(post.offs[t + 1] - post.offs[t]);
      run_prep_span(post.t[t], cnt, gt, gs);
    }
  }
  __syncthreads();
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  const int arow = warp * 16 + (lane & 15);
  for (int ch = c0; ch < c1; ++ch) {
    const int i = ch - c0, b = i % kClNS;
    if (threadIdx.x == 0 && ch + kClNS - 1 < c1) {
      fence_proxy_async_smem();  // the slot's last generic reads (iteration i-1) before TMA
      issue(ch + kClNS - 1, (i + kClNS - 1) % kClNS);
    }
    const bool more = ch + 1 < c1;
    if (more) fr.load(F, ldf, kd, o.rc, ch + 1, vecf);  // next unit's factor, in flight
    mbar_wait(&full[b], static_cast<uint32_t>((i / kClNS) & 1));
    const uint32_t abase = smem_u32(sm + b * L::STAGE_AL);
    const uint32_t fbase = abase + L::ACT;
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      uint32_t a[4];
      ldsm_x4(swz(abase, arow, k16 * 2 + (lane >> 4)), a);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int rh = n * 8 + g, rl = rh + ROWS;
        const uint32_t h0 = lds_u32(swz(fbase, rh, k16 * 2) + 4 * tq);
        const uint32_t h1 = lds_u32(swz(fbase, rh, k16 * 2 + 1) + 4 * tq);
        const uint32_t l0 = lds_u32(swz(fbase, rl, k16 * 2) + 4 * tq);
        const uint32_t l1 = lds_u32(swz(fbase, rl, k16 * 2 + 1) + 4 * tq);
        mma_bf16(acc[n], a, h0, h1);
        mma_bf16(acc[n], a, l0, l1);
      }
    }
    // the next stage's factor planes (its previous unit was consumed two
    // barriers ago); the barrier below publishes them
    if (more) fr.store(smem_u32(sm + ((i + 1) % kClNS) * L::STAGE_AL) + L::ACT);
    __syncthreads();
  }
  thin_stamp(o, 2);
  // this CTA's partial slab [TM][ROWS] fp32 in the (drained) ring
  float* slab = reinterpret_cast<float*>(sm);
  const int ra = warp * 16 + g;
#pragma unroll
  for (int n = 0; n < NT; ++n) {
    const int j = n * 8 + 2 * tq;
    *reinterpret_cast<float2*>(slab + ra * ROWS + j) = make_float2(acc[n][0], acc[n][1]);
    *reinterpret_cast<float2*>(slab + (ra + 8) * ROWS + j) = make_float2(acc[n][2], acc[n][3]);
  }
  cluster_sync();  // every slab of the cluster written (release / acquire at cluster scope)
  const bool vec_out = (o.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(o.out) & 15) == 0;
  const bool vec_pad = o.pad && (o.ldp & 3) == 0 && (reinterpret_cast<uintptr_t>(o.pad) & 7) == 0;
  constexpr int C4 = ROWS / 4;
  const uint32_t slab_u32 = smem_u32(slab);
  for (int idx = threadIdx.x; idx < RP * C4; idx += TTHREADS) {
    const int tr = s * RP + idx / C4, j = 4 * (idx % C4);
    const uint32_t off = slab_u32 + static_cast<uint32_t>((tr * ROWS + j) * 4);
    float vv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int q = 0; q < CL; ++q) {  // rank order: deterministic sums
      float x0, x1, x2, x3;
      asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                   : "r"(mapa(off, static_cast<uint32_t>(q))));
      vv[0] += x0;
      vv[1] += x1;
      vv[2] += x2;
      vv[3] += x3;
    }
    thin_store4(o, static_cast<int64_t>(tile) * TM + tr, j, vv, m, vec_out, vec_pad);
  }
  thin_pad_zero<ROWS>(o, static_cast<int64_t>(tile) * TM + s * RP, RP, m, vec_pad);
  cluster_sync();  // no CTA leaves while a peer may still read its slab
  thin_stamp(o, 3);
}

// out[n, j] += scale · Σ_t act[t, n] · Vt[j, t]   (Vt = V transposed, hi/lo bf16 planes)
// Column j == rc of the product (the ones column) goes to colsum.
template <int NT>
__global__ void __launch_bounds__(TTHREADS, 3)
    k_colmma(const __grid_constant__ CUtensorMap act_map, const __grid_constant__ CUtensorMap fac_map,
             int64_t nd, int tchunks, int units, const ThinOut o) {
  using L = ThinSmem<NT>;
  constexpr int ROWS = L::ROWS;
  extern __shared__ __align__(16) unsigned char thin_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(thin_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + TNS * L::STAGE_AL);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  thin_stamp(o, 0);
  const int u0 = static_cast<int>(static_cast<int64_t>(blockIdx.x) * units / gridDim.x);
  const int u1 = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * units / gridDim.x);
  auto issue = [&](int u, int slot) {
    const int nt = u / tchunks, ch = u - nt * tchunks;
    unsigned char* st = sm + slot * L::STAGE_AL;
    mbar_arrive_expect_tx(&full[slot], L::STAGE);
#pragma unroll
    for (int h = 0; h < TM / 64; ++h)  // [64 tokens x TM n] as 64-n boxes, 8 KB apart
      tma_load_2d(st + h * 8192, &act_map, &full[slot], nt * TM + h * 64, ch * TILE);
    tma_load_2d(st + L::ACT, &fac_map, &full[slot], ch * TILE, 0);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < TNS; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    tma_prefetch_desc(&act_map);
    tma_prefetch_desc(&fac_map);
  }
  pdl_trigger();
  pdl_wait();  // activations / factor planes / counters come from earlier kernels
  if (threadIdx.x == 0) {
    for (int c = 0; c < TNS - 1; ++c)
      if (u0 + c < u1) issue(u0 + c, c);
  }
  __syncthreads();
  float acc[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) acc[n][0] = acc[n][1] = acc[n][2] = acc[n][3] = 0.0f;
  // A fragment (M = n, K = t) from the [t][n] tile via transposed ldmatrix:
  // lane l addresses row t = (l & 7) + 8*(l >> 4) (+16 per k16), n chunk warp*2 + ((l >> 3) & 1)
  const int trow = (lane & 7) + ((lane >> 4) << 3), nchunk = warp * 2 + ((lane >> 3) & 1);
  const uint32_t nhalf = static_cast<uint32_t>(nchunk >> 3) * 8192u;  // which 64-n box
  for (int u = u0; u < u1; ++u) {
    const int i = u - u0, b = i % TNS;
    if (threadIdx.x == 0 && u + TNS - 1 < u1) {
      fence_proxy_async_smem();
      issue(u + TNS - 1, (i + TNS - 1) % TNS);
    }
    mbar_wait(&full[b], static_cast<uint32_t>((i / TNS) & 1));
    if (i == 0) thin_stamp(o, 1);
    if (u + 1 == u1) thin_stamp(o, 2);
    const uint32_t abase = smem_u32(sm + b * L::STAGE_AL);
    const uint32_t fbase = abase + L::ACT;
#pragma unroll
    for (int k16 = 0; k16 < 4; ++k16) {
      uint32_t a[4];
      ldsm_x4_t(swz(abase + nhalf, trow + 16 * k16, nchunk & 7), a);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int rh = n * 8 + g, rl = rh + ROWS;
        const uint32_t h0 = lds_u32(swz(fbase, rh, k16 * 2) + 4 * tq);
        const uint32_t h1 = lds_u32(swz(fbase, rh, k16 * 2 + 1) + 4 * tq);
        const uint32_t l0 = lds_u32(swz(fbase, rl, k16 * 2) + 4 * tq);
        const uint32_t l1 = lds_u32(swz(fbase, rl, k16 * 2 + 1) + 4 * tq);
        mma_bf16(acc[n], a, h0, h1);
        mma_bf16(acc[n], a, l0, l1);
      }
    }
    __syncthreads();
    const int nt = u / tchunks;
    if (u + 1 == u1 || (u + 1) / tchunks != nt)  // leaving this n tile
      thin_flush<NT>(acc, nt, tchunks, units, o, nd);
  }
  thin_stamp(o, 3);
}

// One launch for a layer pass's small conversion / zeroing jobs (PrepBatch):
// blocks are partitioned among the tasks in proportion to their sizes (host
// computed), so each block resolves its task once and runs a 32-bit
// grid-stride loop over that task's index space.
__global__ void __launch_bounds__(256) k_prep(const PrepBatch b, const PrepBlocks pbk) {
  pdl_trigger();
  pdl_wait();
  int t = 0;
  while (static_cast<int>(blockIdx.x) >= pbk.first[t + 1]) ++t;
  const PrepTask& k = b.t[t];
  const uint32_t count = static_cast<uint32_t>(b.offs[t + 1] - b.offs[t]);
  const uint32_t stride = static_cast<uint32_t>(pbk.first[t + 1] - pbk.first[t]) * blockDim.x;
  run_prep_span(k, count, (blockIdx.x - pbk.first[t]) * blockDim.x + threadIdx.x, stride);
}

int sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

int blocks_for(int64_t work) {
  int64_t b = (work + 255) / 256;
  if (b > 16 * sms()) b = 16 * sms();
  return static_cast<int>(b < 1 ? 1 : b);
}

// CTAs per launch: at most one resident wave, and at most kMaxContrib CTAs per
// output tile (the tile's last arriver reads every contributor's slot: with a
// resident wave over few tiles — 4 token tiles at 512 tokens — that serial
// read was most of the launch).
int max_contrib() {
  static const int v = [] {
    const char* e = getenv("MLRA_THIN_MAXC");
    return e && atoi(e) > 0 ? atoi(e) : 16;
  }();
  return v;
}
template <typename K>
int wave_ctas(K kernel, int smem, int64_t units, int64_t tiles) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, TTHREADS, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t cap = static_cast<int64_t>(per_sm) * sms();
  const int64_t by_tiles = tiles * max_contrib();
  if (by_tiles < cap) cap = by_tiles;
  return static_cast<int>(units < cap ? units : cap);
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// bf16 [outer x inner] (row stride ld elements), box 64 x box_outer, SWIZZLE_128B
cudaError_t thin_map(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t ld,
                     int box_outer) {
  auto enc = encoder();
  if (!enc || ld % 8 || reinterpret_cast<uintptr_t>(base) % 16) return cudaErrorInvalidValue;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                         strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Grid of one launch: one resident wave. The dynamic-smem opt-in is set first,
// so the occupancy query (and the workspace sized from it) matches the launch.
template <int NT>
int thin_ctas(bool row, int64_t units, int64_t tiles) {
  const int smem = ThinSmem<NT>::BYTES;
  static bool attr_row = false, attr_col = false;
  bool& attr = row ? attr_row : attr_col;
  if (!attr) {
    const cudaError_t e =
        row ? cudaFuncSetAttribute(k_rowmma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
            : cudaFuncSetAttribute(k_colmma<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return 0;
    attr = true;
  }
  return row ? wave_ctas(k_rowmma<NT>, smem, units, tiles)
             : wave_ctas(k_colmma<NT>, smem, units, tiles);
}

template <int NT>
void ws_size_nt(bool row, int64_t m, int64_t d, int64_t* ws_floats, int64_t* n_cnt) {
  const int64_t tiles = row ? (m + TM - 1) / TM : (d + TM - 1) / TM;
  const int64_t chunks = row ? (d + TILE - 1) / TILE : (m + TILE - 1) / TILE;
  const int64_t units = tiles * chunks;
  const int64_t ctas = units > 0 ? thin_ctas<NT>(row, units, tiles) : 0;
  *ws_floats = ctas * 2 * TM * 8 * NT;
  *n_cnt = tiles;
}

template <int NT>
cudaError_t rowmma_nt(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                      const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t ldw, int64_t r,
                      ThinOut o, cudaStream_t st) {
  constexpr int ROWS = 8 * NT;
  const int64_t tb = (m + TM - 1) / TM;
  const int64_t kchunks = (kd + TILE - 1) / TILE;
  const int64_t units = tb * kchunks;
  if (units <= 0) return cudaSuccess;
  if (units > INT32_MAX || lo != hi + ROWS * ldw || !o.ws || !o.cnt || !o.out)
    return cudaErrorInvalidValue;
  CUtensorMap am, fm;
  cudaError_t e = thin_map(&am, act, kd, m, lda, TM);
  if (e == cudaSuccess) e = thin_map(&fm, hi, ldw, 2 * ROWS, ldw, 2 * ROWS);
  if (e != cudaSuccess) return e;
  const int smem = ThinSmem<NT>::BYTES;
  o.rc = static_cast<int>(r);
  const int ctas = thin_ctas<NT>(true, units, tb);
  if (ctas <= 0 || o.ws_floats < static_cast<int64_t>(ctas) * 2 * TM * ROWS)
    return cudaErrorInvalidValue;
  return launch_pdl(k_rowmma<NT>, dim3(ctas), dim3(TTHREADS), smem, st, true, am, fm, m,
                    static_cast<int>(kchunks), static_cast<int>(units), o);
}

template <int NT>
cudaError_t colmma_nt(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                      const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t ldv, int64_t r,
                      ThinOut o, cudaStream_t st) {
  constexpr int ROWS = 8 * NT;
  const int64_t nb = (nd + TM - 1) / TM;
  const int64_t tchunks = (m + TILE - 1) / TILE;
  const int64_t units = nb * tchunks;
  if (units <= 0) return cudaSuccess;
  if (units > INT32_MAX || lo != hi + ROWS * ldv || !o.ws || !o.cnt || !o.out)
    return cudaErrorInvalidValue;
  CUtensorMap am, fm;
  cudaError_t e = thin_map(&am, act, nd, m, lda, TILE);
  if (e == cudaSuccess) e = thin_map(&fm, hi, ldv, 2 * ROWS, ldv, 2 * ROWS);
  if (e != cudaSuccess) return e;
  const int smem = ThinSmem<NT>::BYTES;
  const int ctas = thin_ctas<NT>(false, units, nb);
  if (ctas <= 0 || o.ws_floats < static_cast<int64_t>(ctas) * 2 * TM * ROWS)
    return cudaErrorInvalidValue;
  o.rc = static_cast<int>(r);
  return launch_pdl(k_colmma<NT>, dim3(ctas), dim3(TTHREADS), smem, st, true, am, fm, nd,
                    static_cast<int>(tchunks), static_cast<int>(units), o);
}

template <int NT, int CL>
cudaError_t rowmma_cl_nt(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                         const float* F, int64_t ldf, int64_t r, ThinOut o, const PrepBatch& post,
                         cudaStream_t st) {
  const int64_t tb = (m + TM - 1) / TM;
  const int64_t kchunks = (kd + TILE - 1) / TILE;
  if (tb * CL > INT32_MAX || kchunks > INT32_MAX || !o.out) return cudaErrorInvalidValue;
  CUtensorMap am;
  cudaError_t e = thin_map(&am, act, kd, m, lda, TM);
  if (e != cudaSuccess) return e;
  constexpr int smem = ThinSmem<NT, kClNS>::BYTES;
  static bool attr = false;
  if (!attr) {
    e = cudaFuncSetAttribute(k_rowmma_cl<NT, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess && CL > 8)
      e = cudaFuncSetAttribute(k_rowmma_cl<NT, CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  o.rc = static_cast<int>(r);
  return launch_pdl(k_rowmma_cl<NT, CL>, dim3(static_cast<unsigned>(tb * CL)), dim3(TTHREADS), smem,
                    st, true, am, F, ldf, kd, m, static_cast<int>(kchunks), o, post);
}

}  // namespace

cudaError_t launch_prep(const PrepBatch& b, cudaStream_t st) {
  if (b.n == 0 || b.offs[b.n] == 0) return cudaSuccess;
  PrepBlocks pbk{};
  int nb = 0;
  for (int t = 0; t < b.n; ++t) {
    const int64_t count = b.offs[t + 1] - b.offs[t];
    if (count >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
    int64_t want = (count + 4 * 256 - 1) / (4 * 256);  // ~4 elements per thread
    if (want > 4 * sms()) want = 4 * sms();
    pbk.first[t] = nb;
    nb += static_cast<int>(want);  // zero-size tasks get no block
  }
  pbk.first[b.n] = nb;
  if (nb == 0) return cudaSuccess;
  return launch_pdl(k_prep, dim3(nb), dim3(256), 0, st, true, b, pbk);
}

int thin_rows(int64_t r, bool ones) { return static_cast<int>((r + (ones ? 1 : 0) + 7) / 8 * 8); }

#define MLRA_NT_DISPATCH(NTV, CALL)            \
  switch (NTV) {                               \
    case 1: return CALL(1);                    \
    case 2: return CALL(2);                    \
    case 3: return CALL(3);                    \
    case 4: return CALL(4);                    \
    case 5: return CALL(5);                    \
    case 6: return CALL(6);                    \
    case 7: return CALL(7);                    \
    case 8: return CALL(8);                    \
    case 9: return CALL(9);                    \
    default: return cudaErrorInvalidValue;     \
  }

void thin_ws_size(bool row, int64_t m, int64_t d, int64_t r, bool ones, int64_t* ws_floats,
                  int64_t* n_cnt) {
  *ws_floats = *n_cnt = 0;
#define CALL_WS(N) (ws_size_nt<N>(row, m, d, ws_floats, n_cnt), 0)
  const int nt = thin_rows(r, ones) / 8;
  switch (nt) {
    case 1: CALL_WS(1); break;
    case 2: CALL_WS(2); break;
    case 3: CALL_WS(3); break;
    case 4: CALL_WS(4); break;
    case 5: CALL_WS(5); break;
    case 6: CALL_WS(6); break;
    case 7: CALL_WS(7); break;
    case 8: CALL_WS(8); break;
    case 9: CALL_WS(9); break;
    default: break;
  }
#undef CALL_WS
}

cudaError_t launch_rowmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                          const __nv_bfloat16* wt_hi, const __nv_bfloat16* wt_lo, int64_t ldw,
                          int64_t r, const ThinOut& o, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
#define CALL_ROW(N) rowmma_nt<N>(act, lda, m, kd, wt_hi, wt_lo, ldw, r, o, st)
  MLRA_NT_DISPATCH(thin_rows(r, false) / 8, CALL_ROW)
#undef CALL_ROW
}

cudaError_t launch_colmma(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t nd,
                          const __nv_bfloat16* vt_hi, const __nv_bfloat16* vt_lo, int64_t ldv,
                          int64_t r, const ThinOut& o, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
#define CALL_COL(N) colmma_nt<N>(act, lda, m, nd, vt_hi, vt_lo, ldv, r, o, st)
  MLRA_NT_DISPATCH(thin_rows(r, o.colsum != nullptr) / 8, CALL_COL)
#undef CALL_COL
}

// The fused row product (k_rowmma_cl) serves ranks <= 32 above 512 tokens by
// default: at r = 64 its in-kernel factor split (64 x 64 fp32 per unit) costs
// more than the prep launch it saves (cfg4, r = 64: 2.38 vs 2.28 ms per step),
// and at <= 512 tokens (<= 4 token tiles: <= 64 CTAs in 16-CTA clusters) its
// serial phases cost more than the prep launch too (cfg1: 98.0 vs 96.5 us per
// graphed step); cfg2 / cfg3 at r = 16 / 8 and 1024+ tokens gain (profiles/r04/,
// profiles/r05/). MLRA_THIN_CL=1 forces it for r <= 64 at any token count,
// MLRA_THIN_CL=0 selects the range kernel + prep launch (read per call: A/B
// runs and tests).
constexpr int64_t kThinFusedMinTokens = 513;
bool thin_fused_ok(int64_t r, int64_t m) {
  const char* e = getenv("MLRA_THIN_CL");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return r > 0 && r <= 64;
  return r > 0 && r <= 32 && m >= kThinFusedMinTokens;
}

cudaError_t launch_rowmma_fused(const __nv_bfloat16* act, int64_t lda, int64_t m, int64_t kd,
                                const float* F, int64_t ldf, int64_t r, const ThinOut& o,
                                const PrepBatch& post, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  if (r <= 0 || r > 64 || post.n > kMaxPrep) return cudaErrorInvalidValue;
  // 8 CTAs per 128-token tile when that fills the SMs, else 16
  const bool c8 = (m + TM - 1) / TM * 8 >= sms();
#define CALL_CL(N) (c8 ? rowmma_cl_nt<N, 8>(act, lda, m, kd, F, ldf, r, o, post, st) \
                       : rowmma_cl_nt<N, 16>(act, lda, m, kd, F, ldf, r, o, post, st))
  MLRA_NT_DISPATCH(thin_rows(r, false) / 8, CALL_CL)
#undef CALL_CL
}

}  // namespace mlra

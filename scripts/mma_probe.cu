// mma_probe.cu — tensor-pipe ceiling for the qgemm MMA shapes (dev tool).
// Back-to-back tcgen05.mma from fixed (zeroed) shared memory, no loads:
//   mode 0: cta_group::1, M=128, N=256, one accumulator
//   mode 1: cta_group::2, M=256, N=256, two accumulators (qgemm2's shape)
//   mode 2: cta_group::2, M=256, N=256, one accumulator
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2309_16119_b200/csrc/ptx.cuh"

using namespace mlra;

template <int MODE>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536 + 64);
  const int warp = threadIdx.x >> 5;
  constexpr bool PAIR = MODE != 0;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) {
    if (PAIR) tmem_alloc2(slot, 512); else tmem_alloc(slot, 512);
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const bool leader = !PAIR || cluster_ctarank() == 0;
  if (warp == 1 && leader && (threadIdx.x & 31) == 0) {
    const uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, 256, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = sdesc_sw128(a + k * 32, 16, 1024);
        if (MODE == 1) {
          for (int acc = 0; acc < 2; ++acc)
            tc_mma_f16_2sm(tmem + acc * 256, ad, sdesc_sw128(b + acc * 16384 + k * 32, 16, 1024),
                           idesc, 1);
        } else if (MODE == 2) {
          tc_mma_f16_2sm(tmem, ad, sdesc_sw128(b + k * 32, 16, 1024), idesc, 1);
        } else {
          tc_mma_f16(tmem, ad, sdesc_sw128(b + k * 32, 16, 1024), idesc, 1);
        }
      }
      if ((it & 7) == 7 || it == iters - 1) {  // bound the queue: wait every 8 k-blocks
        if (PAIR) tc_commit_2sm_mc(bar, 0x1); else tc_commit(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
      }
    }
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  if (PAIR) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (PAIR) tmem_dealloc2(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

template <int MODE>
void run(int iters) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  cudaMemset(cyc, 0, 148 * 8);
  const int smem = 65536 + 128;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = MODE == 0 ? 1 : 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaLaunchKernelEx(&cfg, probe<MODE>, iters, cyc);  // warm-up
  cudaEventRecord(s);
  cudaLaunchKernelEx(&cfg, probe<MODE>, iters, cyc);
  cudaEventRecord(e);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  // MACs per k-block per SM
  const double macs_per_sm = MODE == 0 ? 128.0 * 256 * 64 : (MODE == 1 ? 2 * 128.0 * 256 * 64 : 128.0 * 256 * 64);
  const double flops = 2.0 * macs_per_sm * 148 * iters;
  printf("mode %d: %s  %.3f ms  %.1f TFLOP/s  cycles/k-block(SM) %.0f  (ideal %d)\n", MODE,
         cudaGetErrorString(err), ms, flops / (ms * 1e-3) / 1e12, double(mx) / iters,
         MODE == 1 ? 1024 : 512);
}

int main() {
  const int iters = 20000;
  run<0>(iters);
  run<1>(iters);
  run<2>(iters);
  return 0;
}

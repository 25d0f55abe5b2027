// Dev probe: HBM read bandwidth of TMA streaming with different box shapes
// (the row product's access pattern): a [R x C] bf16 matrix read in boxes of
// {64 cols, BR rows}, NB consecutive 64-col chunks per stage, CL CTAs per row
// tile (each a contiguous column range), NS-deep ring; no compute.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__global__ void __launch_bounds__(256) k_stream(const __grid_constant__ CUtensorMap map, int R, int C,
                                                int BR, int NB, int CL, int NS, int stage_bytes,
                                                unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * stage_bytes);
  const int tile = blockIdx.x / CL, s = blockIdx.x % CL;
  const int nch = C / 64;
  const int c0 = nch * s / CL, c1 = nch * (s + 1) / CL;
  const int nst = (c1 - c0 + NB - 1) / NB;
  if (threadIdx.x == 0) {
    for (int b = 0; b < NS; ++b)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&full[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int st, int slot) {
    const int cb = c0 + st * NB;
    const int n = (c1 - cb) < NB ? (c1 - cb) : NB;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&full[slot])),
                 "r"(n * BR * 128));
    for (int i = 0; i < n; ++i)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
          ::"r"(su32(sm + slot * stage_bytes + i * BR * 128)), "l"(&map), "r"((cb + i) * 64),
          "r"(tile * BR), "r"(su32(&full[slot]))
          : "memory");
  };
  if (threadIdx.x == 0)
    for (int b = 0; b < NS - 1 && b < nst; ++b) issue(b, b);
  unsigned acc = 0;
  for (int i = 0; i < nst; ++i) {
    const int b = i % NS;
    if (threadIdx.x == 0 && i + NS - 1 < nst) issue(i + NS - 1, (i + NS - 1) % NS);
    uint32_t ok = 0;
    const uint32_t ph = (i / NS) & 1;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(su32(&full[b])), "r"(ph));
    acc += sm[b * stage_bytes + threadIdx.x * 4];
    __syncthreads();
  }
  if (acc == 0xFFFFFFFF) sink[0] = acc;
}

__global__ void k_ldg(const uint4* p, size_t n, unsigned long long* sink) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

int main() {
  const int R = 4096;
  const int Cs[2] = {11008, 4096};
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  char* flush;
  cudaMalloc(&flush, 512 << 20);
  for (int C : Cs) {
    void* mat;
    const size_t bytes = (size_t)R * C * 2;
    cudaMalloc(&mat, bytes);
    cudaMemset(mat, 1, bytes);
    struct Cfg { int BR, NB, CL, NS; };
    const Cfg cfgs[] = {{128, 1, 8, 3}, {128, 1, 8, 6}, {128, 1, 16, 3}, {128, 2, 8, 3},
                        {64, 2, 4, 3}, {32, 4, 2, 3}, {16, 8, 1, 3}, {32, 8, 2, 3}, {64, 4, 4, 3},
                        {32, 4, 2, 6}, {64, 2, 8, 3}};
    for (const Cfg& c : cfgs) {
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
      cuuint64_t str[1] = {(cuuint64_t)C * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)c.BR};
      cuuint32_t es[2] = {1, 1};
      if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, str, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        continue;
      }
      const int stage = c.BR * 128 * c.NB;
      const int smem = 1024 + c.NS * stage + 8 * c.NS;
      cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int grid = (R / c.BR) * c.CL;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e9, tot = 0;
      for (int it = 0; it < 12; ++it) {
        cudaMemsetAsync(flush, it, 512 << 20);
        cudaEventRecord(a);
        k_stream<<<grid, 256, smem>>>(m, R, C, c.BR, c.NB, c.CL, c.NS, stage, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it >= 2) { tot += ms; if (ms < best) best = ms; }
      }
      cudaError_t e = cudaGetLastError();
      printf("{\"C\": %d, \"BR\": %d, \"NB\": %d, \"CL\": %d, \"NS\": %d, \"grid\": %d, \"smem\": %d, "
             "\"best_us\": %.2f, \"avg_us\": %.2f, \"GBps_avg\": %.0f, \"err\": \"%s\"}\n",
             C, c.BR, c.NB, c.CL, c.NS, grid, smem, best * 1e3, tot / 10 * 1e3,
             bytes / (tot / 10 * 1e-3) / 1e9, cudaGetErrorString(e));
    }
    {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float tot = 0;
      for (int it = 0; it < 12; ++it) {
        cudaMemsetAsync(flush, it, 512 << 20);
        cudaEventRecord(a);
        k_ldg<<<148 * 8, 256>>>(reinterpret_cast<const uint4*>(mat), bytes / 16, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it >= 2) tot += ms;
      }
      printf("{\"C\": %d, \"ldg_linear\": true, \"avg_us\": %.2f, \"GBps_avg\": %.0f}\n", C,
             tot / 10 * 1e3, bytes / (tot / 10 * 1e-3) / 1e9);
    }
    cudaFree(mat);
  }
  return 0;
}

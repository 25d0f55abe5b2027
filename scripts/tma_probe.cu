// Probe: which TMA descriptor shapes are legal (u8 / f32, small boxes, no swizzle).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "../paper_2309_16119_b200/csrc/ptx.cuh"

using namespace mlra;

__global__ void probe(const __grid_constant__ CUtensorMap m, int bytes, int c0, int c1, float* out) {
  __shared__ __align__(1024) uint8_t buf[16384];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_2d(buf, &m, &bar, c0, c1);
  }
  mbar_wait(&bar, 0);
  out[threadIdx.x] = buf[threadIdx.x];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  void* g;
  cudaMalloc(&g, 1 << 24);
  cudaMemset(g, 1, 1 << 24);
  float* out;
  cudaMalloc(&out, 4096);
  struct Case { const char* name; CUtensorMapDataType dt; int es; unsigned long long inner, outer; unsigned bi, bo; CUtensorMapL2promotion l2; };
  Case cases[] = {
      {"u8 128x256 box 32x128 L2_256", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128, 256, 32, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
      {"u8 128x256 box 32x128 L2_none", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128, 256, 32, 128, CU_TENSOR_MAP_L2_PROMOTION_NONE},
      {"f32 8x256 box 4x128 L2_256", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 8, 256, 4, 128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B},
      {"f32 8x256 box 4x128 L2_none", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 8, 256, 4, 128, CU_TENSOR_MAP_L2_PROMOTION_NONE},
      {"f32 64x256 box 16x128 L2_none", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 64, 256, 16, 128, CU_TENSOR_MAP_L2_PROMOTION_NONE},
      {"u8 1536x256 box 48x128 L2_none", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 1536, 256, 48, 128, CU_TENSOR_MAP_L2_PROMOTION_NONE},
  };
  for (auto& c : cases) {
    CUtensorMap m;
    cuuint64_t dims[2] = {c.inner, c.outer};
    cuuint64_t strides[1] = {c.inner * c.es};
    cuuint32_t box[2] = {c.bi, c.bo};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, c.dt, 2, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, c.l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    probe<<<1, 128>>>(m, c.bi * c.bo * c.es, 0, 0, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%-34s encode=%d run=%s\n", c.name, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;  // context is dead after an exception
  }
  return 0;
}

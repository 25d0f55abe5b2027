// Pair-kernel family d1: dX (MN-major weight tile), stream-K / split-K schedules.
#include "qgemm2_kernel.cuh"

namespace mlra {
cudaError_t qgemm2_launch_d1(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool w_tma,
                             bool out_f32, cudaStream_t stream) {
  return dispatch2<true, true>(maps, q, p, w_tma, out_f32, stream);
}
}  // namespace mlra

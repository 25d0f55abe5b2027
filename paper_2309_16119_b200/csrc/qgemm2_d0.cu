// Pair-kernel family d0: dX (MN-major weight tile), whole tiles.
#include "qgemm2_kernel.cuh"

namespace mlra {
cudaError_t qgemm2_launch_d0(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p, bool w_tma,
                             bool out_f32, cudaStream_t stream) {
  return dispatch2<true, false>(maps, q, p, w_tma, out_f32, stream);
}
}  // namespace mlra

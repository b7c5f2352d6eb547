// Instantiation of the fused tracker, the Cauchy endgame and the batched LU solve for N = 14 (see tracker.cuh, endgame.cuh, zgesv.cuh).
#include "endgame.cuh"
#include "zgesv.cuh"
namespace hcb {
cudaError_t launch_tracker_14(const TrackArgs &A, int device, cudaStream_t s, TrackerPlan *p) {
  return launch_tracker_n<14>(A, device, s, p);
}
// the wide latency layout (one track per warp on 32 lanes), chosen for batches that under-fill the GPU
cudaError_t launch_tracker_wide_14(const TrackArgs &A, int device, cudaStream_t s, TrackerPlan *p) {
  return launch_tracker_n<14, 32>(A, device, s, p);
}
cudaError_t launch_zgesv_14(int64_t batch, const double2 *A, const double2 *b, double2 *x, int32_t *info,
                           double pivot_rel, cudaStream_t s) {
  return launch_zgesv_n<14>(batch, A, b, x, info, pivot_rel, s);
}
cudaError_t launch_endgame_14(const TrackArgs &A, int device, cudaStream_t s) {
  return launch_endgame_n<14>(A, device, s);
}
cudaError_t launch_endgame_wide_14(const TrackArgs &A, int device, cudaStream_t s) {
  return launch_endgame_n<14, 32>(A, device, s);
}
}  // namespace hcb

// lane_inst.cu -- the lane-per-path list kernel (lane_kernel.cuh), float32
// and int8 element types, behind two C launchers for runtime.cu.
#include "lane_kernel.cuh"

extern "C" cudaError_t pb_lane_launch(const pb::lk::LParams *p, int mode, int grid, size_t smem, cudaStream_t st) {
    return mode == 0 ? pb::lk::lane_launch_t<float>(p, grid, smem, st)
                     : pb::lk::lane_launch_t<int8_t>(p, grid, smem, st);
}
extern "C" cudaError_t pb_lane_occupancy(int mode, size_t smem, int fpc, int *bps) {
    return mode == 0 ? pb::lk::lane_occ_t<float>(smem, fpc, bps) : pb::lk::lane_occ_t<int8_t>(smem, fpc, bps);
}

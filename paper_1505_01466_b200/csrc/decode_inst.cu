// decode_inst.cu -- one (element type, warps per frame, paths per warp)
// instantiation of the decode kernel; compiled once per shape with
// -DPB_T=<float|int8_t> -DPB_W=<w> -DPB_PPW=<p> -DPB_CHG=<0|1> -DPB_TAG=<tag> (see _native.py).
#include "decode_kernel.cuh"

#define PB_CAT2(a, b) a##b
#define PB_CAT(a, b) PB_CAT2(a, b)

extern "C" cudaError_t PB_CAT(pb_launch_, PB_TAG)(const pb::Params *p, int grid, size_t smem, cudaStream_t st) {
    return pb::launch_t<PB_T, PB_W, PB_PPW, PB_CHG>(p, grid, smem, st);
}
extern "C" cudaError_t PB_CAT(pb_occ_, PB_TAG)(size_t smem, int fpc, int *bps) {
    return pb::occ_t<PB_T, PB_W, PB_PPW, PB_CHG>(smem, fpc, bps);
}

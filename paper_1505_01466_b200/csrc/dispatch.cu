// dispatch.cu -- maps (mode, warps per frame, paths per warp) to the
// separately compiled kernel instantiation (shapes.def).
#include <cuda_runtime.h>
#include <stdint.h>

#include "decoder.cuh"

// experiments may build a subset of the shapes (_native.build, PB_SHAPES)
#ifndef PB_SHAPES_DEF
#define PB_SHAPES_DEF "shapes.def"
#endif

#define PB_SHAPE(tag, T, mode, W, P, CHG)                                                                         \
    extern "C" cudaError_t pb_launch_##tag(const pb::Params *p, int grid, size_t smem, cudaStream_t st); \
    extern "C" cudaError_t pb_occ_##tag(size_t smem, int fpc, int *bps);
#include PB_SHAPES_DEF
#undef PB_SHAPE

extern "C" int pb_shape_supported(int mode, int warps, int ppw, int chg) {
#define PB_SHAPE(tag, T, md, W, P, CHG) \
    if (mode == md && warps == W && ppw == P && chg == CHG) return 1;
#include PB_SHAPES_DEF
#undef PB_SHAPE
    return 0;
}

extern "C" cudaError_t pb_launch_decode(const pb::Params *p, int mode, int warps, int ppw, int chg, int grid, size_t smem,
                                        cudaStream_t stream) {
#define PB_SHAPE(tag, T, md, W, P, CHG) \
    if (mode == md && warps == W && ppw == P && chg == CHG) return pb_launch_##tag(p, grid, smem, stream);
#include PB_SHAPES_DEF
#undef PB_SHAPE
    return cudaErrorInvalidValue;
}

extern "C" cudaError_t pb_occupancy(int mode, int warps, int ppw, int chg, size_t smem, int fpc, int *blocks_per_sm) {
#define PB_SHAPE(tag, T, md, W, P, CHG) \
    if (mode == md && warps == W && ppw == P && chg == CHG) return pb_occ_##tag(smem, fpc, blocks_per_sm);
#include PB_SHAPES_DEF
#undef PB_SHAPE
    return cudaErrorInvalidValue;
}

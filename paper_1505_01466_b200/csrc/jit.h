// jit.h -- per-code specialised lane kernel (jit.cu): source generation, NVRTC
// compilation with an in-tree cubin cache, module loading and launch through
// the driver API.  Both libraries are dlopen'ed, so the decoder library loads
// (and the generic kernels run) without them.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "decoder.cuh"

namespace pb {
namespace jit {

// what the generated kernel is specialised on
struct Spec {
    int N = 0, n = 0, k = 0, L = 0, mode = 0, has_crc = 0;
    uint32_t crc_const = 0;
    lk::LLayout lay{};
    std::vector<lk::LOp> prog;
    int final_op = -1;
    int policy = 1;  // pb_options.specialize (> 0)
    int G = 1;       // frames per warp (list sizes <= 16): lane = frame slot * 32/G + path slot
    int fpc = 16;    // warps per CTA the kernel is compiled for: __launch_bounds__(32 * fpc, 1)
};

// policy bits beyond 1 (= everything compile-time)
enum : int {
    POL_FULL = 1,
    POL_RT_TARGET = 2,     // leaf chain targets read at run time: fewer variants (3.64 against 4.07 Gbit/s)
    POL_CHAIN_LEVELS = 4,  // Combine chains level by level (default: the unrolled form, all loads independent:
                           // c3 L=32 4.49 -> 4.62 Gbit/s)
    POL_SCAN_PIPE2 = 8,    // wide-leaf scans software-pipelined over blocks of 2 quads (default)
    POL_ASG_LOOP = 64,     // survivor hand-over as a loop over set bits (keys in local memory; default at L <= 2)
};

// The generated translation unit and, per op, the variant id the kernel
// switches on (LParams::vid).
std::string generate(const Spec &sp, std::vector<uint16_t> &vid, int *n_variants);

struct Kernel;  // a loaded module + function (shared between handles of the same code)

// Compile (or fetch from the cubin cache) and load into the current context of `device`.  device-free when
// load == false (prebuild: fills the cache only).  nullptr + err on failure.
Kernel *acquire(const std::string &source, bool load, int device, std::string &err, bool *cache_hit,
                double *compile_s);
void release(Kernel *k);
cudaError_t launch(Kernel *k, const lk::LParams *p, int grid, int threads, size_t smem, cudaStream_t st,
                   std::string &err);
// resident CTAs per SM of the loaded kernel (0 on failure)
int occupancy(Kernel *k, int threads, size_t smem);
int registers(Kernel *k);
std::string cache_dir();

}  // namespace jit
}  // namespace pb

// decoder.cuh -- device program, layouts and launch parameters shared by the
// host runtime (runtime.cu) and the decode kernels (decode_kernel.cu).
#pragma once
#ifndef __CUDACC_RTC__
#include <stdint.h>
#else  // NVRTC (the per-code specialised lane kernel, jit.cpp): no host headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef short int16_t;
typedef unsigned short uint16_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned long size_t;
#endif

namespace pb {

constexpr int kMaxLog = 16;     // N <= 65536
constexpr int kMaxL = 32;       // selection runs on one warp: one lane per source path
constexpr int kMaxCand = 8;
constexpr int kInlineOps = 1536;  // op programs up to this long travel in the kernel parameters (24 KB)

// threads per CTA the kernels are compiled for (__launch_bounds__): the
// register budget per thread is 65536 / PB_MAXT.  512 = 16 single-warp frames
// per SM at 128 registers: the decode is latency-bound, and 16 resident
// frames beat 8 frames at 255 registers by 30-45 % (c3 L=32 1.86 -> 2.41,
// c5 L=16 1.96 -> 2.93 Gbit/s) despite ~0.9 KB of spills (to L1).
#ifndef PB_MAXT
#define PB_MAXT 512
#endif
constexpr int kMaxThreads = PB_MAXT;
// Shapes with <= 4 path slots per warp (L <= 4, one warp per frame) are
// compiled for 1024 threads (64 registers, 32 resident frames per SM): their
// per-frame state is small and more frames win (same-box A/B: c1 L=4
// 2.36 -> 2.98, c3 L=2 6.06 -> 8.19 Gbit/s).  At 8 paths per warp it was
// mixed (c2 +11 %, c3 L=8 -7 %) and those shapes stay at PB_MAXT.
#ifndef PB_MAXT_SMALL
#define PB_MAXT_SMALL 1024
#endif
__host__ __device__ constexpr int shape_max_threads(int warps, int ppw) {
    return warps == 1 && ppw <= 4 ? PB_MAXT_SMALL : kMaxThreads;
}

// Device op kinds.  Combines never appear: each leaf carries its chain of
// combines.
enum : int8_t { DK_F = 0, DK_G = 1, DK_R0 = 2, DK_REP = 3, DK_R1 = 4, DK_SPC = 5, DK_NOP = 6 };

// how an op reads stage n-1 (never stored): recomputed from the channel
enum : int8_t { VM_NONE = 0, VM_F = 1, VM_G = 2 };

struct __align__(16) DOp {
    int8_t kind;     // DK_*
    int8_t stage;    // F/G: stage read (writes stage-1); leaf: its stage t
    int8_t pin;      // active paths before the op
    int8_t pout;     // active paths after (leaf)
    int8_t target;   // leaf: slot s* its chain of combines ends in (n = root)
    int8_t ncand;    // leaf: candidates per path C
    int8_t select;   // leaf: pin*ncand > L (a real 2L->L selection)
    int8_t vmode;    // how this op reads stage n-1 (VM_*), else VM_NONE
    int32_t off;     // leaf: first u index covered
    int8_t lgi, lgo; // one warp per frame: log2 lanes per path for pin / pout paths
    // list kernel, F / G fused into the leaf that reads its output (PB_FUSE_LEAF):
    // -1 on the F / G (skipped), 1 / 2 on the leaf (reads f / g of its parent's
    // stored rows); else 0.  The single-path kernel ignores it.
    int8_t fuse;
};
static_assert(sizeof(DOp) == 16, "DOp is one 16-byte load");

// Per-frame storage plan.  Offsets in bytes from the frame's shared-memory
// block, or from its global scratch block for alpha stages >= a_gfrom.
// Alpha rows are quad-interleaved: the PPW rows a warp owns are interleaved
// four elements (one quad) at a time with an XOR swizzle; with E = max(4, 2^s)
// elements per row, quad x of row r starts at element
//   (r / PPW) * PPW * E + (x * PPW + ((r % PPW) ^ (x & min(PPW, 8) - 1))) * 4
// so a warp whose lanes are paths reads 32 quads of 512 contiguous bytes with
// one 128-bit access each, and the lanes of one path spread over the banks.
struct FrameLayout {
    int ch_off;                 // channel LLRs, N elements of T
    int a_off[kMaxLog];         // alpha stage s (s <= n-2)
    int a_gfrom;                // stages >= a_gfrom live in global scratch
    int b_off[kMaxLog];         // beta slot s (s <= n-1): L rows, uint32 words
    int b_gfrom;                // beta slots >= b_gfrom live in global scratch
    int b_stride[kMaxLog];      // row stride, words
    int pm_off;                 // double [2][L]    path metrics (double-buffered)
    int ia_off;                 // uint32 [2][idx_stride][L] alpha row per stage, 4 per word
    int ib_off;                 // uint32 [2][idx_stride][L] beta row per slot, 4 per word
    int idx_stride;             // words per path = ceil(n / 4)
    int cd_off;                 // double [2][L][8] candidate deltas (by leaf parity)
    int clrb_off;               // uint16 [2][L][4] least reliable positions
    int cflag_off;              // uint8 [2][L] parity / ones-first
    int asg_off;                // uint8 [2][L][2] survivor -> (source, cand)
    int hard_off;               // uint32 [2][L][hard_words] hard decisions
    int hard_words;
    int root_off;               // uint32 [root_words] winner codeword scratch
    int root_words;
    int smem_bytes;             // per frame (16-byte multiple)
    int gbytes;                 // per frame global scratch (256-byte multiple)
};

struct Params {
    const DOp *prog;
    int n_ops;
    const uint32_t *xsyn4;      // [N/32][8][16] codeword-domain syndrome nibble tables
    const uint32_t *info_pos;   // [k] payload positions (u index)
    int N, n, k, L;
    int ppw;                    // paths per warp (rows per interleave block), power of two
    int lppw;                   // log2(ppw)
    int has_crc;
    uint32_t crc_const;
    int final_op;               // index of the last leaf
    const void *llr;
    int in_type;                // PB_IN_*
    long long batch;
    uint8_t *info_out;          // [B][k] or null
    uint8_t *crc_ok;            // [B] or null
    double *pm_out;             // [B] or null
    int32_t *paths_used;        // [B] or null
    uint32_t *path_cw;          // paths mode: [B][L][root_words] packed, or null
    double *path_pm;            // [B][L]
    uint8_t *path_crc;          // [B][L]
    unsigned char *gscratch;    // [CTA slots][gbytes]
    long long *op_cycles;       // debug: per-op clock64 deltas of CTA 0's first frame, or null
    int ablate;                 // timing experiments only (PB_ABLATE): skip parts, wrong results
    const int32_t *frame_map;   // adaptive pass: frame f reads / writes row frame_map[f], or null
    const int32_t *batch_dev;   // adaptive pass: frame count on the device (<= batch), or null
    int fpc;                    // frames per CTA (W warps each)
    int prog_smem;              // stage the op program in shared memory (after the frames' blocks)
    int sync_mask;              // CTA barrier after ops with (index & mask) == 0; -1: none
    FrameLayout lay;
    // the op program in the kernel's parameter space (constant bank: a
    // warp-uniform load per op, no L1 / register residency) when it fits
    int prog_inline;
    DOp iprog[kInlineOps];
};

// ---------------------------------------------------------------------
// Lane-per-path list kernel (lane_kernel.cuh): one warp per frame, lane q =
// path slot q (L <= 32), per-path state (metric, row indices, leaf data) in
// registers, the channel in shared memory, the top two stages (n-1, n-2)
// recomputed from it instead of stored.
namespace lk {
constexpr int kMaxOps = 2048;  // the op program travels in the kernel parameters (16 KB)
enum : uint8_t { K_F = 0, K_G = 1, K_R0 = 2, K_REP = 3, K_R1 = 4, K_SPC = 5, K_NOP = 6 };
// where an op's input stage lives: a stored row in shared memory / global
// scratch, recomputed stage n-1 (f / g of the channel halves), recomputed
// stage n-2, or the channel itself (a root leaf)
enum : uint8_t { S_SM = 0, S_GL = 1, S_V1 = 2, S_V2 = 3, S_CH = 4 };
enum : uint8_t { LF_SELECT = 1, LF_V1G = 2, LF_V2G = 4, LF_FUSE_F = 8, LF_FUSE_G = 16,
                 // this op is the last reader of the global-scratch stage it reads: the stage's
                 // lines are discarded from the L2 afterwards (dead until rewritten: no write-back)
                 LF_LAST = 32 };
constexpr int LF_FUSE_SHIFT = 3;  // (flags >> 3) & 3: 0 plain leaf, 1 / 2 the F / G before it folded into its reads

struct __align__(8) LOp {
    uint8_t kind;    // K_*
    uint8_t stage;   // F / G: stage read (writes stage - 1); leaf: its stage t
    uint8_t pin;     // active paths before the op
    uint8_t pout;    // active paths after (leaf)
    uint8_t ncand;   // leaf: candidates per path (2 / 4 / 8; 0 for Rate-0)
    uint8_t src;     // S_*: where the input stage lives (a fused leaf: its parent's stage)
    uint8_t aux;     // F / G: S_SM / S_GL of the output stage; leaf: chain target slot (n = root)
    uint8_t flags;   // LF_*: selection needed; recomputed stages' F / G modes; fused F / G; LF_LAST
};
static_assert(sizeof(LOp) == 8, "LOp is one 8-byte load");

struct LLayout {
    int ch_off;               // channel(s), N elements of T per frame (shared memory, or global: ch_gl)
    int a_off[kMaxLog];       // stored alpha stage s: quad-interleaved rows, 32 rows
    uint32_t a_gl;            // bit s: stage s in global scratch
    int b_off[kMaxLog];       // beta slot s: 32 rows of b_stride[s] words
    int b_stride[kMaxLog];
    uint32_t b_gl;            // bit s: slot s in global scratch
    int asg_off;              // uint8 [32] survivor -> (source << 3 | cand)
    int met_off;              // double [32] survivor metrics
    int root_off;             // uint32 [max(1, N/32)] codeword scratch (finalise)
    int hard_off;             // global: uint32 [hard_words][32] hard decisions of leaves wider than 32
    int smem_bytes;           // per frame (16-byte multiple)
    int gbytes;               // per frame global scratch (256-byte multiple)
    int ch_gl;                // 1: the channel lives in global scratch (ch_off is an offset there): list sizes
                              // <= 16, where the frames sharing a warp would otherwise fill shared memory
};

struct LParams {
    const uint32_t *xsyn4;
    const uint32_t *info_pos;
    int N, n, k, L, has_crc;
    uint32_t crc_const;
    int n_ops, final_op;
    const void *llr;
    int in_type;
    long long batch;
    uint8_t *info_out;
    uint8_t *crc_ok;
    double *pm_out;
    int32_t *paths_used;
    uint32_t *path_cw;
    double *path_pm;
    uint8_t *path_crc;
    unsigned char *gscratch;
    const int32_t *frame_map;
    const int32_t *batch_dev;
    int fpc;
    int sync_mask;
    long long *op_cycles;       // profiling build: clock64 at the start of each op (CTA 0, frame slot 0), or null
    LLayout lay;
    LOp prog[kMaxOps];
    uint16_t vid[kMaxOps];      // specialised build (jit.cpp): op i runs variant vid[i] of PB_JIT_OPS
};
// per-code constants of the specialised build (kJit in the generated source)
struct JitCode {
    int N, n, k, L, has_crc;
    uint32_t crc_const;
    int n_ops, final_op;
    int G;  // frames per warp
};
}  // namespace lk

// ---------------------------------------------------------------------
// Single-path (L = 1) pass: polaris.fastssc.execute_schedule
// (fastssc.py:20-83) and the first stage of AdaptiveDecoder
// (listdec.py:437-459).  One warp per frame, lanes over elements; the frame
// keeps one alpha row per stage and one beta word row per slot in shared
// memory.
struct SscLayout {
    int ch_off;                 // channel LLRs, N elements of T
    int a_off[kMaxLog];         // alpha stage s (s <= n-2), 2^s elements, contiguous
    int b_off[kMaxLog];         // beta slot s (s <= n-1), max(1, 2^s / 32) words
    int root_off;               // codeword x, max(1, N / 32) words
    int smem_bytes;             // per frame (16-byte multiple)
};

enum : int { SSC_LIST_L1 = 0, SSC_FAST = 1, SSC_ADAPTIVE = 2 };

// threads per CTA of k_ssc (__launch_bounds__): 1024 = 32 frames per SM at 64
// registers, the channel in global scratch to fit them
#ifndef PB_SSC_MAXT
#define PB_SSC_MAXT 1024
#endif

struct SscParams {
    const DOp *prog;
    int n_ops;
    const uint32_t *xsyn4;      // codeword-domain CRC syndrome nibble tables
    const uint32_t *info_pos;   // [k]
    int N, n, k;
    int has_crc;
    uint32_t crc_const;
    int semantics;              // SSC_*: leaf decisions of the L = 1 list decoder or of fastssc
    const void *llr;
    int in_type;
    long long batch;
    uint8_t *info_out;          // [B][k] or null
    uint8_t *crc_ok;            // [B] or null
    double *pm_out;             // [B] or null
    int32_t *paths_used;        // [B] or null
    uint8_t *invoked;           // [B] or null (adaptive: 1 = the list decoder takes the frame)
    int32_t *fail_idx;          // adaptive: frames whose CRC failed (unordered)
    int32_t *fail_count;        // adaptive: their number
    uint32_t *cw_out;           // [B][N/32] packed codeword, or null
    unsigned char *gch;         // channel in global scratch ([CTA slots][N] of T), or null: shared memory
    int fpc;                    // frames (warps) per CTA
    SscLayout lay;
};

// On-device frame generation (frame_gen.cu)
namespace gen {
struct GenParams {
    int N, n, k, crc_w;
    const uint32_t *info_pos;   // [k + crc_w] u positions (payload, then CRC)
    const uint32_t *hu;         // [k] CRC syndrome row of payload bit j
    uint32_t crc_const;
    unsigned long long seed;
    long long first, count;
    float sigma, scale;         // noise std, LLR scale 2 / sigma^2
    int out_type;               // 0 float32, 1 int8
    void *llr;                  // [count][N]
    uint32_t *payload;          // [count][kw] packed bits (bit i of word i/32), or null
    int kw;
};
}  // namespace gen

}  // namespace pb

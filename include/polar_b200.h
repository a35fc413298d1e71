/*
 * polar_b200.h -- C ABI of the B200 Fast-SSC list-CRC polar decoder.
 *
 * Drop-in boundary for the reference's list-decode call
 *   polaris.listdec.ListDecoder(schedule, list_size)      listdec.py:171-185
 *   ListDecoder.decode(llr) -> DecodeResult                listdec.py:289-308
 *   ListDecoder.decode_paths(llr) -> list[PathOutcome]     listdec.py:275-287
 *   polaris.decode(llr, schedule, list_size)               listdec.py:462-468
 * (reference root: /root/reference/pkg/src/polaris/).  The reference has no
 * FFI of its own (pure Python); these entry points are what a ctypes / cffi
 * binding of that call would bind -- see INTEGRATION.md.
 *
 * Plain C types only: no torch or CUDA types cross the boundary (the stream is
 * an opaque cudaStream_t passed as void*).  All pointers may be host or
 * device memory; the library detects which.
 */
#ifndef POLAR_B200_H
#define POLAR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PB_API_VERSION 1

/* return codes (0 = success).  The Python layer maps PB_EINVAL to
 * ValueError (same messages as the reference) and the rest to RuntimeError. */
#define PB_OK 0
#define PB_EINVAL -1     /* bad argument: list size, LLR width, schedule ... */
#define PB_ECUDA -2      /* CUDA runtime error (message via pb_last_error) */
#define PB_EINTERNAL -3  /* internal invariant violated */
#define PB_ENOMEM -4     /* device / host allocation failed */

/* schedule op kinds; numbering of schedule.KIND_CODE in the Python package.
 * Mirrors polaris.schedule.NodeKind (schedule.py:29-41). */
#define PB_OP_F 0
#define PB_OP_G 1
#define PB_OP_COMBINE 2
#define PB_OP_RATE0 3
#define PB_OP_RATE1 4
#define PB_OP_REP 5
#define PB_OP_SPC 6

/* arithmetic modes */
#define PB_MODE_F32 0   /* float32 LLRs, float64 path metrics (reference numerics) */
#define PB_MODE_INT8 1  /* int8 saturating LLRs, integer path metrics */

/* input LLR element types for pb_decode / pb_decode_paths */
#define PB_IN_F32 0     /* float32 [batch][N]; int8 mode quantises clip(rint(4x),+-127) */
#define PB_IN_I8 1      /* int8 [batch][N] (int8 mode only) */

/* A polar code: reference polaris.codes.CodeSpec (codes.py:201-265) with its
 * CrcConfig (codes.py:29-61) flattened. crc_width 0 = no CRC. */
typedef struct pb_code {
    int32_t N;               /* block length, power of two, 2..65536 */
    int32_t k;               /* payload bits (CRC excluded), >= 1 */
    const uint8_t *frozen_mask; /* [N] host pointer, 1 = frozen */
    int32_t crc_width;       /* 0, 8, 16 or 32 */
    uint32_t crc_poly;       /* normal form, implicit leading term */
    uint32_t crc_init;
    int32_t crc_reflect;     /* 1 = LSB-first register (IEEE CRC-32 style) */
    uint32_t crc_xor_out;
} pb_code;

/* One schedule step: reference polaris.schedule.NodeOp (schedule.py:44-58). */
typedef struct pb_op {
    int32_t kind;            /* PB_OP_* */
    int32_t size;
    int32_t stage;           /* log2(size) */
    int32_t side;            /* 0 left / 1 right child of the parent */
    int32_t spc_truncated;
} pb_op;

typedef struct pb_handle pb_handle;

/* Explicit launch / planning options (no hidden global state: nothing is
 * read from the environment).  Zero-initialise and set what you need; 0 in
 * any field means "the measured default".  Pass NULL for all defaults. */
typedef struct pb_options {
    int32_t size;             /* sizeof(pb_options) (forward compatibility); 0 = this version */
    int32_t kernel;           /* list kernel: 0 auto (lane-per-path kernel for L > 16 when its plan fits),
                                 1 interpreted multi-shape kernel, 2 lane-per-path kernel (PB_EINVAL if it
                                 cannot be planned) */
    int32_t warps_per_frame;  /* interpreted kernel: warps per frame (1, 2, 4, 8; 0 = 1) */
    int32_t frames_per_sm;    /* resident frames per SM target (0 = launch bound / 32, 16 for L > 16) */
    int32_t sync_every;       /* CTA regroup period in ops (power of two; 0 = auto; -1 = never) */
    int32_t recompute_stages; /* lane kernel: top stages recomputed from the channel (1 or 2; 0 = auto:
                                 2 for float32, 1 for int8) */
    int32_t chunk_frames;     /* host-buffer pipeline chunk in frames (0 = one wave of resident frames,
                                 six for adaptive decoding) */
    int32_t grid_sms;         /* use at most this many SMs (0 = all) */
    int32_t l1_list_kernel;   /* 1: list size 1 through the list kernel instead of the single-path pass */
    int32_t fuse;             /* lane kernel op fusion: 0 auto (everything measured faster), -1 none, else a
                                 bit set: 1 = a leaf reads f / g of its parent's row (its own row is never
                                 stored), 4 = a global-scratch stage is discarded from the L2 after its last
                                 read */
    int32_t specialize;       /* lane kernel compiled per code (NVRTC, cubin cached next to the library): every
                                 distinct op of the schedule becomes one instantiation with stage, placements,
                                 offsets and path counts as constants -- the paper's unrolled decoder.
                                 0 auto (on; the generic kernels run if NVRTC is unavailable), -1 off
                                 (generic kernels), 1 on (PB_ECUDA if it cannot be built); larger values are
                                 explicit policy bits for experiments (csrc/jit.h: 1 | 2 leaf chain targets at
                                 run time, | 4 level-by-level chains, | 8 pipelined wide-leaf scans, | 64
                                 survivor hand-over as a loop) */
    int32_t frames_per_warp;  /* specialised lane kernel, list sizes <= 16: this many frames share one warp
                                 (lane = frame slot x path slot; at most 32 / pow2(L)); 0 auto (32 / pow2(L),
                                 halved until three warps fit an SM), 1 = one frame per warp (the interpreted
                                 kernel for L <= 16) */
    int32_t channel_global;   /* specialised lane kernel: 1 = the channel LLRs live in global scratch (read
                                 through L1 / L2) instead of shared memory, which then holds more warps and
                                 alpha stages; -1 = shared memory; 0 auto (global for list sizes <= 16) */
} pb_options;

/* Build a decoder for (code, schedule, list size) on a CUDA device.
 * Replaces ListDecoder.__init__ (listdec.py:171-185): validates the list size
 * (ValueError "list size X must be >= 1"), re-validates the op list against
 * the schedule grammar (schedule.py:159-201), and uploads the lowered device
 * program, CRC syndrome tables and payload positions.
 * list_size: 1..32 (PB_EINVAL above 32 in this version).  At list size 1,
 * pb_decode runs the single-path kernel with the list decoder's leaf rules
 * (identical results, ~30x faster than a one-path list decode). */
int pb_create(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
              int device, pb_handle **out);

/* pb_create with explicit options (opts may be NULL = pb_create). */
int pb_create_ex(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                 int device, const pb_options *opts, pb_handle **out);

/* The per-code specialised lane kernel (pb_options.specialize) without a
 * device.  pb_jit_source: the generated translation unit (buf may be NULL;
 * *needed = bytes incl. the terminator, *n_variants = distinct op bodies).
 * pb_jit_prebuild: compile it with NVRTC into the cubin cache next to the
 * library (the build step does this for the BASELINE configurations, so a GPU
 * box never compiles them).  PB_EINVAL when the lane kernel cannot be planned
 * for the code, PB_ECUDA when NVRTC is unavailable or the compilation fails. */
int pb_jit_source(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                  const pb_options *opts, char *buf, int64_t cap, int64_t *needed, int32_t *n_variants);
int pb_jit_prebuild(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                    const pb_options *opts, int32_t *cache_hit, double *compile_s);

/* Decode `batch` frames.  Replaces ListDecoder.decode (listdec.py:289-308),
 * batched.  llr: [batch][N] of in_type.  Outputs (each may be NULL):
 *   info_out   uint8 [batch][k]  payload bits of the chosen path (0/1 bytes)
 *   crc_ok     uint8 [batch]     DecodeResult.crc_ok
 *   pm_out     double[batch]     DecodeResult.chosen_pm
 *   paths_used int32 [batch]     DecodeResult.paths_used
 * Host buffers: synchronous (staged through device memory on `stream`).
 * All-device buffers: asynchronous on `stream` (a cudaStream_t; NULL = default).
 */
int pb_decode(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *info_out,
              uint8_t *crc_ok, double *pm_out, int32_t *paths_used, void *stream);

/* Every surviving path of every frame: ListDecoder.decode_paths
 * (listdec.py:275-287).  codewords: uint8 [batch][list_size][N] (root bit
 * estimates x, one byte per bit), path_pm double [batch][list_size],
 * path_crc uint8 [batch][list_size], paths_used int32 [batch]; rows beyond
 * paths_used[b] are zero.  Host buffers only; synchronous. */
int pb_decode_paths(pb_handle *h, const void *llr, int in_type, int64_t batch,
                    uint8_t *codewords, double *path_pm, uint8_t *path_crc,
                    int32_t *paths_used, void *stream);

/* Adaptive decoding: AdaptiveDecoder.decode (listdec.py:437-459), batched.
 * A single-path Fast-SSC pass (fastssc.py:20-83) decodes every frame; frames
 * whose CRC passes keep that result (paths_used 1, invoked_list 0), the rest
 * are re-decoded by the list decoder of this handle (invoked_list 1).  The
 * failing frames are queued on the device: no host round trip between the
 * two kernels.  Outputs as pb_decode plus invoked_list uint8 [batch] (may be
 * NULL).  PB_EINVAL "adaptive decoding needs a CRC in the code spec" for a
 * code without CRC (the reference raises ValueError in the constructor). */
int pb_decode_adaptive(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *info_out,
                       uint8_t *crc_ok, double *pm_out, int32_t *paths_used, uint8_t *invoked_list,
                       void *stream);

/* The single-path pass alone: polaris.fastssc.execute_schedule
 * (fastssc.py:20-83).  codewords uint8 [batch][N] (one byte per bit),
 * pm_out double [batch].  Host buffers only; synchronous. */
int pb_fastssc(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *codewords,
               double *pm_out, void *stream);

/* On-device frame generation for throughput sweeps: frames
 * first_frame .. first_frame+count-1 of the (seed, Eb/N0) stream for this
 * handle's code -- payload bits, CRC attach (encode.py:56-73), polar encode
 * (encode.py:29-53), BPSK-AWGN LLRs 2y/sigma^2 clamped (sim.py:79-91).
 * Counter-based Philox4x32-10 per frame: shard- and batch-split invariant,
 * statistically equivalent to (not bit-identical with) the reference's numpy
 * stream.  llr_out [count][N] float32 (out_type PB_IN_F32) or int8
 * (PB_IN_I8, clip(rint(4 llr), +-127)); payload_out [count][ceil(k/32)]
 * packed bits or NULL.  Device buffers; asynchronous on `stream`. */
int pb_generate_frames(pb_handle *h, uint64_t seed, double ebn0_db, int64_t first_frame, int64_t count,
                       int out_type, void *llr_out, uint32_t *payload_out, void *stream);

/* Frame / bit error counters (sim.py:_chunk_counts) of decoded payload bytes
 * info [batch][k] against packed payloads [batch][ceil(k/32)], ADDED per
 * chunk of `chunk` frames into counts [ceil(batch/chunk)][3] uint64 =
 * (frames, frame errors, bit errors).  Device buffers; async on `stream`. */
int pb_count_errors(pb_handle *h, const uint8_t *info, const uint32_t *payload, int64_t batch, int chunk,
                    uint64_t *counts, void *stream);

/* Release the handle and its device memory. */
int pb_destroy(pb_handle *h);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *pb_last_error(void);

/* Launch configuration / storage plan the handle chose, as a JSON string
 * owned by the handle (valid until pb_destroy). */
const char *pb_plan_json(pb_handle *h);

/* Kernel launches issued by this handle so far (for launch accounting). */
int64_t pb_launch_count(pb_handle *h);

/* Device time of the most recent pb_decode's decode kernel, in milliseconds,
 * measured with CUDA events on the launch stream (0 if unavailable). */
double pb_last_kernel_ms(pb_handle *h);

/* API version (PB_API_VERSION). */
int pb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* POLAR_B200_H */

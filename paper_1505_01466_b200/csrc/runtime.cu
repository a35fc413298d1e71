// runtime.cu -- native host runtime behind include/polar_b200.h.
//
//   * validates the reference schedule (grammar of schedule.py:159-201) and
//     lowers it to the device program: root F/G become mode switches for the
//     never-stored stage n-1, every leaf absorbs the Combines that follow it
//     (its "chain"), and the active-path count before/after every op is
//     resolved statically (it does not depend on the data)
//   * builds the CRC tables: per-u-position syndrome rows (codes.py:127-156 as
//     an affine GF(2) map) transformed into the codeword domain (x = u G_N),
//     as nibble tables: a survivor's CRC check is one XOR pass over its root
//     codeword at the end of the frame
//   * plans the per-frame storage (shared memory vs global scratch per alpha
//     stage) for the interpreted kernel and the lane-per-path kernel
//     (lane_lower / plan_lane: frames per warp, channel placement, fused
//     leaves, last readers), has jit.cu compile the lane kernel for the code
//     (make_jit_spec), sizes the persistent grids, stages host buffers,
//     orders launches that share a handle's scratch, times launches.  Every
//     knob is an explicit pb_options field (no environment reads).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/polar_b200.h"
#include "decoder.cuh"
#include "jit.h"

#ifndef PB_PROFILE
#define PB_PROFILE 0
#endif

extern "C" cudaError_t pb_launch_decode(const pb::Params *p, int mode, int warps, int ppw, int chg, int grid, size_t smem,
                                        cudaStream_t stream);
extern "C" cudaError_t pb_occupancy(int mode, int warps, int ppw, int chg, size_t smem, int fpc, int *blocks_per_sm);
extern "C" int pb_shape_supported(int mode, int warps, int ppw, int chg);
extern "C" cudaError_t pb_lane_launch(const pb::lk::LParams *p, int mode, int grid, size_t smem, cudaStream_t st);
extern "C" cudaError_t pb_lane_occupancy(int mode, size_t smem, int fpc, int *bps);
extern "C" cudaError_t pb_launch_ssc(const pb::SscParams *p, int mode, int grid, cudaStream_t st);
extern "C" cudaError_t pb_occupancy_ssc(int mode, int fpc, size_t smem_frame, int *bps);
extern "C" cudaError_t pb_launch_gen(const pb::gen::GenParams *p, int sms, cudaStream_t st);
extern "C" cudaError_t pb_launch_errcount(const uint8_t *info, const uint32_t *payload, long long batch, int k, int kw,
                                       int chunk, unsigned long long *counts, int sms, cudaStream_t st);
#include <cmath>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(PB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PB_CUDA(call)                                   \
    do {                                                \
        cudaError_t _e = (call);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

uint32_t rev_bits(uint32_t v, int w) {
    uint32_t r = 0;
    for (int i = 0; i < w; ++i) {
        r = (r << 1) | (v & 1u);
        v >>= 1;
    }
    return r;
}

struct Crc {
    int w;
    uint32_t poly, init, xor_out;
    bool reflect;
    uint32_t mask() const { return w == 32 ? 0xffffffffu : ((1u << w) - 1u); }
    uint32_t step(uint32_t reg, int b) const {  // codes.py:79-118
        if (reflect) {
            uint32_t rp = rev_bits(poly, w);
            return ((reg ^ (uint32_t)b) & 1u) ? (reg >> 1) ^ rp : reg >> 1;
        }
        uint32_t fb = ((reg >> (w - 1)) ^ (uint32_t)b) & 1u;
        return ((reg << 1) & mask()) ^ (fb ? poly : 0u);
    }
    uint32_t start() const { return reflect ? rev_bits(init, w) : init; }
    // checksum value -> append-order bit vector (bit j = j-th appended bit)
    uint32_t append_word(uint32_t value) const {  // codes.py:121-124
        if (reflect) return value & mask();
        return rev_bits(value & mask(), w);
    }
};

struct Handle;

}  // namespace

struct pb_handle {
    int device = 0, mode = 0, L = 0, N = 0, n = 0, k = 0;
    pb::Params base{};
    std::vector<pb::DOp> prog;
    pb::DOp *d_prog = nullptr;
    uint32_t *d_xsyn4 = nullptr, *d_info = nullptr;
    int grid = 0, blocks_per_sm = 0, sms = 0, warps = 1, ppw = 1;
    int fpc = 1;  // frames per CTA
    bool chg = false;  // channel in global scratch (not shared memory)
    size_t smem_frame = 0;
    size_t prog_smem = 0;  // bytes of the op program staged after the frames (0: read from global)
    unsigned char *d_scratch = nullptr;
    size_t scratch_bytes = 0;
    // staging (host-buffer calls)
    void *d_in = nullptr;
    size_t d_in_cap = 0;
    unsigned char *d_out = nullptr;
    size_t d_out_cap = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // last use of the per-handle device scratch (alpha/beta global scratch,
    // single-path channel scratch, adaptive failure queue): every launch
    // waits on it and records it, so kernels of one handle never overlap,
    // whichever streams the calls use (pipelined chunks included)
    cudaEvent_t ev_busy = nullptr;
    bool busy_recorded = false;
    // pipelined host-buffer calls: two internal streams + join events
    cudaStream_t aux[2] = {nullptr, nullptr};
    cudaEvent_t evs = nullptr, evj[2] = {nullptr, nullptr};
    bool timed = false;
    long long launches = 0;
    std::string plan_json;
    // single-path pass (L = 1 decodes, adaptive decoding): k_ssc
    bool ssc_ok = false;
    pb::SscParams ssc{};
    int ssc_grid = 0;
    bool l1_ssc = false;         // route L = 1 decodes through k_ssc
    bool ssc_chg = false;        // k_ssc channel in global scratch
    unsigned char *d_ssc_ch = nullptr;
    int32_t *d_fail = nullptr;   // adaptive: failing frame indices + per-chunk counts
    size_t d_fail_cap = 0;
    int chunk_frames = 0;           // pb_options::chunk_frames
    // lane-per-path list kernel (lane_kernel.cuh), L in 17..32
    bool lane = false;
    pb::lk::LParams *lp = nullptr;  // host copy of the launch parameters (IO fields per call)
    int lane_fpc = 0, lane_grid = 0;  // frames per CTA, CTAs
    int lane_fpw = 1;                 // frames per warp (specialised kernel, list sizes <= 16)
    size_t lane_smem = 0;           // per CTA
    unsigned char *d_lane_scratch = nullptr;
    pb::jit::Kernel *jk = nullptr;  // the lane kernel specialised for this code (jit.cu), or null: generic
    std::string jit_info;           // plan_json fragment about the specialised kernel
    // on-device frame generation: all K info positions, payload syndrome rows
    uint32_t *d_info_all = nullptr, *d_hu = nullptr;
    int crc_w = 0;
    uint32_t gen_crc_const = 0;
};

namespace {

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// options of the handle being created (pb_options, zero = default)
struct Opts {
    int kernel = 0, warps = 0, fps = 0, sync_every = 0, recompute = 0, chunk = 0, grid_sms = 0, l1_list = 0, fuse = 0, specialize = 0, fpw = 0, chg = 0;
};
Opts read_opts(const pb_options *o) {
    Opts r;
    if (!o) return r;
    r.kernel = o->kernel;
    r.warps = o->warps_per_frame;
    r.fps = o->frames_per_sm;
    r.sync_every = o->sync_every;
    r.recompute = o->recompute_stages;
    r.chunk = o->chunk_frames;
    r.grid_sms = o->grid_sms;
    r.l1_list = o->l1_list_kernel;
    // fields added after the first version: present when the caller's struct is long enough
    if (o->size == 0 || o->size >= (int)(offsetof(pb_options, fuse) + sizeof(int32_t))) r.fuse = o->fuse;
    if (o->size == 0 || o->size >= (int)(offsetof(pb_options, specialize) + sizeof(int32_t))) r.specialize = o->specialize;
    if (o->size == 0 || o->size >= (int)(offsetof(pb_options, frames_per_warp) + sizeof(int32_t))) r.fpw = o->frames_per_warp;
    if (o->size == 0 || o->size >= (int)(offsetof(pb_options, channel_global) + sizeof(int32_t))) r.chg = o->channel_global;
    return r;
}
// sync_every (ops, power of two) -> the kernels' barrier mask; dflt = mask
int sync_mask_of(int every, int dflt) {
    if (every < 0) return -1;
    if (every == 0) return dflt;
    int p = 1;
    while (p < every) p <<= 1;
    return p - 1;
}

// grammar walk: node(lo, hi, side) := leaf | F node(lo,mid,0) G node(mid,hi,1) Combine
bool walk(const pb_op *ops, int n_ops, int &pos, int lo, int hi, int side, std::string &err) {
    int size = hi - lo, stage = 0;
    while ((1 << stage) < size) ++stage;
    if (pos >= n_ops) {
        err = "schedule ends early";
        return false;
    }
    const pb_op &op = ops[pos];
    if (op.size != size || op.stage != stage || op.side != side) {
        err = "op " + std::to_string(pos) + " does not match the schedule grammar";
        return false;
    }
    if (op.kind == PB_OP_RATE0 || op.kind == PB_OP_RATE1 || op.kind == PB_OP_REP || op.kind == PB_OP_SPC) {
        if (op.kind == PB_OP_SPC && size < 4) {
            err = "SPC leaf of size " + std::to_string(size) + " (needs >= 4)";
            return false;
        }
        ++pos;
        return true;
    }
    if (op.kind != PB_OP_F || size < 2) {
        err = "op " + std::to_string(pos) + ": expected F or a leaf";
        return false;
    }
    ++pos;
    int mid = lo + size / 2;
    if (!walk(ops, n_ops, pos, lo, mid, 0, err)) return false;
    if (pos >= n_ops || ops[pos].kind != PB_OP_G || ops[pos].size != size || ops[pos].side != side) {
        err = "op " + std::to_string(pos) + ": expected G " + std::to_string(size);
        return false;
    }
    ++pos;
    if (!walk(ops, n_ops, pos, mid, hi, 1, err)) return false;
    if (pos >= n_ops || ops[pos].kind != PB_OP_COMBINE || ops[pos].size != size || ops[pos].side != side) {
        err = "op " + std::to_string(pos) + ": expected Combine " + std::to_string(size);
        return false;
    }
    ++pos;
    return true;
}

int n_cands(int kind, int size, int L) {
    if (kind == PB_OP_RATE0) return 1;
    if (kind == PB_OP_REP || (kind == PB_OP_RATE1 && size == 1)) return 2;
    if (kind == PB_OP_RATE1) return 4;
    return L != 2 ? 8 : 2;  // SPC, listdec.py:387
}

int align_up(int x, int a) { return (x + a - 1) / a * a; }

}  // namespace


// ---- lane-per-path kernel plan (lane_kernel.cuh): lowering + storage.
// Stages n-1 and n-2 are recomputed from the channel by F / G ops (never
// stored); a leaf AT one of those stages reads a staging row in global
// scratch that the F / G before it writes.  Returns false (the interpreted
// kernel is used) when the plan does not fit.
static bool is_leaf_kind(int k) { return k == PB_OP_RATE0 || k == PB_OP_RATE1 || k == PB_OP_REP || k == PB_OP_SPC; }

struct LanePlan {
    pb::lk::LLayout lay{};
    std::vector<pb::lk::LOp> prog;
    int final_op = -1;
};

// Pure host part: storage layout and the lowered program (no device).
static bool lane_lower(int N, int n, int L, int mode, const pb_op *ops, int n_ops, const std::vector<pb::DOp> &dprog,
                       const Opts &opt, LanePlan &out, std::string &why, int G = 1, bool chg = false) {
    using namespace pb::lk;
    (void)L;
    const int es = mode == PB_MODE_F32 ? 4 : 1;
    // measured (c3 L=32): float32 3.09 Gbit/s with n-2 recomputed vs 2.86 stored;
    // int8 3.53 stored vs 2.89 recomputed (small rows, costly conversions)
    const int NV = n >= 2 ? std::max(1, std::min(2, opt.recompute ? opt.recompute : (mode == PB_MODE_F32 ? 2 : 1))) : 1;
    auto virt = [&](int s) { return s < n && s >= n - NV; };
    if ((int)dprog.size() > kMaxOps) {
        why = "op program too long";
        return false;
    }
    // op fusion (pb_options.fuse): bit 0 = leaves read f / g of their parent's row,
    // bit 2 = dead global-scratch stages are discarded from the L2 after their last read
    const int fuse = opt.fuse < 0 ? 0 : (opt.fuse == 0 ? 1 | 4 : opt.fuse);
    // a leaf folds the F / G before it into its reads when that op reads a
    // stored row or the channel (not a recomputed stage)
    auto leaf_fusable = [&](int i) {
        return (fuse & 1) && i + 1 < n_ops && (ops[i].kind == PB_OP_F || ops[i].kind == PB_OP_G) &&
               is_leaf_kind(ops[i + 1].kind) && (ops[i].stage == n || !virt(ops[i].stage));
    };
    bool staged[pb::kMaxLog] = {};
    for (int i = 0; i + 1 < n_ops; ++i)
        if ((ops[i].kind == PB_OP_F || ops[i].kind == PB_OP_G) && virt(ops[i].stage - 1) &&
            is_leaf_kind(ops[i + 1].kind) && !leaf_fusable(i))
            staged[ops[i].stage - 1] = true;
    LLayout lay{};
    const int smem_cap = 227 * 1024;
    const int target_fps = std::max(1, opt.fps ? opt.fps : 16);
    const int budget = smem_cap / target_fps / 16 * 16;
    int off = 0, goff = 0;
    lay.ch_off = 0;
    lay.ch_gl = chg ? 1 : 0;
    if (chg)
        goff = align_up(G * N * es, 256);  // the channels in global scratch (first region)
    else
        off = align_up(G * N * es, 16);  // the warp's G frames' channels, interleaved quad by quad
    lay.asg_off = off;
    off = align_up(off + 32, 8);
    lay.met_off = off;
    off += 256;
    lay.root_off = off;
    off = align_up(off + std::max(1, N / 32) * 4, 16);
    const int b_sm = 6;  // beta slots 0..5 in shared memory (1 word per row)
    for (int s = 0; s < n; ++s) {
        const int words = std::max(1, (1 << s) / 32);
        lay.b_stride[s] = words > 1 ? words + 1 : 1;
        const int bytes = 32 * lay.b_stride[s] * 4;
        if (s < b_sm && off + bytes <= budget) {
            lay.b_off[s] = off;
            off = align_up(off + bytes, 16);
        } else {
            lay.b_gl |= 1u << s;
            lay.b_off[s] = goff;
            goff = align_up(goff + bytes, 128);
        }
    }
    bool spill = false;
    for (int s = 0; s < n; ++s) {
        if (virt(s) && !staged[s]) continue;
        const int bytes = 32 * std::max(4, 1 << s) * es;
        if (!virt(s) && !spill && off + bytes <= budget) {
            lay.a_off[s] = off;
            off = align_up(off + bytes, 16);
        } else {
            if (!virt(s)) spill = true;
            lay.a_gl |= 1u << s;
            lay.a_off[s] = goff;
            goff = align_up(goff + bytes, 256);
        }
    }
    {
        // hard words of Rate-1 / SPC leaves wider than 32 (read back by their survivors)
        int mmax = 0;
        for (int i = 0; i < n_ops; ++i)
            if ((ops[i].kind == PB_OP_RATE1 || ops[i].kind == PB_OP_SPC) && ops[i].size > 32)
                mmax = std::max(mmax, ops[i].size);
        lay.hard_off = goff;
        goff = align_up(goff + (mmax / 32) * 32 * 4, 256);
    }
    lay.smem_bytes = align_up(off, 16);
    lay.gbytes = align_up(goff, 256);
    if (lay.smem_bytes > smem_cap) {
        why = "shared-memory plan too large";
        return false;
    }
    auto src_of = [&](int s) -> uint8_t {
        if (s == n) return S_CH;
        if (s == n - 1) return S_V1;
        if (NV == 2 && s == n - 2) return S_V2;
        return ((lay.a_gl >> s) & 1u) ? S_GL : S_SM;
    };
    // lowering (the interpreted kernel's program gives each leaf's path
    // counts, candidates and Combine chain target)
    std::vector<LOp> prog;
    int di = 0, final_op = -1;
    bool v1g = false, v2g = false;
    uint8_t pend_fuse = 0, pend_src = 0;
    for (int i = 0; i < n_ops; ++i) {
        const pb_op &op = ops[i];
        if (op.kind == PB_OP_COMBINE) continue;
        const pb::DOp &d = dprog[di++];
        if (op.kind == PB_OP_F || op.kind == PB_OP_G) {
            const int s = op.stage;
            const uint8_t flags = (v1g ? LF_V1G : 0) | (v2g ? LF_V2G : 0);
            if (s == n) v1g = op.kind == PB_OP_G;
            if (NV == 2 && s == n - 1) v2g = op.kind == PB_OP_G;
            const bool out_virtual = virt(s - 1);
            if (leaf_fusable(i)) {  // the leaf after it reads f / g of this op's source
                pend_fuse = op.kind == PB_OP_F ? LF_FUSE_F : LF_FUSE_G;
                pend_src = src_of(s);
                continue;
            }
            if (out_virtual && !staged[s - 1]) continue;  // a mode switch only
            if (out_virtual && !(i + 1 < n_ops && is_leaf_kind(ops[i + 1].kind))) continue;
            LOp l{};
            l.kind = op.kind == PB_OP_F ? K_F : K_G;
            l.stage = (uint8_t)s;
            l.pin = l.pout = (uint8_t)d.pin;
            l.src = src_of(s);
            l.aux = ((lay.a_gl >> (s - 1)) & 1u) ? S_GL : S_SM;
            l.flags = flags | ((fuse & 4) && op.kind == PB_OP_G && l.src == S_GL ? LF_LAST : 0);
            prog.push_back(l);
            continue;
        }
        LOp l{};
        l.kind = d.kind == pb::DK_R0 ? K_R0 : d.kind == pb::DK_REP ? K_REP : d.kind == pb::DK_R1 ? K_R1 : K_SPC;
        l.stage = (uint8_t)op.stage;
        l.pin = (uint8_t)d.pin;
        l.pout = (uint8_t)d.pout;
        l.ncand = (uint8_t)(d.kind == pb::DK_R0 ? 0 : d.ncand);
        l.src = pend_fuse ? pend_src : op.stage == n ? S_CH : (virt(op.stage) ? S_GL : src_of(op.stage));
        l.aux = (uint8_t)d.target;
        l.flags = (uint8_t)((d.select ? LF_SELECT : 0) | (v1g ? LF_V1G : 0) | (v2g ? LF_V2G : 0) | pend_fuse);
        // last reader of a global-scratch stage: a leaf reading its own row, or g of its parent's
        if ((fuse & 4) && l.src == S_GL && pend_fuse != LF_FUSE_F) l.flags |= LF_LAST;
        pend_fuse = 0;
        final_op = (int)prog.size();
        prog.push_back(l);
        // skip the Combines the leaf absorbed (the interpreted program did too)
        if (op.side == 1) {
            int j = i + 1;
            while (j < n_ops && ops[j].kind == PB_OP_COMBINE) {
                const int sd = ops[j].side, tg = ops[j].stage;
                ++j;
                if (sd == 0 || tg == n) break;
            }
            i = j - 1;
        }
    }
    if ((int)prog.size() > kMaxOps) {
        why = "op program too long";
        return false;
    }
    out.lay = lay;
    out.prog = prog;
    out.final_op = final_op;
    return true;
}

// The specialised kernel's input (jit.cu) for one code and option set: its own
// lowering (the fusions only the specialised build implements), the frames per
// CTA it is compiled for (its launch bound).  Pure host code, shared by
// pb_create_ex and the device-free pb_jit_source / pb_jit_prebuild.
static const int kLaneSmemCap = 227 * 1024;
static bool make_jit_spec(int N, int n, int k, int L, int mode, int has_crc, uint32_t crc_const, const pb_op *ops,
                          int n_ops, const std::vector<pb::DOp> &dprog, const Opts &opt, pb::jit::Spec &sp,
                          LanePlan &pl, std::string &why) {
    Opts jo = opt;
    // frames per warp (pb_options.frames_per_warp): 32 / pow2(L) frames share a warp's lanes
    int Lp = 1;
    while (Lp < L) Lp <<= 1;
    // shared memory a warp needs at least: its G channels, the fixed tables, beta slots 0..5 and alpha
    // stages 0..4 (the rest of its share goes to the next alpha stages)
    const int es0 = mode == PB_MODE_F32 ? 4 : 1;
    // channels in global scratch (pb_options.channel_global; auto: list sizes <= 16, where the channels of
    // the frames sharing a warp would fill shared memory -- c3 L=2 9.1 -> 27.6, c3 L=8 9.5 -> 14.5, c1 L=4
    // 7.5 -> 12.4, c2 L=8 15.5 -> 17.2, c5 L=16 3.5 (interpreted) -> 5.9 Gbit/s; neutral at L=32)
    const bool chg = opt.chg > 0 || (opt.chg == 0 && L <= 16);
    auto need = [&](int g) { return (chg ? 0 : g * N * es0) + 1024 + 6 * 132 + 32 * (4 + 4 + 4 + 8 + 16) * es0; };
    int G = opt.fpw > 1 ? std::min(opt.fpw, 32 / Lp) : 1;
    if (opt.fpw == 0 && L <= 16) {
        // auto: every lane a path slot, but at least three warps per SM (measured, Gbit/s: c3 L=2 16 frames
        // per warp = 1 warp per SM 5.3, 8 = 3 warps 8.9; c3 L=8 4 frames 8.9, 2 frames 8.2; c2 L=8 4 frames
        // 13.6, 2 frames 9.7; c1 L=4 8 frames 7.1, 4 frames 6.9)
        G = 32 / Lp;
        while (G > 1 && kLaneSmemCap / need(G) < 3) G >>= 1;
        // long codes: the channels leave room for too few frames (c5 N=8192 L=16: 6 frames per SM,
        // 2.7 Gbit/s against the interpreted kernel's 3.4): stay with the interpreted kernel
        if (G * std::min(16, kLaneSmemCap / need(G)) < 16) {
            why = "too few resident frames per SM for the lane kernel at this block length";
            return false;
        }
    }
    while (G & (G - 1)) G &= G - 1;  // a power of two
    if (G > 1) jo.fps = std::max(1, std::min(opt.fps ? opt.fps : 16, kLaneSmemCap / need(G)));
    if (!lane_lower(N, n, L, mode, ops, n_ops, dprog, jo, pl, why, G, chg)) return false;
    sp.G = G;
    const int fps = std::max(1, std::min(32, jo.fps ? jo.fps : 16));
    sp.N = N, sp.n = n, sp.k = k, sp.L = L, sp.mode = mode;
    sp.has_crc = has_crc, sp.crc_const = crc_const;
    sp.lay = pl.lay, sp.prog = pl.prog, sp.final_op = pl.final_op;
    // auto / 1: everything compile-time, unrolled chains, wide-leaf scans pipelined over 2-quad blocks
    // (c3 L=32: 4.61 -> 4.65 Gbit/s; 4-quad blocks 4.62); other values: explicit policy bits (jit.h)
    sp.policy = opt.specialize <= 1 ? (pb::jit::POL_FULL | pb::jit::POL_SCAN_PIPE2) : opt.specialize;
    // survivor hand-over: unrolled with static key indices (c3 L=32 4.67 -> 4.96, int8 5.11 -> 5.67, c2 L=8
    // 13.9 -> 15.3 Gbit/s: no local-memory round trip), except at L = 2 where the loop over the set bits
    // measured faster (c3 L=2 8.9 against 7.5)
    if (opt.specialize <= 1 && L <= 2) sp.policy |= pb::jit::POL_ASG_LOOP;
    sp.fpc = std::max(1, std::min(fps, kLaneSmemCap / std::max(16, pl.lay.smem_bytes)));
    return true;
}

static bool plan_lane(pb_handle *h, const pb_op *ops, int n_ops, const std::vector<pb::DOp> &dprog, const Opts &opt,
                      std::string &why) {
    using namespace pb::lk;
    const int N = h->N, n = h->n, L = h->L, mode = h->mode;
    LanePlan pl;
    int fpc = 0, bps = 0, nvar = 0;
    std::vector<uint16_t> vid;
    std::string jit_err = "not requested";
    // ---- the kernel specialised for this code (jit.cu) ...
    if (opt.specialize >= 0) {
        pb::jit::Spec sp;
        LanePlan jp;
        std::string jwhy;
        if (make_jit_spec(N, n, h->k, L, mode, h->base.has_crc, h->base.crc_const, ops, n_ops, dprog, opt, sp, jp,
                          jwhy)) {
            const std::string src = pb::jit::generate(sp, vid, &nvar);
            bool hit = false;
            double secs = 0.0;
            h->jk = pb::jit::acquire(src, true, h->device, jit_err, &hit, &secs);
            if (h->jk && pb::jit::occupancy(h->jk, 32 * sp.fpc, (size_t)sp.fpc * jp.lay.smem_bytes) >= 1) {
                pl = jp;
                fpc = sp.fpc;
                bps = 1;
                h->lane_fpw = sp.G;
                char jb[512];
                snprintf(jb, sizeof jb, "\"specialised\": {\"variants\": %d, \"registers\": %d, \"cache_hit\": %s, "
                         "\"compile_s\": %.1f}", nvar, pb::jit::registers(h->jk), hit ? "true" : "false", secs);
                h->jit_info = jb;
            } else {
                if (h->jk) jit_err = "the specialised kernel does not fit one CTA per SM";
                pb::jit::release(h->jk);
                h->jk = nullptr;
            }
        } else {
            jit_err = jwhy;
        }
        if (!h->jk && opt.specialize > 0) {
            why = "specialised kernel unavailable: " + jit_err;
            return false;
        }
    }
    // ---- ... or the generic kernel (compiled for 16 frames per CTA, one frame per warp)
    if (!h->jk && L <= 16 && opt.kernel != 2) {
        why = "list size <= 16 without the specialised kernel: " + jit_err;
        return false;
    }
    if (!h->jk) {
        Opts go = opt;
        go.fps = std::min(16, opt.fps ? opt.fps : 16);
        if (!lane_lower(N, n, L, mode, ops, n_ops, dprog, go, pl, why)) return false;
        fpc = std::min(go.fps, kLaneSmemCap / std::max(16, pl.lay.smem_bytes));
        while (fpc >= 1) {
            if (pb_lane_occupancy(mode, (size_t)fpc * pl.lay.smem_bytes, fpc, &bps) == cudaSuccess && bps >= 1) break;
            cudaGetLastError();
            --fpc;
        }
        if (fpc < 1) {
            why = "no resident CTA";
            return false;
        }
        std::string e2;
        for (char c : jit_err.substr(0, 300)) e2 += (c == '"' || c == '\\' || c == '\n') ? ' ' : c;
        h->jit_info = "\"specialised\": null, \"specialised_why\": \"" + e2 + "\"";
    }
    const LLayout &lay = pl.lay;
    LParams *lp = new LParams();
    std::memset(lp, 0, sizeof(LParams));
    lp->xsyn4 = h->d_xsyn4;
    lp->info_pos = h->d_info;
    lp->N = N;
    lp->n = n;
    lp->k = h->k;
    lp->L = L;
    lp->has_crc = h->base.has_crc;
    lp->crc_const = h->base.crc_const;
    lp->n_ops = (int)pl.prog.size();
    lp->final_op = pl.final_op;
    lp->fpc = fpc;
    // CTA regroup period in ops.  Generic kernel: every 8 (measured c3 L=32: every 8 3.23, 32 3.09,
    // 4 3.12, never 2.46 Gbit/s); the specialised kernel has fewer, longer ops: every 32 (every 4
    // 4.19, 8 4.31, 16 4.42, 32 4.48, never 3.98 Gbit/s)
    lp->sync_mask = fpc > 1 ? sync_mask_of(opt.sync_every, h->jk ? 31 : 7) : -1;
    lp->lay = lay;
    std::copy(pl.prog.begin(), pl.prog.end(), lp->prog);
    if (h->jk) std::copy(vid.begin(), vid.end(), lp->vid);
    h->lp = lp;
    h->lane_fpc = fpc * h->lane_fpw;  // frames per CTA
    h->lane_grid = h->sms * bps;
    h->lane_smem = (size_t)fpc * lay.smem_bytes;
    if (lay.gbytes) {
        cudaError_t e = cudaMalloc(&h->d_lane_scratch, (size_t)h->lane_grid * fpc * lay.gbytes);  // per warp
        if (e != cudaSuccess) {
            cudaGetLastError();
            delete lp;
            h->lp = nullptr;
            pb::jit::release(h->jk);
            h->jk = nullptr;
            why = "scratch allocation failed";
            return false;
        }
    }
    lp->gscratch = h->d_lane_scratch;
    h->lane = true;
    return true;
}

// CRC syndrome rows per u position (affine map of codes.py:127-156) and the
// constant a passing codeword's syndrome equals.  Pure host code.
static void crc_rows(const pb_code *code, const std::vector<int> &info, int N, std::vector<uint32_t> &Hu,
                     uint32_t &crc_const) {
    const int w = code->crc_width;
    Hu.assign(N, 0u);
    crc_const = 0;
    if (w) {
        Crc crc{w, code->crc_poly, code->crc_init, code->crc_xor_out, code->crc_reflect != 0};
        const int k = code->k;
        uint32_t v = crc.step(0u, 1);  // injection of one input bit
        for (int j = k - 1; j >= 0; --j) {
            Hu[info[j]] = crc.append_word(v);
            v = crc.step(v, 0);
        }
        uint32_t reg = crc.start();
        for (int j = 0; j < k; ++j) reg = crc.step(reg, 0);
        crc_const = crc.append_word(reg ^ crc.xor_out);
        for (int j = 0; j < w; ++j) Hu[info[k + j]] = 1u << j;
    }

}

// Lower the reference's op list (schedule.py:44-58) to the device program:
// Combines are absorbed by the leaf before them, every op carries its path
// counts.  Pure host code (no device).
static bool lower_program(const pb_op *ops, int n_ops, int n, int L, std::vector<pb::DOp> &prog, int &final_op,
                          int &max_hard, std::string &err) {
    int P = 1, vstate = pb::VM_F, leaf_off = 0;
    final_op = -1;
    max_hard = 1;
    for (int i = 0; i < n_ops; ++i) {
        const pb_op &op = ops[i];
        pb::DOp d{};
        if (op.kind == PB_OP_F || op.kind == PB_OP_G) {
            if (op.stage == n) {
                vstate = op.kind == PB_OP_F ? pb::VM_F : pb::VM_G;
                d.kind = pb::DK_NOP;
            } else {
                d.kind = op.kind == PB_OP_F ? pb::DK_F : pb::DK_G;
                d.vmode = op.stage == n - 1 ? (int8_t)vstate : (int8_t)pb::VM_NONE;
            }
            d.stage = (int8_t)op.stage;
            d.pin = (int8_t)P;
            d.pout = (int8_t)P;
            prog.push_back(d);
            continue;
        }
        if (op.kind == PB_OP_COMBINE) {
            err = "invalid schedule: Combine not preceded by a right-child leaf";
            return false;
        }
        const int t = op.stage, m = op.size;
        const int C = n_cands(op.kind, m, L);
        d.kind = op.kind == PB_OP_RATE0 ? pb::DK_R0
                 : op.kind == PB_OP_REP ? pb::DK_REP
                 : op.kind == PB_OP_RATE1 ? pb::DK_R1
                                          : pb::DK_SPC;
        d.stage = (int8_t)t;
        d.pin = (int8_t)P;
        d.ncand = (int8_t)C;
        const int pout = op.kind == PB_OP_RATE0 ? P : std::min(L, P * C);
        d.pout = (int8_t)pout;
        d.select = (int8_t)(op.kind != PB_OP_RATE0 && P * C > L);
        d.vmode = t == n - 1 ? (int8_t)vstate : (int8_t)pb::VM_NONE;
        d.off = leaf_off;
        if ((op.kind == PB_OP_RATE1 && m > 1) || op.kind == PB_OP_SPC) max_hard = std::max(max_hard, m);
        // chain of Combines absorbed by this leaf
        int target = t;
        if (op.side == 1) {
            int j = i + 1;
            for (;;) {
                if (j >= n_ops || ops[j].kind != PB_OP_COMBINE || ops[j].stage != target + 1) {
                    err = "invalid schedule: broken Combine chain";
                    return false;
                }
                target = ops[j].stage;
                int sd = ops[j].side;
                ++j;
                if (sd == 0 || target == n) break;
            }
            i = j - 1;
        }
        d.target = (int8_t)target;
        leaf_off += m;
        P = pout;
        final_op = (int)prog.size();
        prog.push_back(d);
    }
    return true;
}

extern "C" {

const char *pb_last_error(void) { return g_err.c_str(); }
int pb_version(void) { return PB_API_VERSION; }

int pb_create(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode, int device,
              pb_handle **out) {
    return pb_create_ex(code, ops, n_ops, list_size, mode, device, nullptr, out);
}

int pb_create_ex(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode, int device,
                 const pb_options *opts, pb_handle **out) {
    g_err.clear();
    const Opts opt = read_opts(opts);
    if (opt.kernel < 0 || opt.kernel > 2) return fail(PB_EINVAL, "pb_options.kernel must be 0, 1 or 2");
    if (opt.warps != 0 && opt.warps != 1 && opt.warps != 2 && opt.warps != 4 && opt.warps != 8)
        return fail(PB_EINVAL, "pb_options.warps_per_frame must be 1, 2, 4 or 8");
    if (opt.recompute < 0 || opt.recompute > 2) return fail(PB_EINVAL, "pb_options.recompute_stages must be 0, 1 or 2");
    if (!out || !code || !ops) return fail(PB_EINVAL, "null argument");
    *out = nullptr;
    if (list_size < 1) return fail(PB_EINVAL, "list size " + std::to_string(list_size) + " must be >= 1");
    if (list_size > pb::kMaxL)
        return fail(PB_EINVAL, "list size " + std::to_string(list_size) + " exceeds the supported maximum 32");
    if (mode != PB_MODE_F32 && mode != PB_MODE_INT8) return fail(PB_EINVAL, "unknown mode");
    const int N = code->N;
    if (N < 2 || (N & (N - 1)) || N > (1 << pb::kMaxLog))
        return fail(PB_EINVAL, "block length " + std::to_string(N) + " is not a power of two in [2, 65536]");
    int n = 0;
    while ((1 << n) < N) ++n;
    if (!code->frozen_mask) return fail(PB_EINVAL, "frozen mask missing");
    const int w = code->crc_width;
    if (w != 0 && w != 8 && w != 16 && w != 32) return fail(PB_EINVAL, "unsupported CRC width");
    std::vector<int> info;
    for (int i = 0; i < N; ++i)
        if (!code->frozen_mask[i]) info.push_back(i);
    if (code->k < 1 || code->k + w != (int)info.size())
        return fail(PB_EINVAL, "payload + CRC does not match the unfrozen positions");
    {
        int pos = 0;
        std::string err;
        if (!walk(ops, n_ops, pos, 0, N, 0, err)) return fail(PB_EINVAL, "invalid schedule: " + err);
        if (pos != n_ops) return fail(PB_EINVAL, "invalid schedule: trailing ops");
    }

    pb_handle *h = new pb_handle();
    h->chunk_frames = opt.chunk;
    h->device = device;
    h->mode = mode;
    h->L = list_size;
    h->N = N;
    h->n = n;
    h->k = code->k;
    const int L = list_size;

    // ---- CRC syndrome rows per u position
    std::vector<uint32_t> Hu;
    uint32_t crc_const = 0;
    crc_rows(code, info, N, Hu, crc_const);

    // ---- lower the schedule
    int final_op = -1, max_hard = 1;
    {
        std::string err;
        if (!lower_program(ops, n_ops, n, L, h->prog, final_op, max_hard, err)) {
            delete h;
            return fail(PB_EINVAL, err);
        }
    }
    // ---- storage plan
    const int es = mode == PB_MODE_F32 ? 4 : 1;
    // frame shape: W warps per frame, PPW (power of two) path slots per warp
    int warps = opt.warps ? opt.warps : 1;
    auto shape_ppw = [&](int wv) {
        int p = 1;
        while (p * wv < L) p <<= 1;
        return p;
    };
    if (!pb_shape_supported(mode, warps, shape_ppw(warps), 0)) warps = 1;
    int ppw = shape_ppw(warps), lppw = 0;
    while ((1 << lppw) < ppw) ++lppw;
    const int rows = ppw * warps;  // alpha rows, padded to whole interleave blocks
    h->ppw = ppw;
    h->warps = warps;
    // lanes per path of each op's input / output path count (one warp per frame)
    for (pb::DOp &d : h->prog) {
        auto lg = [&](int np) {
            const int act = std::max(1, std::min(np, ppw));
            int c = 0;
            while ((1 << c) < act) ++c;
            return (int8_t)(5 - c);
        };
        d.lgi = lg(d.pin);
        d.lgo = lg(d.pout);
    }
    const int smem_cap = 227 * 1024;
    // resident frames per SM: one warp each, up to the launch bound
    const int target_fps = std::max(1, opt.fps ? opt.fps : pb::shape_max_threads(warps, ppw) / 32);
    // Per-frame layout for a channel in shared memory or in global scratch.
    auto plan_layout = [&](bool chg, pb::FrameLayout &lay) {
        lay = pb::FrameLayout{};
        int off = 0, goff = 0;
        lay.ch_off = 0;
        if (chg)
            goff = align_up(N * es, 256);  // global scratch, before the global alpha stages
        else
            off = align_up(N * es, 16);
        // beta slots: the top ones (largest) may go to global scratch
        // (PB_BETA_GLOBAL_FROM) to leave shared memory to more frames
        // (measured: slots >= 6 global for c3 / c5 / int8 at 16 frames per SM;
        // the freed shared memory also grows the L1 that caches the global rows)
        lay.b_gfrom = std::min(n, 6);
        for (int s = 0; s < n; ++s) {
            int words = std::max(1, (1 << s) / 32);
            lay.b_stride[s] = words > 1 ? words + 1 : 1;
            if (s >= lay.b_gfrom) {
                lay.b_off[s] = goff;
                goff = align_up(goff + L * lay.b_stride[s] * 4, 256);
            } else {
                lay.b_off[s] = off;
                off = align_up(off + L * lay.b_stride[s] * 4, 16);
            }
        }
        // per-path arrays: stride `rows` (= PPW * W >= L, compile-time in the
        // kernel), index vectors (kMaxLog + 3) / 4 words per path
        const int iw = (pb::kMaxLog + 3) / 4;
        lay.pm_off = off;
        off = align_up(off + 2 * rows * 8, 16);
        lay.idx_stride = std::max(1, (n + 3) / 4);  // index words in use per path (4 stages per word)
        lay.ia_off = off;
        off = align_up(off + 2 * rows * iw * 4, 16);
        lay.ib_off = off;
        off = align_up(off + 2 * rows * iw * 4, 16);
        const int nbuf = warps > 1 ? 2 : 1;  // candidate buffers (by leaf parity across warps)
        lay.cd_off = off;
        off = align_up(off + nbuf * rows * pb::kMaxCand * 8, 16);
        lay.clrb_off = off;
        off = align_up(off + nbuf * rows * 4 * 2, 16);
        lay.cflag_off = off;
        off = align_up(off + nbuf * rows, 16);
        lay.asg_off = off;
        off = align_up(off + nbuf * 2 * rows, 16);
        lay.hard_words = std::max(1, max_hard / 32);
        lay.hard_off = off;
        off = align_up(off + nbuf * rows * lay.hard_words * 4, 16);
        lay.root_words = std::max(1, N / 32);
        lay.root_off = off;
        off = align_up(off + lay.root_words * 4, 16);

        const int budget = std::max(off, smem_cap / target_fps - 1024);
        // alpha stages s = 0 .. n-2 (n-1 is recomputed), lowest stages first into
        // shared memory, the rest into per-frame global scratch (L2-resident)
        int s_global = n - 1;
        // quad-interleaved rows: at least one quad (4 elements) per row
        for (int s = 0; s <= n - 2; ++s) {
            int bytes = align_up(rows * std::max(4, 1 << s) * es, 16);
            if (off + bytes > budget) {
                s_global = s;
                break;
            }
            lay.a_off[s] = off;
            off += bytes;
        }
        lay.a_gfrom = s_global;
        for (int s = s_global; s <= n - 2; ++s) {
            lay.a_off[s] = goff;
            goff = align_up(goff + rows * std::max(4, 1 << s) * es, 256);
        }
        lay.gbytes = goff;
        lay.smem_bytes = align_up(off, 16);
    };
    // The channel moves to global scratch (L1/L2; it is read only by the
    // stage n-1 ops) when that buys more frames per SM or keeps more alpha
    // stages in shared memory; int8 channels are small and stay.
    pb::FrameLayout &lay = h->base.lay;
    {
        pb::FrameLayout ls, lg;
        plan_layout(false, ls);
        plan_layout(true, lg);
        auto fps_of = [&](const pb::FrameLayout &l) { return std::min(target_fps, smem_cap / std::max(1, l.smem_bytes)); };
        bool chg = fps_of(lg) > fps_of(ls) || (fps_of(lg) == fps_of(ls) && lg.a_gfrom > ls.a_gfrom);
        chg = chg && pb_shape_supported(mode, warps, ppw, 1);
        h->chg = chg;
        lay = chg ? lg : ls;
    }
    if (lay.smem_bytes > smem_cap) {
        delete h;
        return fail(PB_EINVAL, "code too large for the per-frame shared-memory plan (" +
                                   std::to_string(lay.smem_bytes) + " bytes)");
    }
    h->smem_frame = lay.smem_bytes;
    // A leaf reads f / g of its parent's rows directly when those are in
    // shared memory (PB_FUSE_LEAF; int8 only, the kernels compile it for the
    // int8 shapes alone): the F / G before it (the one that would store the
    // leaf's LLRs) is skipped -- one op, one row store and one row load fewer
    // per leaf.  Stage n-1 parents are recomputed from the channel and
    // global-scratch parents keep their F / G.
    if (mode == PB_MODE_INT8) {
        for (size_t i = 1; i < h->prog.size(); ++i) {
            pb::DOp &d = h->prog[i], &pf = h->prog[i - 1];
            const bool leaf = d.kind == pb::DK_R0 || d.kind == pb::DK_REP || d.kind == pb::DK_R1 || d.kind == pb::DK_SPC;
            const bool fg = pf.kind == pb::DK_F || pf.kind == pb::DK_G;
            const int ps = d.stage + 1;
            if (leaf && fg && pf.stage == ps && ps <= n - 2 && ps < lay.a_gfrom && pf.pin == d.pin) {
                pf.fuse = -1;
                d.fuse = pf.kind == pb::DK_F ? 1 : 2;
            }
        }
    }

    {
        // host-side launch parameters (device pointers are filled in below)
        pb::Params &pr = h->base;
        pr.N = N;
        pr.n = n;
        pr.k = code->k;
        pr.L = L;
        pr.ppw = ppw;
        pr.lppw = lppw;
        pr.has_crc = w != 0;
        pr.crc_const = crc_const;
        pr.final_op = final_op;
        pr.n_ops = (int)h->prog.size();
        pr.fpc = 1;
        pr.sync_mask = -1;
        pr.prog_smem = 0;
        // measured (same-box A/B): +3 % c3 L=32, +4 % c5 L=16, +1 % int8
        // L=32 over a global-memory program; -4 % at 8 paths per warp (c3 L=8)
        pr.prog_inline = (int)h->prog.size() <= pb::kInlineOps && ppw >= 16;
        if (pr.prog_inline) std::copy(h->prog.begin(), h->prog.end(), pr.iprog);
    }
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        delete h;
        return cuda_fail(e, "cudaSetDevice");
    }
    cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, device);
    if (opt.grid_sms > 0) h->sms = std::min(h->sms, opt.grid_sms);
    e = pb_occupancy(mode, h->warps, h->ppw, h->chg, h->smem_frame, 1, &h->blocks_per_sm);
    if (e != cudaSuccess || h->blocks_per_sm < 1) {
        delete h;
        return cuda_fail(e == cudaSuccess ? cudaErrorInvalidConfiguration : e, "occupancy");
    }
    // Every frame resident on an SM goes into one CTA (frames per CTA = frames
    // per SM).  The frames run the same op program and start together, so the
    // SM's warps stay close in the code and share instruction fetch; one CTA
    // per frame lets them drift apart over the batch and thrash the I-cache
    // (measured: no_instructions stalls 8.7% -> 16.5%, -25% throughput).
    // (A CTA barrier after every op to force lockstep measured slower.)
    {
        int fpc = std::min(h->blocks_per_sm, pb::shape_max_threads(h->warps, h->ppw) / 32 / h->warps);  // launch bound
        while (fpc > 1 && (size_t)fpc * h->smem_frame > (size_t)smem_cap) --fpc;
        int bps = 0;
        while (fpc > 1) {
            e = pb_occupancy(mode, h->warps, h->ppw, h->chg, fpc * h->smem_frame, fpc, &bps);
            if (e == cudaSuccess && bps >= 1) break;
            --fpc;
        }
        if (fpc == 1) bps = h->blocks_per_sm;
        h->fpc = fpc;
        h->blocks_per_sm = bps;
    }
    h->grid = h->sms * h->blocks_per_sm;
    // (the op program is read through L1 / the constant bank; staging it in
    // shared memory measured neutral at L=32 and -10 % at L=8)

    // ---- single-path pass plan (k_ssc): one warp per frame, up to
    // PB_SSC_MAXT/32 frames per CTA; the channel goes to global scratch when
    // that fits more frames (shared memory holds alpha, beta, codeword)
    {
        pb::SscLayout &sl = h->ssc.lay;
        auto plan = [&](bool chg) {
            int off = 0;
            sl.ch_off = 0;
            off = chg ? 0 : align_up(N * es, 16);
            for (int s = 0; s <= n - 2; ++s) {
                sl.a_off[s] = off;
                off = align_up(off + (1 << s) * es, 16);
            }
            for (int s = 0; s < n; ++s) {
                sl.b_off[s] = off;
                off = align_up(off + std::max(1, (1 << s) / 32) * 4, 16);
            }
            sl.root_off = off;
            off = align_up(off + std::max(1, N / 32) * 4, 16);
            sl.smem_bytes = off;
            return off;
        };
        const int maxf = PB_SSC_MAXT / 32;
        const int fs = plan(false), fg = plan(true);
        const bool chg = std::min(maxf, smem_cap / std::max(1, fg)) > std::min(maxf, smem_cap / std::max(1, fs));
        const int off = plan(chg);
        int sfpc = std::min(maxf, smem_cap / std::max(1, off));
        int bps = 0;
        while (sfpc >= 1) {
            if (pb_occupancy_ssc(mode, sfpc, off, &bps) == cudaSuccess && bps >= 1) break;
            --sfpc;
        }
        cudaGetLastError();
        if (sfpc >= 1 && bps >= 1) {
            h->ssc_ok = true;
            h->ssc.fpc = sfpc;
            h->ssc_grid = h->sms * bps;
            h->ssc_chg = chg;
        }
        h->l1_ssc = h->ssc_ok && L == 1 && !opt.l1_list;
    }

    // ---- device tables
    if ((e = cudaMalloc(&h->d_prog, sizeof(pb::DOp) * h->prog.size())) != cudaSuccess ||
        (e = cudaMalloc(&h->d_xsyn4, sizeof(uint32_t) * 128 * std::max(1, N / 32))) != cudaSuccess ||
        (e = cudaMalloc(&h->d_info, sizeof(uint32_t) * std::max(1, code->k))) != cudaSuccess) {
        pb_destroy(h);
        return cuda_fail(e, "cudaMalloc tables");
    }
    std::vector<uint32_t> info_k(info.begin(), info.begin() + code->k);
    {
        std::vector<uint32_t> all(info.begin(), info.end()), hu(code->k);
        for (int j = 0; j < code->k; ++j) hu[j] = Hu[info[j]];
        if ((e = cudaMalloc(&h->d_info_all, sizeof(uint32_t) * all.size())) != cudaSuccess ||
            (e = cudaMalloc(&h->d_hu, sizeof(uint32_t) * std::max<size_t>(1, hu.size()))) != cudaSuccess) {
            pb_destroy(h);
            return cuda_fail(e, "cudaMalloc generator tables");
        }
        cudaMemcpy(h->d_info_all, all.data(), sizeof(uint32_t) * all.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(h->d_hu, hu.data(), sizeof(uint32_t) * hu.size(), cudaMemcpyHostToDevice);
        h->crc_w = w;
        h->gen_crc_const = crc_const;
    }
    cudaMemcpy(h->d_prog, h->prog.data(), sizeof(pb::DOp) * h->prog.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(h->d_info, info_k.data(), sizeof(uint32_t) * code->k, cudaMemcpyHostToDevice);
    {
        // codeword-domain syndrome rows Hx[j] = XOR_{i subset of j} Hu[i]
        // (x = u G_N, G_N[j][i] = 1 iff i subset of j), as nibble tables per
        // 32-bit codeword word: T[w][nb][v] = XOR of Hx[32 w + 4 nb + b], b in v
        std::vector<uint32_t> Hx = Hu;
        for (int hb = 1; hb < N; hb <<= 1)
            for (int j = 0; j < N; ++j)
                if (j & hb) Hx[j] ^= Hx[j ^ hb];
        const int nw = std::max(1, N / 32);
        std::vector<uint32_t> T((size_t)nw * 128, 0u);
        for (int wi = 0; wi < nw; ++wi)
            for (int nb = 0; nb < 8; ++nb)
                for (int v = 0; v < 16; ++v)
                    for (int b = 0; b < 4; ++b) {
                        const int j = 32 * wi + 4 * nb + b;
                        if (((v >> b) & 1) && j < N) T[(size_t)wi * 128 + nb * 16 + v] ^= Hx[j];
                    }
        cudaMemcpy(h->d_xsyn4, T.data(), sizeof(uint32_t) * T.size(), cudaMemcpyHostToDevice);
    }
    if (lay.gbytes) {
        h->scratch_bytes = (size_t)h->grid * h->fpc * lay.gbytes;
        if ((e = cudaMalloc(&h->d_scratch, h->scratch_bytes)) != cudaSuccess) {
            pb_destroy(h);
            return cuda_fail(e, "cudaMalloc scratch");
        }
    }
    if (h->ssc_ok && h->ssc_chg) {
        if ((e = cudaMalloc(&h->d_ssc_ch, (size_t)h->ssc_grid * h->ssc.fpc * N * es)) != cudaSuccess) {
            pb_destroy(h);
            return cuda_fail(e, "cudaMalloc single-path channel scratch");
        }
    }
    cudaEventCreate(&h->ev0);
    cudaEventCreate(&h->ev1);

    pb::Params &pr = h->base;
    pr.prog = h->d_prog;
    pr.n_ops = (int)h->prog.size();
    pr.xsyn4 = h->d_xsyn4;
    pr.info_pos = h->d_info;
    pr.N = N;
    pr.n = n;
    pr.k = code->k;
    pr.L = L;
    pr.ppw = ppw;
    pr.lppw = lppw;
    pr.has_crc = w != 0;
    pr.crc_const = crc_const;
    pr.final_op = final_op;
    pr.gscratch = h->d_scratch;
    pr.op_cycles = nullptr;
    pr.ablate = 0;
    pr.fpc = h->fpc;
    pr.prog_smem = h->prog_smem ? 1 : 0;
    // The CTA's frames drift apart op by op (data-dependent selection and
    // memory latencies) and then miss in the instruction cache separately; a
    // CTA barrier every 32 ops regroups them.  Measured: +30% for L >= 16
    // (c3 L=32 1.40 -> 1.82, int8 1.51 -> 1.99, c5 1.48 -> 1.93 Gbit/s), a
    // slight loss for the short per-op code of L <= 8.
    pr.sync_mask = h->fpc > 1 ? sync_mask_of(opt.sync_every, h->ppw * h->warps >= 16 ? 31 : -1) : -1;

    {
        pb::SscParams &sp = h->ssc;
        sp.prog = h->d_prog;
        sp.n_ops = (int)h->prog.size();
        sp.xsyn4 = h->d_xsyn4;
        sp.info_pos = h->d_info;
        sp.N = N;
        sp.n = n;
        sp.k = code->k;
        sp.has_crc = w != 0;
        sp.crc_const = crc_const;
        sp.gch = h->d_ssc_ch;
    }

    std::string lane_why = "list size <= 16";
    if (opt.kernel == 1) {
        lane_why = "interpreted kernel requested";
    } else if ((L > 16 || opt.kernel == 2 || (opt.fpw != 1 && opt.fpw >= 0 && opt.specialize >= 0 && L > 1)) &&
               h->warps == 1 && opt.warps <= 1) {
        plan_lane(h, ops, n_ops, h->prog, opt, lane_why);
    } else if (h->warps != 1) {
        lane_why = "several warps per frame requested";
    }
    if (!h->lane && opt.specialize > 0 && lane_why.rfind("specialised kernel unavailable", 0) == 0) {
        const std::string why = lane_why;
        pb_destroy(h);
        return fail(PB_ECUDA, why);
    }
    if (opt.kernel == 2 && !h->lane) {
        const std::string why = lane_why;
        pb_destroy(h);
        return fail(PB_EINVAL, "lane-per-path kernel unavailable: " + why);
    }

    char buf[1024];
    snprintf(buf, sizeof buf,
             "{\"N\": %d, \"k\": %d, \"L\": %d, \"mode\": \"%s\", \"ops\": %d, \"device_ops\": %d, "
             "\"smem_per_frame\": %d, \"alpha_global_from_stage\": %d, \"global_scratch_per_frame\": %d, "
             "\"frames_per_sm\": %d, \"sms\": %d, \"grid\": %d, \"block\": %d, \"warps_per_frame\": %d, "
             "\"paths_per_warp\": %d, \"frames_per_cta\": %d, \"channel_in_global\": %d, "
             "\"ssc\": {\"smem_per_frame\": %d, \"frames_per_cta\": %d, \"grid\": %d, \"l1_decodes\": %d, \"channel_in_global\": %d}}",
             N, code->k, L, mode == PB_MODE_F32 ? "f32" : "int8", n_ops, (int)h->prog.size(),
             lay.smem_bytes, lay.a_gfrom, lay.gbytes, h->blocks_per_sm * h->fpc, h->sms, h->grid,
             32 * h->warps * h->fpc, h->warps, h->ppw, h->fpc, (int)h->chg, h->ssc.lay.smem_bytes,
             h->ssc_ok ? h->ssc.fpc : 0, h->ssc_grid, (int)h->l1_ssc, (int)h->ssc_chg);
    h->plan_json = buf;
    if (h->plan_json.size() > 1) {
        char lb[512];
        if (h->lane)
            snprintf(lb, sizeof lb,
                     ", \"lane_kernel\": {\"ops\": %d, \"smem_per_frame\": %d, \"global_scratch_per_frame\": %d, "
                     "\"frames_per_cta\": %d, \"frames_per_warp\": %d, \"grid\": %d, \"alpha_global_mask\": %u, "
                     "\"beta_global_mask\": %u, ",
                     h->lp->n_ops, h->lp->lay.smem_bytes, h->lp->lay.gbytes, h->lane_fpc, h->lane_fpw, h->lane_grid,
                     h->lp->lay.a_gl, h->lp->lay.b_gl);
        else
            snprintf(lb, sizeof lb, ", \"lane_kernel\": null, \"lane_kernel_why\": \"%s\"}", lane_why.c_str());
        h->plan_json.pop_back();
        h->plan_json += lb;
        if (h->lane) h->plan_json += h->jit_info + "}}";
    }
    *out = h;
    return PB_OK;
}

// ---- the specialised lane kernel without a device: its generated source
// (tests, inspection) and a cache prebuild (build step; NVRTC needs no GPU)
static int jit_spec_of(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                       const pb_options *opts, pb::jit::Spec &sp) {
    const Opts opt = read_opts(opts);
    if (!code || !ops || !code->frozen_mask) return fail(PB_EINVAL, "null argument");
    if (list_size < 1 || list_size > pb::kMaxL) return fail(PB_EINVAL, "list size out of range");
    if (mode != PB_MODE_F32 && mode != PB_MODE_INT8) return fail(PB_EINVAL, "unknown mode");
    const int N = code->N;
    if (N < 2 || (N & (N - 1)) || N > (1 << pb::kMaxLog)) return fail(PB_EINVAL, "bad block length");
    int n = 0;
    while ((1 << n) < N) ++n;
    std::vector<int> info;
    for (int i = 0; i < N; ++i)
        if (!code->frozen_mask[i]) info.push_back(i);
    if (code->k < 1 || code->k + code->crc_width != (int)info.size())
        return fail(PB_EINVAL, "payload + CRC does not match the unfrozen positions");
    {
        int pos = 0;
        std::string err;
        if (!walk(ops, n_ops, pos, 0, N, 0, err) || pos != n_ops) return fail(PB_EINVAL, "invalid schedule: " + err);
    }
    std::vector<uint32_t> Hu;
    uint32_t crc_const = 0;
    crc_rows(code, info, N, Hu, crc_const);
    std::vector<pb::DOp> dprog;
    int final_op = -1, max_hard = 1;
    std::string err;
    if (!lower_program(ops, n_ops, n, list_size, dprog, final_op, max_hard, err)) return fail(PB_EINVAL, err);
    LanePlan pl;
    if (!make_jit_spec(N, n, code->k, list_size, mode, code->crc_width != 0, crc_const, ops, n_ops, dprog, opt, sp, pl,
                       err))
        return fail(PB_EINVAL, "lane-per-path kernel unavailable: " + err);
    return PB_OK;
}

int pb_jit_source(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                  const pb_options *opts, char *buf, int64_t cap, int64_t *needed, int32_t *n_variants) {
    g_err.clear();
    pb::jit::Spec sp;
    if (int rc = jit_spec_of(code, ops, n_ops, list_size, mode, opts, sp)) return rc;
    std::vector<uint16_t> vid;
    int nv = 0;
    const std::string src = pb::jit::generate(sp, vid, &nv);
    if (needed) *needed = (int64_t)src.size() + 1;
    if (n_variants) *n_variants = nv;
    if (buf && cap > 0) {
        const size_t c = std::min<size_t>((size_t)cap - 1, src.size());
        std::memcpy(buf, src.data(), c);
        buf[c] = 0;
    }
    return PB_OK;
}

int pb_jit_prebuild(const pb_code *code, const pb_op *ops, int n_ops, int list_size, int mode,
                    const pb_options *opts, int32_t *cache_hit, double *compile_s) {
    g_err.clear();
    pb::jit::Spec sp;
    if (int rc = jit_spec_of(code, ops, n_ops, list_size, mode, opts, sp)) return rc;
    std::vector<uint16_t> vid;
    const std::string src = pb::jit::generate(sp, vid, nullptr);
    std::string err;
    bool hit = false;
    double secs = 0.0;
    if (!pb::jit::acquire(src, false, 0, err, &hit, &secs)) return fail(PB_ECUDA, err);
    if (cache_hit) *cache_hit = hit;
    if (compile_s) *compile_s = secs;
    return PB_OK;
}

int pb_destroy(pb_handle *h) {
    if (!h) return PB_OK;
    cudaFree(h->d_prog);
    cudaFree(h->d_xsyn4);
    cudaFree(h->d_info);
    cudaFree(h->d_scratch);
    cudaFree(h->d_in);
    cudaFree(h->d_out);
    cudaFree(h->d_fail);
    cudaFree(h->d_ssc_ch);
    cudaFree(h->d_info_all);
    cudaFree(h->d_hu);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    for (int j = 0; j < 2; ++j) {
        if (h->aux[j]) cudaStreamDestroy(h->aux[j]);
        if (h->evj[j]) cudaEventDestroy(h->evj[j]);
    }
    if (h->evs) cudaEventDestroy(h->evs);
    if (h->ev_busy) cudaEventDestroy(h->ev_busy);
    cudaFree(h->d_lane_scratch);
    pb::jit::release(h->jk);
    delete h->lp;
    delete h;
    return PB_OK;
}

const char *pb_plan_json(pb_handle *h) { return h ? h->plan_json.c_str() : ""; }
long long pb_launch_count_impl(pb_handle *h) { return h ? h->launches : 0; }
int64_t pb_launch_count(pb_handle *h) { return h ? h->launches : 0; }

double pb_last_kernel_ms(pb_handle *h) {
    if (!h || !h->timed) return 0.0;
    float ms = 0.f;
    if (cudaEventSynchronize(h->ev1) != cudaSuccess) return 0.0;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    return ms;
}

}  // extern "C"

namespace {

int ensure(void **p, size_t *cap, size_t need) {
    if (*cap >= need) return PB_OK;
    cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    size_t sz = std::max(need, (size_t)1 << 20);
    cudaError_t e = cudaMalloc(p, sz);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc staging");
    *cap = sz;
    return PB_OK;
}

// Output staging regions of a batch in h->d_out: info [B][k], crc_ok [B],
// pm [B] doubles, paths_used [B] int32, invoked [B].
struct OutLayout {
    size_t ok, pm, pu, inv, total;
    explicit OutLayout(int64_t batch, int k) {
        const size_t big_info = (size_t)batch * k;
        ok = (big_info + 255) / 256 * 256;
        pm = ok + ((size_t)batch + 255) / 256 * 256;
        pu = pm + (size_t)batch * 8;
        inv = pu + ((size_t)batch * 4 + 255) / 256 * 256;
        total = inv + (size_t)batch;
    }
};

// Device buffers of one decode call (one chunk of a pipelined call).
struct Job {
    const void *llr;
    int64_t batch;
    uint8_t *info, *ok, *inv;
    double *pm;
    int32_t *pu;
    int32_t *fail_idx, *fail_count;  // adaptive only
};

// Launch the kernels of one decode on `st`:
//   list decode (L >= 2)  k_decode
//   L = 1                 k_ssc with the list decoder's leaf semantics
//   adaptive              k_ssc (fastssc semantics) settles the frames whose
//                         CRC passes and queues the rest; k_decode then takes
//                         the queued frames (count and rows read on the device)
// Order a launch on `st` after the handle's previous kernels (scratch reuse).
int scratch_acquire(pb_handle *h, cudaStream_t st) {
    if (!h->ev_busy) PB_CUDA(cudaEventCreateWithFlags(&h->ev_busy, cudaEventDisableTiming));
    if (h->busy_recorded) PB_CUDA(cudaStreamWaitEvent(st, h->ev_busy, 0));
    return PB_OK;
}
// the lane kernel: the per-code specialised build when the handle has one
cudaError_t lane_launch(pb_handle *h, const pb::lk::LParams *lp, int grid, cudaStream_t st) {
    if (!h->jk) return pb_lane_launch(lp, h->mode, grid, h->lane_smem, st);
    // a batch smaller than one CTA's frame slots runs only the warps it needs (as lane_launch_t)
    const long long need = (lp->batch + h->lane_fpw - 1) / h->lane_fpw;
    const int warps = grid == 1 && need < lp->fpc && !lp->batch_dev ? (int)need : lp->fpc;
    std::string err;
    const cudaError_t e = pb::jit::launch(h->jk, lp, grid, 32 * warps, h->lane_smem, st, err);
    if (e != cudaSuccess) g_err = err;
    return e;
}

int scratch_release(pb_handle *h, cudaStream_t st) {
    PB_CUDA(cudaEventRecord(h->ev_busy, st));
    h->busy_recorded = true;
    return PB_OK;
}

int run_kernels_unordered(pb_handle *h, const pb::Params &base, int in_type, const Job &j, bool adaptive,
                          cudaStream_t st);
int run_kernels(pb_handle *h, const pb::Params &base, int in_type, const Job &j, bool adaptive, cudaStream_t st) {
    if (j.batch <= 0) return PB_OK;
    int rc = scratch_acquire(h, st);
    if (rc) return rc;
    rc = run_kernels_unordered(h, base, in_type, j, adaptive, st);
    if (rc) return rc;
    return scratch_release(h, st);
}
int run_kernels_unordered(pb_handle *h, const pb::Params &base, int in_type, const Job &j, bool adaptive,
                          cudaStream_t st) {
    const bool use_ssc = adaptive || h->l1_ssc;
    if (use_ssc) {
        if (adaptive) PB_CUDA(cudaMemsetAsync(j.fail_count, 0, sizeof(int32_t), st));
        pb::SscParams sp = h->ssc;
        sp.semantics = adaptive ? pb::SSC_ADAPTIVE : pb::SSC_LIST_L1;
        sp.llr = j.llr;
        sp.in_type = in_type;
        sp.batch = j.batch;
        sp.info_out = j.info;
        sp.crc_ok = j.ok;
        sp.pm_out = j.pm;
        sp.paths_used = j.pu;
        sp.invoked = j.inv;
        sp.fail_idx = j.fail_idx;
        sp.fail_count = j.fail_count;
        sp.cw_out = nullptr;
        const int grid = (int)std::min<long long>(h->ssc_grid, (j.batch + sp.fpc - 1) / sp.fpc);
        cudaError_t e = pb_launch_ssc(&sp, h->mode, grid, st);
        if (e != cudaSuccess) return cuda_fail(e, "single-path kernel launch");
        h->launches += 1;
        if (!adaptive) return PB_OK;
    }
    if (h->lane) {
        pb::lk::LParams *lp = h->lp;
        lp->llr = j.llr;
        lp->in_type = in_type;
        lp->batch = j.batch;
        lp->info_out = j.info;
        lp->crc_ok = j.ok;
        lp->pm_out = j.pm;
        lp->paths_used = j.pu;
        lp->path_cw = nullptr;
        lp->path_pm = nullptr;
        lp->path_crc = nullptr;
        lp->frame_map = adaptive ? j.fail_idx : nullptr;
        lp->batch_dev = adaptive ? j.fail_count : nullptr;
        lp->op_cycles = nullptr;
        const int grid = (int)std::min<long long>(h->lane_grid, (j.batch + h->lane_fpc - 1) / h->lane_fpc);
        cudaError_t e = lane_launch(h, lp, grid, st);
        if (e != cudaSuccess) return cuda_fail(e, "lane decode kernel launch");
        h->launches += 1;
        return PB_OK;
    }
    pb::Params pr = base;
    pr.llr = j.llr;
    pr.in_type = in_type;
    pr.batch = j.batch;
    pr.info_out = j.info;
    pr.crc_ok = j.ok;
    pr.pm_out = j.pm;
    pr.paths_used = j.pu;
    pr.path_cw = nullptr;
    pr.path_pm = nullptr;
    pr.path_crc = nullptr;
    pr.frame_map = adaptive ? j.fail_idx : nullptr;
    pr.batch_dev = adaptive ? j.fail_count : nullptr;
    const int grid = (int)std::min<long long>(h->grid, (j.batch + h->fpc - 1) / h->fpc);
    cudaError_t e = pb_launch_decode(&pr, h->mode, h->warps, h->ppw, h->chg, grid, h->smem_frame * h->fpc + h->prog_smem, st);
    if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
    h->launches += 1;
    return PB_OK;
}

int ensure_fail(pb_handle *h, int64_t batch, int chunks) {
    return ensure((void **)&h->d_fail, &h->d_fail_cap, ((size_t)batch + 64 + (size_t)chunks) * sizeof(int32_t));
}

// Host-buffer decode of a large batch in chunks over two internal streams:
// chunk i's copy-in overlaps chunk i-1's kernels and copy-out (the copies
// only overlap when the host buffers are pinned).  The user stream orders
// the whole call; last_kernel_ms spans it.
int decode_pipelined(pb_handle *h, const pb::Params &base, const void *llr, int in_type, size_t in_es, int64_t batch,
                     long long chunk, uint8_t *info_out, uint8_t *crc_ok, double *pm_out, int32_t *paths_used,
                     uint8_t *invoked, bool adaptive, cudaStream_t st) {
    const size_t in_bytes = (size_t)batch * h->N * in_es;
    int rc = ensure(&h->d_in, &h->d_in_cap, in_bytes);
    if (rc) return rc;
    const OutLayout ol(batch, h->k);
    rc = ensure((void **)&h->d_out, &h->d_out_cap, ol.total);
    if (rc) return rc;
    const int nchunks = (int)((batch + chunk - 1) / chunk);
    if (adaptive && (rc = ensure_fail(h, batch, nchunks))) return rc;
    for (int j = 0; j < 2; ++j) {
        if (!h->aux[j]) PB_CUDA(cudaStreamCreateWithFlags(&h->aux[j], cudaStreamNonBlocking));
        if (!h->evj[j]) PB_CUDA(cudaEventCreateWithFlags(&h->evj[j], cudaEventDisableTiming));
    }
    if (!h->evs) PB_CUDA(cudaEventCreateWithFlags(&h->evs, cudaEventDisableTiming));
    PB_CUDA(cudaEventRecord(h->evs, st));
    for (int j = 0; j < 2; ++j) PB_CUDA(cudaStreamWaitEvent(h->aux[j], h->evs, 0));
    PB_CUDA(cudaEventRecord(h->ev0, h->aux[0]));
    unsigned char *din = static_cast<unsigned char *>(h->d_in);
    const unsigned char *hin = static_cast<const unsigned char *>(llr);
    int i = 0;
    for (long long f0 = 0; f0 < batch; f0 += chunk, ++i) {
        cudaStream_t sa = h->aux[i & 1];
        const long long nb = std::min<long long>(chunk, batch - f0);
        const size_t io = (size_t)f0 * h->N * in_es, ib = (size_t)nb * h->N * in_es;
        PB_CUDA(cudaMemcpyAsync(din + io, hin + io, ib, cudaMemcpyDefault, sa));
        Job jb{};
        jb.llr = din + io;
        jb.batch = nb;
        jb.info = info_out ? h->d_out + (size_t)f0 * h->k : nullptr;
        jb.ok = crc_ok ? h->d_out + ol.ok + f0 : nullptr;
        jb.pm = pm_out ? reinterpret_cast<double *>(h->d_out + ol.pm) + f0 : nullptr;
        jb.pu = paths_used ? reinterpret_cast<int32_t *>(h->d_out + ol.pu) + f0 : nullptr;
        jb.inv = invoked ? h->d_out + ol.inv + f0 : nullptr;
        jb.fail_idx = adaptive ? h->d_fail + f0 : nullptr;
        jb.fail_count = adaptive ? h->d_fail + batch + 64 + i : nullptr;
        if ((rc = run_kernels(h, base, in_type, jb, adaptive, sa))) return rc;
        if (info_out)
            PB_CUDA(cudaMemcpyAsync(info_out + (size_t)f0 * h->k, jb.info, (size_t)nb * h->k, cudaMemcpyDefault, sa));
        if (crc_ok) PB_CUDA(cudaMemcpyAsync(crc_ok + f0, jb.ok, (size_t)nb, cudaMemcpyDefault, sa));
        if (pm_out) PB_CUDA(cudaMemcpyAsync(pm_out + f0, jb.pm, (size_t)nb * 8, cudaMemcpyDefault, sa));
        if (paths_used) PB_CUDA(cudaMemcpyAsync(paths_used + f0, jb.pu, (size_t)nb * 4, cudaMemcpyDefault, sa));
        if (invoked) PB_CUDA(cudaMemcpyAsync(invoked + f0, jb.inv, (size_t)nb, cudaMemcpyDefault, sa));
    }
    for (int j = 0; j < 2; ++j) {
        PB_CUDA(cudaEventRecord(h->evj[j], h->aux[j]));
        PB_CUDA(cudaStreamWaitEvent(st, h->evj[j], 0));
    }
    PB_CUDA(cudaEventRecord(h->ev1, st));
    h->timed = true;
    PB_CUDA(cudaStreamSynchronize(st));
    PB_CUDA(cudaGetLastError());
    return PB_OK;
}

int launch_timed(pb_handle *h, const pb::Params &base, int in_type, const Job &j, bool adaptive, cudaStream_t st) {
    if (j.batch <= 0) return PB_OK;
    PB_CUDA(cudaEventRecord(h->ev0, st));
    int rc = run_kernels(h, base, in_type, j, adaptive, st);
    if (rc) return rc;
    PB_CUDA(cudaEventRecord(h->ev1, st));
    h->timed = true;
    return PB_OK;
}

int launch(pb_handle *h, pb::Params &pr, cudaStream_t st) {
    int grid = (int)std::min<long long>(h->grid, (pr.batch + h->fpc - 1) / h->fpc);
    if (grid < 1) return PB_OK;
    int rc = scratch_acquire(h, st);
    if (rc) return rc;
    PB_CUDA(cudaEventRecord(h->ev0, st));
    cudaError_t e;
    if (h->lane) {
        pb::lk::LParams *lp = h->lp;
        lp->llr = pr.llr;
        lp->in_type = pr.in_type;
        lp->batch = pr.batch;
        lp->info_out = pr.info_out;
        lp->crc_ok = pr.crc_ok;
        lp->pm_out = pr.pm_out;
        lp->paths_used = pr.paths_used;
        lp->path_cw = pr.path_cw;
        lp->path_pm = pr.path_pm;
        lp->path_crc = pr.path_crc;
        lp->frame_map = nullptr;
        lp->batch_dev = nullptr;
        lp->op_cycles = pr.op_cycles;
        grid = (int)std::min<long long>(h->lane_grid, (pr.batch + h->lane_fpc - 1) / h->lane_fpc);
        e = lane_launch(h, lp, grid, st);
    } else {
        e = pb_launch_decode(&pr, h->mode, h->warps, h->ppw, h->chg, grid, h->smem_frame * h->fpc + h->prog_smem, st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "decode kernel launch");
    PB_CUDA(cudaEventRecord(h->ev1, st));
    h->timed = true;
    h->launches += 1;
    return scratch_release(h, st);
}

int decode_impl(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *info_out, uint8_t *crc_ok,
                double *pm_out, int32_t *paths_used, uint8_t *invoked, bool adaptive, void *stream) {
    g_err.clear();
    if (!h) return fail(PB_EINVAL, "null handle");
    if (batch < 0) return fail(PB_EINVAL, "negative batch");
    if (in_type != PB_IN_F32 && in_type != PB_IN_I8) return fail(PB_EINVAL, "unknown input type");
    if (in_type == PB_IN_I8 && h->mode != PB_MODE_INT8)
        return fail(PB_EINVAL, "int8 LLR input needs an int8-mode decoder");
    if (adaptive && !h->base.has_crc) return fail(PB_EINVAL, "adaptive decoding needs a CRC in the code spec");
    if (adaptive && !h->ssc_ok)
        return fail(PB_EINVAL, "code too large for the single-path pass's shared-memory plan");
    if (batch == 0) return PB_OK;
    if (!llr) return fail(PB_EINVAL, "null LLR pointer");
    PB_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const size_t in_es = in_type == PB_IN_F32 ? 4 : 1;
    const size_t in_bytes = (size_t)batch * h->N * in_es;

    const bool dev_in = is_device_ptr(llr);
    const bool all_dev = dev_in && (!info_out || is_device_ptr(info_out)) && (!crc_ok || is_device_ptr(crc_ok)) &&
                         (!pm_out || is_device_ptr(pm_out)) && (!paths_used || is_device_ptr(paths_used)) &&
                         (!invoked || is_device_ptr(invoked));
    if (all_dev) {
        int rc = adaptive ? ensure_fail(h, batch, 1) : PB_OK;
        if (rc) return rc;
        Job jb{llr, batch, info_out, crc_ok, invoked, pm_out, paths_used,
               adaptive ? h->d_fail : nullptr, adaptive ? h->d_fail + batch + 64 : nullptr};
        return launch_timed(h, h->base, in_type, jb, adaptive, st);
    }
    // staged path: host buffers in and/or out
    // one wave of resident frames per chunk: the smaller the first copy-in and
    // last copy-out, the less of them is exposed (measured e2e / device-
    // resident: 6 waves 95 %, 1 wave 99 % on c3 L=32); consecutive chunks'
    // kernels overlap across the two streams, hiding each wave's tail
    // (adaptive decoding: 6 waves, so each chunk's list pass over its few
    // CRC failures amortises its launch and its grid-wide occupancy)
    // whole waves of the persistent grid (a partial last wave idles most of the SMs), at least 2048 frames
    const long long wave = h->lane ? (long long)h->lane_grid * h->lane_fpc : (long long)h->grid * h->fpc;
    const long long waves = std::max<long long>(adaptive ? 6 : 1, (2048 + wave - 1) / std::max<long long>(1, wave));
    const long long chunk = std::max<long long>(1, h->chunk_frames > 0 ? (long long)h->chunk_frames : waves * wave);
    if (!dev_in && batch > chunk)
        return decode_pipelined(h, h->base, llr, in_type, in_es, batch, chunk, info_out, crc_ok, pm_out, paths_used,
                                invoked, adaptive, st);
    const void *dllr = llr;
    if (!dev_in) {
        int rc = ensure(&h->d_in, &h->d_in_cap, in_bytes);
        if (rc) return rc;
        PB_CUDA(cudaMemcpyAsync(h->d_in, llr, in_bytes, cudaMemcpyDefault, st));
        dllr = h->d_in;
    }
    const OutLayout ol(batch, h->k);
    int rc = ensure((void **)&h->d_out, &h->d_out_cap, ol.total);
    if (rc) return rc;
    if (adaptive && (rc = ensure_fail(h, batch, 1))) return rc;
    Job jb{};
    jb.llr = dllr;
    jb.batch = batch;
    jb.info = info_out ? h->d_out : nullptr;
    jb.ok = crc_ok ? h->d_out + ol.ok : nullptr;
    jb.pm = pm_out ? reinterpret_cast<double *>(h->d_out + ol.pm) : nullptr;
    jb.pu = paths_used ? reinterpret_cast<int32_t *>(h->d_out + ol.pu) : nullptr;
    jb.inv = invoked ? h->d_out + ol.inv : nullptr;
    jb.fail_idx = adaptive ? h->d_fail : nullptr;
    jb.fail_count = adaptive ? h->d_fail + batch + 64 : nullptr;
    rc = launch_timed(h, h->base, in_type, jb, adaptive, st);
    if (rc) return rc;
    if (info_out) PB_CUDA(cudaMemcpyAsync(info_out, jb.info, (size_t)batch * h->k, cudaMemcpyDefault, st));
    if (crc_ok) PB_CUDA(cudaMemcpyAsync(crc_ok, jb.ok, (size_t)batch, cudaMemcpyDefault, st));
    if (pm_out) PB_CUDA(cudaMemcpyAsync(pm_out, jb.pm, (size_t)batch * 8, cudaMemcpyDefault, st));
    if (paths_used) PB_CUDA(cudaMemcpyAsync(paths_used, jb.pu, (size_t)batch * 4, cudaMemcpyDefault, st));
    if (invoked) PB_CUDA(cudaMemcpyAsync(invoked, jb.inv, (size_t)batch, cudaMemcpyDefault, st));
    PB_CUDA(cudaStreamSynchronize(st));
    PB_CUDA(cudaGetLastError());
    return PB_OK;
}

}  // namespace

extern "C" int pb_decode(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *info_out,
                         uint8_t *crc_ok, double *pm_out, int32_t *paths_used, void *stream) {
    return decode_impl(h, llr, in_type, batch, info_out, crc_ok, pm_out, paths_used, nullptr, false, stream);
}

extern "C" int pb_decode_adaptive(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *info_out,
                                  uint8_t *crc_ok, double *pm_out, int32_t *paths_used, uint8_t *invoked_list,
                                  void *stream) {
    return decode_impl(h, llr, in_type, batch, info_out, crc_ok, pm_out, paths_used, invoked_list, true, stream);
}

// Debug: decode `batch` host frames and return the clock64 cycles each device
// op took for CTA 0's first frame (out: [pb_device_op_count] int64), plus
// the op kinds/stages (kinds/stages may be null).
extern "C" int pb_device_op_count(pb_handle *h) { return h ? (h->lane ? h->lp->n_ops : (int)h->prog.size()) : 0; }
extern "C" int pb_profile_ops(pb_handle *h, const void *llr, int in_type, int64_t batch, long long *cycles,
                              int8_t *kinds, int8_t *stages) {
    if (!h || !llr || !cycles) return fail(PB_EINVAL, "null argument");
#if !PB_PROFILE
    (void)in_type, (void)batch, (void)kinds, (void)stages;
    return fail(PB_EINVAL, "per-op profile needs the profiling build (_native.build(profile=True))");
#endif
    PB_CUDA(cudaSetDevice(h->device));
    const size_t in_bytes = (size_t)batch * h->N * (in_type == PB_IN_F32 ? 4 : 1);
    int rc = ensure(&h->d_in, &h->d_in_cap, in_bytes);
    if (rc) return rc;
    long long *d_cyc = nullptr;
    const size_t ncyc = 12 * std::max<size_t>(h->prog.size(), h->lane ? (size_t)h->lp->n_ops + 1 : 0);
    PB_CUDA(cudaMalloc(&d_cyc, sizeof(long long) * ncyc));
    PB_CUDA(cudaMemset(d_cyc, 0, sizeof(long long) * ncyc));
    PB_CUDA(cudaMemcpy(h->d_in, llr, in_bytes, cudaMemcpyHostToDevice));
    pb::Params pr = h->base;
    pr.llr = h->d_in;
    pr.in_type = in_type;
    pr.batch = batch;
    pr.info_out = nullptr;
    pr.crc_ok = nullptr;
    pr.pm_out = nullptr;
    pr.paths_used = nullptr;
    pr.path_cw = nullptr;
    pr.op_cycles = d_cyc;
    rc = launch(h, pr, 0);
    if (rc) return rc;
    PB_CUDA(cudaDeviceSynchronize());
    PB_CUDA(cudaMemcpy(cycles, d_cyc, sizeof(long long) * 12 * pb_device_op_count(h), cudaMemcpyDeviceToHost));
    if (h->lane) {  // the lane kernel's marks follow its op start times: fetch them too
        std::vector<long long> all(ncyc);
        PB_CUDA(cudaMemcpy(all.data(), d_cyc, sizeof(long long) * ncyc, cudaMemcpyDeviceToHost));
        const int n = h->lp->n_ops;
        // pack [n+1 starts][4n marks] into the caller's buffer (12n longs >= 5n+1)
        std::copy(all.begin(), all.begin() + (n + 1 + 4 * n), cycles);
    }
    cudaFree(d_cyc);
    if (h->lane) {
        // lane kernel: cycles[i] = clock64 at the start of op i (i <= n_ops);
        // converted here to per-op durations in the 12-long rows the tool reads
        const int n = h->lp->n_ops;
        std::vector<long long> t(cycles, cycles + n + 1 + 4 * n);
        for (int i = 0; i < n; ++i) {
            for (int x = 0; x < 12; ++x) cycles[i * 12 + x] = 0;
            cycles[i * 12] = t[i + 1] - t[i];
            cycles[i * 12 + 1] = t[i];
            // leaf phase marks -> the tool's columns: A end (2+0), B end (2+1), C copies (2+7)
            const long long *mk = t.data() + n + 1 + 4 * i;
            cycles[i * 12 + 2 + 0] = mk[0];
            cycles[i * 12 + 2 + 1] = mk[1];
            cycles[i * 12 + 2 + 7] = mk[2];
            if (kinds) kinds[i] = (int8_t)h->lp->prog[i].kind;
            if (stages) stages[i] = (int8_t)h->lp->prog[i].stage;
        }
        return PB_OK;
    }
    for (size_t i = 0; i < h->prog.size(); ++i) {
        if (kinds) kinds[i] = h->prog[i].kind;
        if (stages) stages[i] = h->prog[i].stage;
    }
    return PB_OK;
}

extern "C" int pb_decode_paths(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *codewords,
                               double *path_pm, uint8_t *path_crc, int32_t *paths_used, void *stream) {
    g_err.clear();
    if (!h) return fail(PB_EINVAL, "null handle");
    if (batch < 0) return fail(PB_EINVAL, "negative batch");
    if (in_type != PB_IN_F32 && in_type != PB_IN_I8) return fail(PB_EINVAL, "unknown input type");
    if (in_type == PB_IN_I8 && h->mode != PB_MODE_INT8)
        return fail(PB_EINVAL, "int8 LLR input needs an int8-mode decoder");
    if (batch == 0) return PB_OK;
    if (!llr || !codewords || !path_pm || !path_crc || !paths_used) return fail(PB_EINVAL, "null pointer");
    PB_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int L = h->L, rw = h->base.lay.root_words;
    const size_t in_bytes = (size_t)batch * h->N * (in_type == PB_IN_F32 ? 4 : 1);
    int rc = ensure(&h->d_in, &h->d_in_cap, in_bytes);
    if (rc) return rc;
    PB_CUDA(cudaMemcpyAsync(h->d_in, llr, in_bytes, cudaMemcpyHostToDevice, st));
    const size_t o_cw = 0, n_cw = (size_t)batch * L * rw * 4;
    const size_t o_pm = (n_cw + 255) / 256 * 256;
    const size_t o_crc = o_pm + (size_t)batch * L * 8;
    const size_t o_pu = (o_crc + (size_t)batch * L + 255) / 256 * 256;
    const size_t total = o_pu + (size_t)batch * 4;
    rc = ensure((void **)&h->d_out, &h->d_out_cap, total);
    if (rc) return rc;
    PB_CUDA(cudaMemsetAsync(h->d_out, 0, total, st));
    pb::Params pr = h->base;
    pr.llr = h->d_in;
    pr.in_type = in_type;
    pr.batch = batch;
    pr.info_out = nullptr;
    pr.crc_ok = nullptr;
    pr.pm_out = nullptr;
    pr.paths_used = reinterpret_cast<int32_t *>(h->d_out + o_pu);
    pr.path_cw = reinterpret_cast<uint32_t *>(h->d_out + o_cw);
    pr.path_pm = reinterpret_cast<double *>(h->d_out + o_pm);
    pr.path_crc = h->d_out + o_crc;
    rc = launch(h, pr, st);
    if (rc) return rc;
    std::vector<uint32_t> cw((size_t)batch * L * rw);
    PB_CUDA(cudaMemcpyAsync(cw.data(), pr.path_cw, n_cw, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaMemcpyAsync(path_pm, pr.path_pm, (size_t)batch * L * 8, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaMemcpyAsync(path_crc, pr.path_crc, (size_t)batch * L, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaMemcpyAsync(paths_used, pr.paths_used, (size_t)batch * 4, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaStreamSynchronize(st));
    const int N = h->N;
    for (size_t r = 0; r < (size_t)batch * L; ++r)
        for (int i = 0; i < N; ++i) codewords[r * N + i] = (uint8_t)((cw[r * rw + (i >> 5)] >> (i & 31)) & 1u);
    return PB_OK;
}

// polaris.fastssc.execute_schedule (fastssc.py:20-83): the single-path
// pass alone.  Host buffers only; synchronous.
extern "C" int pb_fastssc(pb_handle *h, const void *llr, int in_type, int64_t batch, uint8_t *codewords,
                          double *pm_out, void *stream) {
    g_err.clear();
    if (!h) return fail(PB_EINVAL, "null handle");
    if (batch < 0) return fail(PB_EINVAL, "negative batch");
    if (in_type != PB_IN_F32 && in_type != PB_IN_I8) return fail(PB_EINVAL, "unknown input type");
    if (in_type == PB_IN_I8 && h->mode != PB_MODE_INT8)
        return fail(PB_EINVAL, "int8 LLR input needs an int8-mode decoder");
    if (!h->ssc_ok) return fail(PB_EINVAL, "code too large for the single-path pass's shared-memory plan");
    if (batch == 0) return PB_OK;
    if (!llr || !codewords || !pm_out) return fail(PB_EINVAL, "null pointer");
    PB_CUDA(cudaSetDevice(h->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int N = h->N, nwd = std::max(1, N / 32);
    const size_t in_bytes = (size_t)batch * N * (in_type == PB_IN_F32 ? 4 : 1);
    int rc = ensure(&h->d_in, &h->d_in_cap, in_bytes);
    if (rc) return rc;
    const size_t n_cw = (size_t)batch * nwd * 4, o_pm = (n_cw + 255) / 256 * 256;
    rc = ensure((void **)&h->d_out, &h->d_out_cap, o_pm + (size_t)batch * 8);
    if (rc) return rc;
    PB_CUDA(cudaMemcpyAsync(h->d_in, llr, in_bytes, cudaMemcpyHostToDevice, st));
    pb::SscParams sp = h->ssc;
    sp.semantics = pb::SSC_FAST;
    sp.llr = h->d_in;
    sp.in_type = in_type;
    sp.batch = batch;
    sp.info_out = nullptr;
    sp.crc_ok = nullptr;
    sp.pm_out = reinterpret_cast<double *>(h->d_out + o_pm);
    sp.paths_used = nullptr;
    sp.invoked = nullptr;
    sp.fail_idx = nullptr;
    sp.fail_count = nullptr;
    sp.cw_out = reinterpret_cast<uint32_t *>(h->d_out);
    const int grid = (int)std::min<long long>(h->ssc_grid, (batch + sp.fpc - 1) / sp.fpc);
    if ((rc = scratch_acquire(h, st))) return rc;
    cudaError_t e = pb_launch_ssc(&sp, h->mode, grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "single-path kernel launch");
    h->launches += 1;
    if ((rc = scratch_release(h, st))) return rc;
    std::vector<uint32_t> cw((size_t)batch * nwd);
    PB_CUDA(cudaMemcpyAsync(cw.data(), sp.cw_out, n_cw, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaMemcpyAsync(pm_out, sp.pm_out, (size_t)batch * 8, cudaMemcpyDeviceToHost, st));
    PB_CUDA(cudaStreamSynchronize(st));
    for (size_t r = 0; r < (size_t)batch; ++r)
        for (int i = 0; i < N; ++i) codewords[r * N + i] = (uint8_t)((cw[r * nwd + (i >> 5)] >> (i & 31)) & 1u);
    return PB_OK;
}

// On-device frames (frame_gen.cu): `count` frames first_frame.. of the
// (seed, Eb/N0) stream of this handle's code, LLRs float32 (out_type
// PB_IN_F32) or int8 (PB_IN_I8) into llr_out [count][N], packed payload bits
// into payload_out [count][ceil(k/32)] (may be NULL).  Device buffers only;
// asynchronous on `stream`.
extern "C" int pb_generate_frames(pb_handle *h, uint64_t seed, double ebn0_db, int64_t first_frame, int64_t count,
                                  int out_type, void *llr_out, uint32_t *payload_out, void *stream) {
    g_err.clear();
    if (!h) return fail(PB_EINVAL, "null handle");
    if (count < 0 || first_frame < 0) return fail(PB_EINVAL, "negative frame range");
    if (out_type != PB_IN_F32 && out_type != PB_IN_I8) return fail(PB_EINVAL, "unknown output type");
    if (count == 0) return PB_OK;
    if (!llr_out) return fail(PB_EINVAL, "null LLR pointer");
    PB_CUDA(cudaSetDevice(h->device));
    pb::gen::GenParams g{};
    g.N = h->N;
    g.n = h->n;
    g.k = h->k;
    g.crc_w = h->crc_w;
    g.info_pos = h->d_info_all;
    g.hu = h->d_hu;
    g.crc_const = h->gen_crc_const;
    g.seed = seed;
    g.first = first_frame;
    g.count = count;
    const double rate = (double)h->k / h->N;  // payload rate, sim.py:70,166
    const double sigma = std::sqrt(1.0 / (2.0 * rate * std::pow(10.0, ebn0_db / 10.0)));
    g.sigma = (float)sigma;
    g.scale = (float)(2.0 / (sigma * sigma));
    g.out_type = out_type == PB_IN_F32 ? 0 : 1;
    g.llr = llr_out;
    g.payload = payload_out;
    g.kw = (h->k + 31) / 32;
    cudaError_t e = pb_launch_gen(&g, h->sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "frame generator launch");
    h->launches += 1;
    return PB_OK;
}

// Error counters of decoded payload bytes info [batch][k] against packed
// payload bits [batch][ceil(k/32)], accumulated (added) per chunk of `chunk`
// frames into counts [ceil(batch/chunk)][3] uint64 = (frames, frame errors,
// bit errors).  Device buffers only; asynchronous on `stream`.
extern "C" int pb_count_errors(pb_handle *h, const uint8_t *info, const uint32_t *payload, int64_t batch, int chunk,
                               uint64_t *counts, void *stream) {
    g_err.clear();
    if (!h) return fail(PB_EINVAL, "null handle");
    if (batch < 0 || chunk < 1) return fail(PB_EINVAL, "bad batch / chunk");
    if (batch == 0) return PB_OK;
    if (!info || !payload || !counts) return fail(PB_EINVAL, "null pointer");
    PB_CUDA(cudaSetDevice(h->device));
    cudaError_t e = pb_launch_errcount(info, payload, batch, h->k, (h->k + 31) / 32, chunk,
                                    reinterpret_cast<unsigned long long *>(counts), h->sms, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "error counter launch");
    h->launches += 1;
    return PB_OK;
}

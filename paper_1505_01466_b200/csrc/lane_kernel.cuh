// lane_kernel.cuh -- lane-per-path Fast-SSC list-CRC decode kernel (sm_100a).
//
// A warp decodes one frame (L > 16: lane q owns path slot q) or 32/pow2(L)
// frames (L <= 16: lane = frame slot x path slot; the specialised build).
// The default list kernel; instantiated generically by lane_inst.cu (every op
// field read at run time) and per code by the translation unit jit.cu
// generates (PB_JIT: fields, layout and code constants folded in).  Built
// around:
//   * per-path state in registers: metric (f64), the row index of every
//     alpha stage / beta slot (8-bit fields), the leaf data a survivor needs
//     from its source (hard word, least reliable positions, parity) --
//     survivors gather it from the source lane with shuffles
//     (listdec.py:397-434 lazy copy == inheriting the source's row indices);
//   * the channel in shared memory (global scratch for L <= 16) and the two
//     top stages n-1, n-2 never stored: every read recomputes them from the
//     channel and the path's beta bits, which halves the per-frame global
//     scratch (c3 L=32: 144 KB -> 70 KB);
//   * leaves that read f / g of their parent's row (the F / G before a leaf
//     is folded into its reads), dead global stages discarded from the L2;
//   * survivor selection on the high 27 bits of the order-preserving metric
//     keys with the lane in the low 5 (one REDUX per max / min), and an exact
//     64-bit resolution of the candidates tied at the threshold
//     (listdec.py:63-100 exactly); per frame when frames share a warp.
#pragma once
#include "decode_kernel.cuh"

// stage n-2 reads specialised on the (n-1, n-2) F / G modes (one loop per
// mode pair) instead of a uniform branch per quad
#ifndef PB_LANE_V2SPEC
#define PB_LANE_V2SPEC 1
#endif
// survivor hand-over by a loop over the set bits (run-time key index: the keys
// live in local memory) instead of the unrolled predicated form
#ifndef PB_ASG_LOOP
#define PB_ASG_LOOP 0
#endif
// specialised build: quads per block of the pipelined wide-leaf scan (0 = off)
#ifndef PB_SCAN_PIPE
#define PB_SCAN_PIPE 0
#endif
// a survivor's chain rows of at least this many words use the unrolled form
// (all slot-word loads independent); the specialised build sets 2
#ifndef PB_CHAIN_CLOSED_MIN
#define PB_CHAIN_CLOSED_MIN 1000000
#endif

// Per-code specialised build (PB_JIT, csrc/jit.cpp): the generated translation
// unit defines, before including this header,
//   __device__ constexpr LLayout kLay   the frame's storage plan
//   __device__ constexpr JitCode kJit   N, n, k, L, CRC constants, op counts
//   PB_JIT_OPS(X)                        X(id, kind, stage, pin, pout, ncand, src, aux, flags)
//                                        one line per distinct op of the schedule (-1 = read at run time)
// so stages, row placements (shared vs global), offsets, path counts and
// selection shapes are compile-time constants in every op body -- the
// paper's unrolled decoder (arXiv 1505.01466 sec. IV: node functions
// specialised on size and position, schedule.py:159-206), with the op
// sequence kept as a table of variant ids instead of straight-line code so
// the SM's warps share the instruction cache.  Without PB_JIT the same
// bodies read everything at run time (the generic kernel: the correctness
// twin and the fallback when NVRTC is unavailable).
#ifdef PB_JIT
#define LK_LAY(P) (::pb::lk::kLay)
#define LK_C(P, f) (::pb::lk::kJit.f)
// frames per warp (list sizes <= 16: a warp's 32 lanes = G frames x 32/G path
// slots; lane = frame slot * 32/G + path slot).  The warp's 32 row slots, the
// row-index bytes, the hard-word columns and the survivor tables are indexed
// by lane as before; selection, the survivor scan and the final pick work on
// the lanes of one frame (segment masks); each frame has its own channel,
// the G channels interleaved quad by quad.
#define LK_G (::pb::lk::kJit.G)
#else
#define LK_LAY(P) ((P).lay)
#define LK_C(P, f) ((P).f)
#define LK_G 1  // the generic kernel: one frame per warp
#endif

namespace pb {
namespace lk {

// An op as the bodies see it: each field a compile-time constant (>= 0) or
// read from the runtime LOp (-1).
template <int KIND = -1, int STAGE = -1, int PIN = -1, int POUT = -1, int NCAND = -1, int SRC = -1, int AUX = -1,
          int FLAGS = -1>
struct Op {
    LOp o;
    __device__ __forceinline__ int kind() const { return KIND >= 0 ? KIND : (int)o.kind; }
    __device__ __forceinline__ int stage() const { return STAGE >= 0 ? STAGE : (int)o.stage; }
    __device__ __forceinline__ int pin() const { return PIN >= 0 ? PIN : (int)o.pin; }
    __device__ __forceinline__ int pout() const { return POUT >= 0 ? POUT : (int)o.pout; }
    __device__ __forceinline__ int ncand() const { return NCAND >= 0 ? NCAND : (int)o.ncand; }
    __device__ __forceinline__ int src() const { return SRC >= 0 ? SRC : (int)o.src; }
    __device__ __forceinline__ int aux() const { return AUX >= 0 ? AUX : (int)o.aux; }
    __device__ __forceinline__ int flags() const { return FLAGS >= 0 ? FLAGS : (int)o.flags; }
};

__device__ __forceinline__ int get8(const uint32_t (&w)[4], int s) {
    const int j = s >> 2;
    const uint32_t x = j == 0 ? w[0] : (j == 1 ? w[1] : (j == 2 ? w[2] : w[3]));
    return (x >> ((s & 3) * 8)) & 0xff;
}
__device__ __forceinline__ void set8(uint32_t (&w)[4], int s, int v) {
    const int sh = (s & 3) * 8, j = s >> 2;
    const uint32_t m = ~(0xffu << sh), vv = (uint32_t)v << sh;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (j == i) w[i] = (w[i] & m) | vv;
}

// min-sum F in one instruction: min.xorsign.abs (FMNMX.XORSIGN |a|, |b|) returns
// min(|a|, |b|) with the XOR of the two signs -- kernels.py:39-48 exactly, zero
// inputs included (a signed zero, numerically the reference's 0).
__device__ __forceinline__ float f_op(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// the inverse of okey (an involution on the bit pattern)
__device__ __forceinline__ double unkey(long long k) {
    return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}

// per-frame warp state
template <typename T>
struct Fr {
    const LParams &P;
    unsigned char *sm;   // frame's shared-memory block
    unsigned char *gs;   // frame's global scratch block
    int lane;
    double pm;           // path metric (listdec.py:146-153)
    uint32_t ia[4];      // alpha row of stage s: byte s
    uint32_t ib[4];      // beta row of slot s: byte s
    // leaf data of the path's last forking leaf decision (kept for the
    // final pick: the root codeword is built from it on demand)
    uint32_t hard;       // hard decisions (leaf size <= 32)
    uint32_t lrb01;      // least reliable positions 0, 1 (16 bits each)
    uint32_t lrb23;      // positions 2, 3
    uint32_t lflag;      // Rep: ones first; SPC: odd parity
    uint32_t dec;        // candidate chosen (0 .. 7)
    uint32_t srcl;       // source lane of that decision

    __device__ __forceinline__ Fr(const LParams &p, unsigned char *s, unsigned char *g)
        : P(p), sm(s), gs(g), lane(threadIdx.x & 31), pm(0.0), hard(0), lrb01(0), lrb23(0), lflag(0), dec(0), srcl(0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) ia[i] = ib[i] = 0u;
    }
    long long *marks = nullptr;  // profiling build: this op's phase marks (CTA 0, frame slot 0, lane 0)
    __device__ __forceinline__ void mark(int k) const {
#if PB_PROFILE
        if (marks) marks[k] = clock64();
#endif
    }
    // frames per warp, path slots per frame, channel quad stride (elements)
    static constexpr int G = LK_G, LP = 32 / LK_G, CQ = 4 * LK_G;
    __device__ __forceinline__ int base() const { return G == 1 ? 0 : lane & ~(LP - 1); }  // frame's first lane
    __device__ __forceinline__ int slot() const { return G == 1 ? lane : lane & (LP - 1); }  // path slot in its frame
    __device__ __forceinline__ unsigned seg() const {  // the lanes of this lane's frame
        return G == 1 ? FULL_MASK : ((1u << LP) - 1u) << base();
    }
    // this lane's frame's channel: quad x at channel() + x * CQ
    __device__ __forceinline__ T *channel() const {
        return reinterpret_cast<T *>((LK_LAY(P).ch_gl ? gs : sm) + LK_LAY(P).ch_off) + (G == 1 ? 0 : 4 * (lane / LP));
    }
    // hard-decision words of leaves wider than 32 (global scratch): word w of
    // lane q's path at [w * 32 + q]
    __device__ __forceinline__ uint32_t *hard_words() const {
        return reinterpret_cast<uint32_t *>(gs + LK_LAY(P).hard_off);
    }
    __device__ __forceinline__ uint32_t *beta_row(int s, int row) const {
        unsigned char *base = ((LK_LAY(P).b_gl >> s) & 1u) ? gs : sm;
        return reinterpret_cast<uint32_t *>(base + LK_LAY(P).b_off[s]) + row * LK_LAY(P).b_stride[s];
    }
    // stored alpha row r of stage s: quad x at element x * 128 (32 rows x 4)
    __device__ __forceinline__ T *a_row(int s, int r) const {
        unsigned char *base = ((LK_LAY(P).a_gl >> s) & 1u) ? gs : sm;
        return reinterpret_cast<T *>(base + LK_LAY(P).a_off[s]) + r * 4;
    }
    // The stored stage s (global scratch) is dead once its last reader is
    // done: every later access is a full rewrite (each F / G covers the whole
    // stage for all paths).  Dropping its lines from the L2 keeps them from
    // being written back to DRAM and from pushing live rows out.
    __device__ __forceinline__ void discard_stage(int s) const {
        const int bytes = 32 * (s < 2 ? 4 : 1 << s) * (int)sizeof(T);
        unsigned char *base = gs + LK_LAY(P).a_off[s];
        for (int off = lane * 128; off < bytes; off += 32 * 128)
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + off) : "memory");
    }
    template <int WHERE>
    __device__ __forceinline__ T *a_row_t(int s, int r) const {
        return reinterpret_cast<T *>((WHERE == S_GL ? gs : sm) + LK_LAY(P).a_off[s]) + r * 4;
    }
};

// ------------------------------------------------------------ sources
// A path's view of one alpha stage: quad(x) = elements 4x .. 4x+3, get(i).

template <typename T>
struct RowLd {  // a stored row (quad stride 128: 32 interleaved rows) or the channel (4)
    const T *p;
    int qs;
    __device__ __forceinline__ void quad(int x, float (&v)[4]) const { V4<T>::ld(p + x * qs, v); }
    __device__ __forceinline__ float get(int i) const { return Elem<T>::ld(p + (i >> 2) * qs + (i & 3)); }
};
// channel addressing: quad x of a frame's channel at ch + x * CQ (CQ = 4 with
// one frame per warp; the frames of a warp interleave quad by quad)
constexpr int CQ = 4 * LK_G;
template <typename T>
__device__ __forceinline__ const T *che(const T *ch, int i) {
    return ch + (i >> 2) * CQ + (i & 3);
}
// stage n-1: f or g of the channel halves (g with the path's left-half bits,
// beta slot n-1)
template <typename T, int MODE = -1>  // MODE >= 0: g known at compile time (MODE & 1)
struct V1Ld {
    const T *ch;
    const uint32_t *b1;
    int half;  // N / 2
    bool g_;
    __device__ __forceinline__ bool gm() const { return MODE >= 0 ? (MODE & 1) != 0 : g_; }
    __device__ __forceinline__ void quad(int x, float (&v)[4]) const {
        float a[4], b[4];
        V4<T>::ld(ch + CQ * x, a);
        V4<T>::ld(ch + CQ * (x + (half >> 2)), b);
        if (gm()) {
            const unsigned bits = b1[x >> 3] >> ((x & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(a[j], b[j], bits, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(a[j], b[j]);
        }
    }
    __device__ __forceinline__ float get(int i) const {
        const float a = Elem<T>::ld(che(ch, i)), b = Elem<T>::ld(che(ch, i + half));
        return gm() ? g_op<T>(a, b, (b1[i >> 5] >> (i & 31)) & 1u) : f_op(a, b);
    }
    // beta words of the 8-quad block starting at quad x (x % 8 == 0), loaded
    // once per block; quadw = quad with them
    struct Words {
        uint32_t w1;
    };
    __device__ __forceinline__ Words words(int x) const { return Words{gm() ? b1[x >> 3] : 0u}; }
    __device__ __forceinline__ void quadw(int x, float (&v)[4], const Words &w) const {
        float a[4], b[4];
        V4<T>::ld(ch + CQ * x, a);
        V4<T>::ld(ch + CQ * (x + (half >> 2)), b);
        if (gm()) {
            const unsigned bits = w.w1 >> ((x & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(a[j], b[j], bits, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(a[j], b[j]);
        }
    }
};
// stage n-2: f or g of two stage n-1 values (beta slot n-2), each f or g of
// two channel values -- four channel loads per element, all lanes reading
// the same address
template <typename T, int MODE = -1>  // MODE >= 0: (g1, g2) = (MODE & 1, MODE >> 1) at compile time
struct V2Ld {
    const T *ch;
    const uint32_t *b1, *b2;
    int q;  // N / 4
    bool g1_, g2_;
    __device__ __forceinline__ bool m1() const { return MODE >= 0 ? (MODE & 1) != 0 : g1_; }
    __device__ __forceinline__ bool m2() const { return MODE >= 0 ? (MODE & 2) != 0 : g2_; }
    __device__ __forceinline__ void quad(int x, float (&v)[4]) const {
        float c0[4], c1[4], c2[4], c3[4];
        V4<T>::ld(ch + CQ * x, c0);
        V4<T>::ld(ch + CQ * (x + (q >> 2)), c1);
        V4<T>::ld(ch + CQ * (x + (q >> 1)), c2);
        V4<T>::ld(ch + CQ * (x + 3 * (q >> 2)), c3);
        float u0[4], u1[4];
        if (m1()) {
            const unsigned bl = b1[x >> 3] >> ((x & 7) * 4);
            const int xh = x + (q >> 2);
            const unsigned bh = b1[xh >> 3] >> ((xh & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                u0[j] = g_op_bits<T>(c0[j], c2[j], bl, j);
                u1[j] = g_op_bits<T>(c1[j], c3[j], bh, j);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                u0[j] = f_op(c0[j], c2[j]);
                u1[j] = f_op(c1[j], c3[j]);
            }
        }
        if (m2()) {
            const unsigned b = b2[x >> 3] >> ((x & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(u0[j], u1[j], b, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(u0[j], u1[j]);
        }
    }
    __device__ __forceinline__ float v1(int i) const {
        const float a = Elem<T>::ld(che(ch, i)), b = Elem<T>::ld(che(ch, i + 2 * q));
        return m1() ? g_op<T>(a, b, (b1[i >> 5] >> (i & 31)) & 1u) : f_op(a, b);
    }
    __device__ __forceinline__ float get(int i) const {
        const float a = v1(i), b = v1(i + q);
        return m2() ? g_op<T>(a, b, (b2[i >> 5] >> (i & 31)) & 1u) : f_op(a, b);
    }
    struct Words {
        uint32_t wl, wh, w2;
    };
    __device__ __forceinline__ Words words(int x) const {
        return Words{m1() ? b1[x >> 3] : 0u, m1() ? b1[(x + (q >> 2)) >> 3] : 0u, m2() ? b2[x >> 3] : 0u};
    }
    __device__ __forceinline__ void quadw(int x, float (&v)[4], const Words &w) const {
        float c0[4], c1[4], c2[4], c3[4];
        V4<T>::ld(ch + CQ * x, c0);
        V4<T>::ld(ch + CQ * (x + (q >> 2)), c1);
        V4<T>::ld(ch + CQ * (x + (q >> 1)), c2);
        V4<T>::ld(ch + CQ * (x + 3 * (q >> 2)), c3);
        const int sh = (x & 7) * 4;
        float u0[4], u1[4];
        if (m1()) {
            const unsigned bl = w.wl >> sh, bh = w.wh >> sh;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                u0[j] = g_op_bits<T>(c0[j], c2[j], bl, j);
                u1[j] = g_op_bits<T>(c1[j], c3[j], bh, j);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                u0[j] = f_op(c0[j], c2[j]);
                u1[j] = f_op(c1[j], c3[j]);
            }
        }
        if (m2()) {
            const unsigned b = w.w2 >> sh;
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(u0[j], u1[j], b, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(u0[j], u1[j]);
        }
    }
};
template <typename T>
__device__ __forceinline__ V1Ld<T> make_v1(const Fr<T> &F, int flags) {
    const int n = LK_C(F.P, n);
    return V1Ld<T>{F.channel(), F.beta_row(n - 1, get8(F.ib, n - 1)), LK_C(F.P, N) >> 1, (flags & LF_V1G) != 0};
}
template <typename T>
__device__ __forceinline__ V2Ld<T> make_v2(const Fr<T> &F, int flags) {
    const int n = LK_C(F.P, n);
    return V2Ld<T>{F.channel(), F.beta_row(n - 1, get8(F.ib, n - 1)), F.beta_row(n - 2, get8(F.ib, n - 2)),
                   LK_C(F.P, N) >> 2, (flags & LF_V1G) != 0, (flags & LF_V2G) != 0};
}
// A leaf's LLRs.  Plain: its stage's stored row (leaves under a recomputed
// stage read the staging row the F / G before them wrote, runtime.cu) or the
// channel (a root leaf).  Fused (LF_FUSE_F / LF_FUSE_G): the F / G that would
// have produced the leaf's row is folded into the read -- the leaf reads the
// two halves of its parent's row (stage t + 1) and applies f, or g with the
// path's left-sibling bits (beta slot t); the row of stage t is never stored
// (listdec.py:317-326 followed by :334-394 on the same values).
template <typename T>
struct LeafLd {
    const T *p;          // the row read: stage t (plain) or t + 1 (fused)
    int qs;              // quad stride in elements (128 stored rows, 4 channel)
    int mode;            // 0 plain, 1 f, 2 g
    int m;               // leaf size
    const uint32_t *bw;  // g: beta row of slot t
    __device__ __forceinline__ void quad(int x, float (&v)[4]) const {
        if (mode == 0) {
            V4<T>::ld(p + x * qs, v);
            return;
        }
        float a[4], b[4];
        V4<T>::ld(p + x * qs, a);
        V4<T>::ld(p + (x + (m >> 2)) * qs, b);
        if (mode == 2) {
            const unsigned bits = bw[x >> 3] >> ((x & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(a[j], b[j], bits, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(a[j], b[j]);
        }
    }
    // the same read in two steps (leaf_scan_lane keeps the next block's loads
    // in flight while it works on the current one)
    struct Raw {
        float a[4], b[4];
        unsigned w;
    };
    __device__ __forceinline__ void raw(int x, Raw &r) const {
        V4<T>::ld(p + x * qs, r.a);
        if (mode != 0) V4<T>::ld(p + (x + (m >> 2)) * qs, r.b);
        if (mode == 2) r.w = bw[x >> 3];
    }
    __device__ __forceinline__ void fin(int x, const Raw &r, float (&v)[4]) const {
        if (mode == 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = r.a[j];
        } else if (mode == 2) {
            const unsigned bits = r.w >> ((x & 7) * 4);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(r.a[j], r.b[j], bits, j);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = f_op(r.a[j], r.b[j]);
        }
    }
    __device__ __forceinline__ float el(int i) const { return Elem<T>::ld(p + (i >> 2) * qs + (i & 3)); }
    __device__ __forceinline__ float get(int i) const {
        if (mode == 0) return el(i);
        const float a = el(i), b = el(i + m);
        return mode == 2 ? g_op<T>(a, b, (bw[i >> 5] >> (i & 31)) & 1u) : f_op(a, b);
    }
};
template <typename T, class OP>
__device__ __forceinline__ LeafLd<T> leaf_src(const Fr<T> &F, const OP &o, int t, const uint32_t (&ia)[4]) {
    const int mode = (o.flags() >> LF_FUSE_SHIFT) & 3;
    const int ps = mode ? t + 1 : t;
    const uint32_t *bw = mode == 2 ? F.beta_row(t, get8(F.ib, t)) : nullptr;
    if (o.src() == S_CH) return LeafLd<T>{F.channel(), CQ, mode, 1 << t, bw};
    return LeafLd<T>{F.a_row(ps, get8(ia, ps)), 128, mode, 1 << t, bw};
}

// ---------------------------------------------------------------- F / G

template <typename T, bool IS_G, int U, class S>
__device__ __forceinline__ void fg_body(const S &src, T *dst, const uint32_t *bw, int h) {
    if (h < 4) {  // stage 1 / 2: one (padded) quad
        float o4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < h; ++i) {
            const float a = src.get(i), b = src.get(i + h);
            o4[i] = IS_G ? g_op<T>(a, b, (bw[0] >> i) & 1u) : f_op(a, b);
        }
        V4<T>::st(dst, o4);
        return;
    }
    const int nq = h >> 2;
    int x0 = 0;
    for (; x0 + U <= nq; x0 += U) {
        float a[U][4], b[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            src.quad(x0 + u, a[u]);
            src.quad(x0 + u + nq, b[u]);
        }
        unsigned wd[(U + 7) / 8];  // 8 quads per 32-bit beta word (x0 is a multiple of U)
#pragma unroll
        for (int w = 0; w < (U + 7) / 8; ++w) wd[w] = IS_G ? bw[(x0 >> 3) + w] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float o[4];
            const unsigned bits = IS_G ? wd[u >> 3] >> (((x0 + u) & 7) * 4) : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = IS_G ? g_op_bits<T>(a[u][j], b[u][j], bits, j) : f_op(a[u][j], b[u][j]);
            V4<T>::st(dst + (x0 + u) * 128, o);
        }
    }
    for (; x0 < nq; ++x0) {
        float a[4], b[4], o[4];
        src.quad(x0, a);
        src.quad(x0 + nq, b);
        const unsigned bits = IS_G ? bw[x0 >> 3] >> ((x0 & 7) * 4) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = IS_G ? g_op_bits<T>(a[j], b[j], bits, j) : f_op(a[j], b[j]);
        V4<T>::st(dst + x0 * 128, o);
    }
}

// F / G over a recomputed source: blocks of 8 quads share their beta words
// (the source's and the G's), loaded once per block; U quads in flight
template <typename T, bool IS_G, int U, class S>
__device__ __forceinline__ void fg_body_v(const S &src, T *dst, const uint32_t *bw, int h) {
    const int nq = h >> 2;  // >= 8 (callers take fg_body below)
    for (int x0 = 0; x0 < nq; x0 += 8) {
        const typename S::Words wa = src.words(x0), wb = src.words(x0 + nq);
        const unsigned wd = IS_G ? bw[x0 >> 3] : 0u;
#pragma unroll 1
        for (int u0 = 0; u0 < 8; u0 += U) {
            float a[U][4], b[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                src.quadw(x0 + u0 + u, a[u], wa);
                src.quadw(x0 + u0 + u + nq, b[u], wb);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float o[4];
                const unsigned bits = IS_G ? wd >> ((u0 + u) * 4) : 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    o[j] = IS_G ? g_op_bits<T>(a[u][j], b[u][j], bits, j) : f_op(a[u][j], b[u][j]);
                V4<T>::st(dst + (x0 + u0 + u) * 128, o);
            }
        }
    }
}

// F / G of stage s into the path's own row of stage s-1 (listdec.py:317-326)
// F / G while a frame still has a single path (the ops before its first
// fork): the frame's lanes split the row's quads instead of one lane walking
// the whole row (specialised build: the path count is a constant there).
template <typename T, bool IS_G, class S>
__device__ __forceinline__ void fg_single_body(const S &src, T *dst, const uint32_t *bw, int nq, int x0, int step) {
    for (int x = x0; x < nq; x += step) {
        float a[4], b[4], o[4];
        src.quad(x, a);
        src.quad(x + nq, b);
        const unsigned bits = IS_G ? bw[x >> 3] >> ((x & 7) * 4) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = IS_G ? g_op_bits<T>(a[j], b[j], bits, j) : f_op(a[j], b[j]);
        V4<T>::st(dst + x * 128, o);
    }
}
template <typename T, bool IS_G, int SRC, int DST, class OP>
__device__ __forceinline__ void fg_single(Fr<T> &F, const OP &o) {
    const int s = o.stage(), nq = 1 << (s - 3), n = LK_C(F.P, n);
    const int b0 = F.base();  // the lane of the frame's only path
    uint32_t ia0[4], ib0[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ia0[j] = __shfl_sync(FULL_MASK, F.ia[j], b0);
        ib0[j] = __shfl_sync(FULL_MASK, F.ib[j], b0);
    }
    T *dst = F.template a_row_t<DST>(s - 1, b0);
    const uint32_t *bw = IS_G ? F.beta_row(s - 1, get8(ib0, s - 1)) : nullptr;
    const int x0 = F.slot(), step = Fr<T>::LP;
    if (SRC == S_V2) {
        const V2Ld<T> v{F.channel(), F.beta_row(n - 1, get8(ib0, n - 1)), F.beta_row(n - 2, get8(ib0, n - 2)),
                        LK_C(F.P, N) >> 2, (o.flags() & LF_V1G) != 0, (o.flags() & LF_V2G) != 0};
        fg_single_body<T, IS_G>(v, dst, bw, nq, x0, step);
    } else if (SRC == S_V1) {
        const V1Ld<T> v{F.channel(), F.beta_row(n - 1, get8(ib0, n - 1)), LK_C(F.P, N) >> 1,
                        (o.flags() & LF_V1G) != 0};
        fg_single_body<T, IS_G>(v, dst, bw, nq, x0, step);
    } else if (SRC == S_CH) {
        fg_single_body<T, IS_G>(RowLd<T>{F.channel(), CQ}, dst, bw, nq, x0, step);
    } else {
        fg_single_body<T, IS_G>(RowLd<T>{F.template a_row_t<SRC>(s, get8(ia0, s)), 128}, dst, bw, nq, x0, step);
    }
    __syncwarp();
    if (SRC == S_GL && (o.flags() & LF_LAST)) F.discard_stage(s);
    set8(F.ia, s - 1, F.lane);
}

template <typename T, bool IS_G, int SRC, int DST, class OP>
__device__ __forceinline__ void fg_op(Fr<T> &F, const OP &o) {
    const int s = o.stage(), h = 1 << (s - 1);
#ifdef PB_JIT
    if (o.pin() == 1 && h >= 4) {
        fg_single<T, IS_G, SRC, DST>(F, o);
        return;
    }
#endif
    if (F.slot() < o.pin()) {
        T *dst = F.template a_row_t<DST>(s - 1, F.lane);
        const uint32_t *bw = IS_G ? F.beta_row(s - 1, get8(F.ib, s - 1)) : nullptr;
        if (SRC == S_V2) {
            // the recomputed stages' F / G modes are fixed for the whole op:
            // one loop per mode pair, no per-quad branches
            const V2Ld<T> v = make_v2(F, o.flags());
            if (h < 32) {
                fg_body<T, IS_G, 2>(v, dst, bw, h);
            } else if (!PB_LANE_V2SPEC) {
                fg_body_v<T, IS_G, 2>(v, dst, bw, h);
            } else switch ((v.g1_ ? 1 : 0) | (v.g2_ ? 2 : 0)) {
                case 0: fg_body_v<T, IS_G, 2>(V2Ld<T, 0>{v.ch, v.b1, v.b2, v.q, false, false}, dst, bw, h); break;
                case 1: fg_body_v<T, IS_G, 2>(V2Ld<T, 1>{v.ch, v.b1, v.b2, v.q, true, false}, dst, bw, h); break;
                case 2: fg_body_v<T, IS_G, 2>(V2Ld<T, 2>{v.ch, v.b1, v.b2, v.q, false, true}, dst, bw, h); break;
                default: fg_body_v<T, IS_G, 2>(V2Ld<T, 3>{v.ch, v.b1, v.b2, v.q, true, true}, dst, bw, h); break;
            }
        } else if (SRC == S_V1) {
            const V1Ld<T> v = make_v1(F, o.flags());
            if (h < 32)
                fg_body<T, IS_G, 4>(v, dst, bw, h);
            else if (v.g_)
                fg_body_v<T, IS_G, 4>(V1Ld<T, 1>{v.ch, v.b1, v.half, true}, dst, bw, h);
            else
                fg_body_v<T, IS_G, 4>(V1Ld<T, 0>{v.ch, v.b1, v.half, false}, dst, bw, h);
        } else if (SRC == S_CH) {
            fg_body<T, IS_G, 4>(RowLd<T>{F.channel(), CQ}, dst, bw, h);
        } else {
            const RowLd<T> src{F.template a_row_t<SRC>(s, get8(F.ia, s)), 128};
            fg_body<T, IS_G, SRC == S_GL ? 8 : 4>(src, dst, bw, h);
        }
    }
    if (SRC == S_GL && (o.flags() & LF_LAST)) {
        __syncwarp();
        F.discard_stage(s);
    }
    set8(F.ia, s - 1, F.lane);
}

// ------------------------------------------------------------- leaves

// numpy float32 pairwise sums (listdec.py:341,348-350): n < 8 sequential;
// 8 <= n <= 128 eight strided accumulators combined ((0+1)+(2+3))+((4+5)+(6+7));
// larger n halves recursively (a balanced tree of 128-element blocks).
// NS = 1: sum min(a,0); NS = 3: (sum min(a,0), sum max(a,0), sum a).
template <int NS, class S>
__device__ __forceinline__ void pw_sums_lane(const S &src, int m, float (&out)[NS]) {
    if (m < 8) {
        float r[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) r[t] = 0.f;
        if (m >= 4) {
            float q[4];
            src.quad(0, q);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc_add<NS>(r, q[j]);
        } else {
            for (int i = 0; i < m; ++i) acc_add<NS>(r, src.get(i));
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) out[t] = r[t];
        return;
    }
    const int blk = m < 128 ? m : 128, nb = m / blk, per = blk >> 3;
    float stk[10][NS];
    float carry[NS];
    for (int b = 0; b < nb; ++b) {
        float acc[8][NS];
        const int xb = (b * blk) >> 2;
        {
            float q0[4], q1[4];
            src.quad(xb, q0);
            src.quad(xb + 1, q1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc_init<NS>(acc[j], q0[j]);
                acc_init<NS>(acc[j + 4], q1[j]);
            }
        }
        for (int r = 1; r < per; ++r) {
            float q0[4], q1[4];
            src.quad(xb + 2 * r, q0);
            src.quad(xb + 2 * r + 1, q1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                acc_add<NS>(acc[j], q0[j]);
                acc_add<NS>(acc[j + 4], q1[j]);
            }
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) {
            const float s01 = __fadd_rn(acc[0][t], acc[1][t]), s23 = __fadd_rn(acc[2][t], acc[3][t]);
            const float s45 = __fadd_rn(acc[4][t], acc[5][t]), s67 = __fadd_rn(acc[6][t], acc[7][t]);
            acc[0][t] = __fadd_rn(__fadd_rn(s01, s23), __fadd_rn(s45, s67));
        }
        // combine block sums in numpy's halving order (binary counter)
#pragma unroll
        for (int t = 0; t < NS; ++t) carry[t] = acc[0][t];
        int lvl = 0;
        while ((b >> lvl) & 1) {
#pragma unroll
            for (int t = 0; t < NS; ++t) carry[t] = __fadd_rn(stk[lvl][t], carry[t]);
            ++lvl;
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) stk[lvl][t] = carry[t];
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) out[t] = carry[t];
}

// Rate-1 / SPC scan: stable K least reliable positions (argsort kind="stable",
// listdec.py:362,375), hard-decision word(s), parity.  Returns the parity;
// `hard` = the hard word when m <= 32.
template <int K, class S>
__device__ __forceinline__ int leaf_scan_lane(const S &src, int m, TopK<K> &tk, uint32_t &hard, uint32_t *hw) {
    tk.init();
    int par = 0;
    hard = 0u;
    if (m >= 32) {
        constexpr int NCH = K == 2 ? 4 : 2;
        TopK<K> tc[NCH];
#pragma unroll
        for (int h = 0; h < NCH; ++h) tc[h].init();
#if defined(PB_JIT) && PB_SCAN_PIPE
        // software pipeline over blocks of QB quads: the loads of block b + 1
        // are issued before block b is scanned (the rows of wide leaves live
        // in global scratch: an L2 round trip per block otherwise)
        constexpr int QB = PB_SCAN_PIPE, EB = 4 * QB, BPW = 32 / EB;  // blocks per 32-bit hard word (4-quad blocks: 4.62 against 4.65 Gbit/s)
        typename S::Raw buf[2][QB];
        const int nb = m / EB;
        auto ld = [&](int b, typename S::Raw(&r)[QB]) {
#pragma unroll
            for (int j = 0; j < QB; ++j) src.raw(b * QB + j, r[j]);
        };
        auto scan = [&](int b, const typename S::Raw(&r)[QB], uint32_t &word) {
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                float q[4];
                src.fin(b * QB + j, r[j], q);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = b * EB + 4 * j + e;
                    word |= (q[e] < 0.f ? 1u : 0u) << (i & 31);
                    tc[(4 * j + e) % NCH].push_scan(fabsf(q[e]), i);
                }
            }
        };
        ld(0, buf[0]);
        uint32_t word = 0u;
        for (int b = 0; b < nb; b += 2) {  // nb is even (m >= 32, EB <= 16)
            ld(b + 1, buf[1]);
            scan(b, buf[0], word);
            if (b + 2 < nb) ld(b + 2, buf[0]);
            scan(b + 1, buf[1], word);
            if (((b + 2) % BPW) == 0) {
                hard = word;
                if (m > 32) hw[((b + 1) / BPW) * 32] = word;
                par ^= __popc(word);
                word = 0u;
            }
        }
#else
        for (int w0 = 0; w0 < m; w0 += 32) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float q[4];
                src.quad((w0 >> 2) + j, q);
#pragma unroll
                for (int e = 0; e < 4; ++e) v[4 * j + e] = q[e];
            }
            uint32_t word = 0u;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                word |= (v[j] < 0.f ? 1u : 0u) << j;
                tc[j % NCH].push_scan(fabsf(v[j]), w0 + j);
            }
            hard = word;
            if (m > 32) hw[(w0 >> 5) * 32] = word;
            par ^= __popc(word);
        }
#endif
        tk = tc[0];
#pragma unroll
        for (int h = 1; h < NCH; ++h)
#pragma unroll
            for (int e = 0; e < K; ++e) tk.insert(tc[h].m[e], tc[h].i[e]);
    } else if (K == 4 && m == 4) {
        // SPC of size 4 (the default cap): every position is a least
        // reliable one -- a stable 5-comparator sort of (|a|, index)
        float q[4];
        src.quad(0, q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            hard |= (q[e] < 0.f ? 1u : 0u) << e;
            tk.m[e] = fabsf(q[e]);
            tk.i[e] = e;
        }
        auto cx = [&](int a, int b) {  // (m, i) lexicographic: a before b
            const bool sw = tk.m[b] < tk.m[a] || (tk.m[b] == tk.m[a] && tk.i[b] < tk.i[a]);
            const float ma = tk.m[a], mb = tk.m[b];
            const int ia = tk.i[a], ib = tk.i[b];
            tk.m[a] = sw ? mb : ma;
            tk.m[b] = sw ? ma : mb;
            tk.i[a] = sw ? ib : ia;
            tk.i[b] = sw ? ia : ib;
        };
        cx(0, 1);
        cx(2, 3);
        cx(0, 2);
        cx(1, 3);
        cx(1, 2);
        par = __popc(hard);
    } else if (m >= 4) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (4 * j < m) {
                float q[4];
                src.quad(j, q);
#pragma unroll
                for (int e = 0; e < 4; ++e) v[4 * j + e] = q[e];
            }
        if (m <= 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < m) {
                    hard |= (v[j] < 0.f ? 1u : 0u) << j;
                    tk.push_scan(fabsf(v[j]), j);
                }
        }
        par = __popc(hard);
    } else {
        for (int j = 0; j < m; ++j) {
            const float a = src.get(j);
            hard |= (a < 0.f ? 1u : 0u) << j;
            tk.push_scan(fabsf(a), j);
        }
        par = __popc(hard);
    }
    return par;
}

// SPC flip sets relative to the ML word over the four LRB slots, emission
// order of listdec.py:157 (_SPC_PAIRS)
__device__ __forceinline__ int lk_flip_mask(int kind, int c, int odd) {
    if (kind == K_R1) return c;  // (), (b1), (b2), (b1, b2)
    const int ml = odd ? 1 : 0;
    return c == 0 ? ml : (kSpcPairs[c - 1] ^ ml);
}

// Phase A of a leaf for this lane's path: Rate-0 adds to the metric;
// forking leaves produce candidate keys okey(pm + delta) in candidate order
// and the leaf data the survivors will need.  Returns false for Rate-0.
template <typename T, class OP>
__device__ __forceinline__ void leaf_phase_a(Fr<T> &F, const OP &o, int kind, long long (&key)[8]) {
    const int t = o.stage(), m = 1 << t;
    const LeafLd<T> src = leaf_src(F, o, t, F.ia);
    if (kind == K_R0) {  // listdec.py:340-346
        float r[1];
        pw_sums_lane<1>(src, m, r);
        F.pm += (double)r[0];
        return;
    }
    double cd[8];
    if (kind == K_REP) {  // listdec.py:347-359
        float r[3];
        pw_sums_lane<3>(src, m, r);
        const bool ones_first = r[2] < 0.f;
        const double neg = (double)r[0], pos = (double)r[1];
        cd[0] = ones_first ? -pos : neg;
        cd[1] = ones_first ? neg : -pos;
        F.lflag = ones_first;
#pragma unroll
        for (int c = 2; c < 8; ++c) cd[c] = 0.0;
    } else if (kind == K_R1) {  // listdec.py:360-372
        TopK<2> tk;
        uint32_t hard;
        leaf_scan_lane<2>(src, m, tk, hard, F.hard_words() + F.lane);
        F.hard = hard;
        F.lrb01 = (uint32_t)tk.i[0] | ((uint32_t)tk.i[1] << 16);
        F.lrb23 = 0u;
        F.lflag = 0u;
        const double w1 = (double)tk.m[0], w2 = (double)tk.m[1];
        cd[0] = 0.0;
        cd[1] = -w1;
        cd[2] = -w2;
        cd[3] = -(w1 + w2);
#pragma unroll
        for (int c = 4; c < 8; ++c) cd[c] = 0.0;
    } else {  // SPC, listdec.py:373-394
        TopK<4> tk;
        uint32_t hard;
        const int par = leaf_scan_lane<4>(src, m, tk, hard, F.hard_words() + F.lane);
        const int odd = par & 1;
        F.hard = hard;
#pragma unroll
        for (int x = 0; x < 4; ++x)
            if (tk.i[x] >= m) tk.i[x] = 0;  // m < 4 never happens (SPC >= 4)
        F.lrb01 = (uint32_t)tk.i[0] | ((uint32_t)tk.i[1] << 16);
        F.lrb23 = (uint32_t)tk.i[2] | ((uint32_t)tk.i[3] << 16);
        F.lflag = odd;
        // deltas: minus the sum of the net flips' magnitudes in ascending
        // position order (Python's sum from 0: 0.0 + w is w exactly, and an
        // empty flip set gives pm + -0.0 == pm).  rbit[x] = bit of LRB slot x
        // in position-rank order; wr[r] = magnitude of the r-th by position.
        uint32_t rbit[4];
        double wr[4];
        if (m == 4) {  // the four positions are 0..3: rank = position
#pragma unroll
            for (int x = 0; x < 4; ++x) rbit[x] = 1u << tk.i[x];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double v = 0.0;
#pragma unroll
                for (int x = 0; x < 4; ++x) v = tk.i[x] == r ? (double)tk.m[x] : v;
                wr[r] = v;
            }
        } else {
            int rk[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                rk[x] = 0;
#pragma unroll
                for (int y = 0; y < 4; ++y) rk[x] += tk.i[y] < tk.i[x] ? 1 : 0;
                rbit[x] = 1u << rk[x];
            }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                double v = 0.0;
#pragma unroll
                for (int x = 0; x < 4; ++x) v = rk[x] == r ? (double)tk.m[x] : v;
                wr[r] = v;
            }
        }
        // flip sets in rank bits: ML {lrb0} if odd, then the pairs of
        // _SPC_PAIRS (listdec.py:157) and all four, each XOR the ML set
        const uint32_t ml = odd ? rbit[0] : 0u;
        uint32_t fr[8];
        fr[0] = ml;
        fr[1] = (rbit[0] | rbit[1]) ^ ml;
        fr[2] = (rbit[0] | rbit[2]) ^ ml;
        fr[3] = (rbit[0] | rbit[3]) ^ ml;
        fr[4] = (rbit[1] | rbit[2]) ^ ml;
        fr[5] = (rbit[1] | rbit[3]) ^ ml;
        fr[6] = (rbit[2] | rbit[3]) ^ ml;
        fr[7] = 0xfu ^ ml;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if ((fr[c] >> r) & 1u) acc += wr[r];
            cd[c] = -acc;
        }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) key[c] = okey(F.pm + cd[c]);
}

// ------------------------------------------------------------ selection

// the top 27 bits of the order-preserving metric key (sign, exponent, 15
// mantissa bits; weakly monotone), low 5 bits free for a lane id
__device__ __forceinline__ int hi27(long long k) { return (int)(k >> 32) & ~31; }

// The survivors of one forking leaf: bit c of the result = candidate c of
// this lane's path survives.  Exactly the list_size best (source, cand)
// pairs by (metric desc, source asc, cand asc) == the bounded heap of
// listdec.py:63-100 (tests/oracles.py:74-89).
//
// Pass 1 finds the L-th best 27-bit key prefix Th by a k-way merge: each
// lane's candidates form a sorted column and expose their best unconsumed
// one; the kept set (slot = lane) trades its worst for the best exposed
// candidate while that is strictly better.  Exposed keys carry their source
// lane and kept keys their slot in the low 5 bits, so one REDUX max / min
// names both lanes (no ballots): 2 independent REDUX per iteration.  Every
// candidate whose prefix is > Th survives; among those == Th the `need`
// best by full key survive, ties to the earlier (source, cand).
// 64-bit max / min and the 4-bit exclusive scan over the lanes of one frame
__device__ __forceinline__ long long seg_max_ll(long long v, unsigned seg) {
    const int hi = (int)(v >> 32);
    const int mh = __reduce_max_sync(seg, hi);
    const unsigned ml = __reduce_max_sync(seg, hi == mh ? (unsigned)v : 0u);
    return ((long long)mh << 32) | ml;
}
__device__ __forceinline__ long long seg_min_ll(long long v, unsigned seg) {
    const int hi = (int)(v >> 32);
    const int mh = __reduce_min_sync(seg, hi);
    const unsigned ml = __reduce_min_sync(seg, hi == mh ? (unsigned)v : 0xffffffffu);
    return ((long long)mh << 32) | ml;
}
// votes = seg where the frames of a warp may have diverged (the tie path of
// the selection), else FULL_MASK: one vote for the whole warp instead of one
// per frame (votes with different masks do not share an instruction: c1 L=4
// 7.1 -> 5.7 Gbit/s when every leaf voted per frame)
__device__ __forceinline__ int seg_excl_scan4(int v, int lane, unsigned seg, unsigned votes) {
    const unsigned below = ((1u << lane) - 1u) & seg;
    int r = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) r += __popc(__ballot_sync(votes, (v >> b) & 1) & below) << b;
    return r;
}

// (lane = the warp lane: it tags the keys; slot = the path slot within the
// frame; seg = the frame's lanes: every reduction runs over them only)
template <int C>
__device__ __forceinline__ unsigned select_mask(const long long (&key)[8], bool valid, int L, int lane, int slot,
                                                unsigned seg) {
    int srt[C];
#pragma unroll
    for (int c = 0; c < C; ++c) srt[c] = (valid ? hi27(key[c]) : INT_MIN) | lane;
    auto cs = [&](int a, int b) {
        const int x = srt[a], y = srt[b];
        srt[a] = max(x, y);
        srt[b] = min(x, y);
    };
    if (C == 2) {
        cs(0, 1);
    } else if (C == 4) {  // Rate-1 columns are already sorted (0 >= -m1 >= -m2 >= -(m1+m2))
        cs(0, 1); cs(2, 3); cs(0, 2); cs(1, 3); cs(1, 2);
    } else {  // Batcher odd-even merge sort, 19 comparators
        cs(0, 1); cs(2, 3); cs(4, 5); cs(6, 7);
        cs(0, 2); cs(1, 3); cs(4, 6); cs(5, 7);
        cs(1, 2); cs(5, 6);
        cs(0, 4); cs(1, 5); cs(2, 6); cs(3, 7);
        cs(2, 4); cs(3, 5);
        cs(1, 2); cs(3, 4); cs(5, 6);
    }
    int kept = slot < L ? ((srt[0] & ~31) | lane) : INT_MAX;
#pragma unroll
    for (int c = 0; c < C; ++c) srt[c] = c + 1 < C ? srt[c + 1 < C ? c + 1 : c] : (INT_MIN | lane);
    int worst;
    for (;;) {
        const int best = __reduce_max_sync(seg, srt[0]);
        worst = __reduce_min_sync(seg, kept);
        if ((best & ~31) <= (worst & ~31)) break;
        if (lane == (best & 31)) {
#pragma unroll
            for (int c = 0; c < C; ++c) srt[c] = c + 1 < C ? srt[c + 1 < C ? c + 1 : c] : (INT_MIN | lane);
        }
        if (lane == (worst & 31)) kept = (best & ~31) | lane;
    }
    const int Th = worst & ~31;
    unsigned mask = 0u, bmask = 0u;
    int gt = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int hk = valid ? hi27(key[c]) : INT_MIN;
        if (hk > Th) {
            mask |= 1u << c;
            ++gt;
        } else if (valid && hk == Th) {
            bmask |= 1u << c;
        }
    }
    const int need = L - (int)__reduce_add_sync(seg, (unsigned)gt);
    const int eqt = (int)__reduce_add_sync(seg, (unsigned)__popc(bmask));
    if (eqt <= need) return mask | bmask;  // the usual case: no surplus at the threshold
    // surplus at Th: full keys decide, then (source, cand)
    long long bmax = LLONG_MIN, bmin = LLONG_MAX;
#pragma unroll
    for (int c = 0; c < C; ++c)
        if ((bmask >> c) & 1u) {
            bmax = max(bmax, key[c]);
            bmin = min(bmin, key[c]);
        }
    if (seg_max_ll(bmax, seg) == seg_min_ll(bmin, seg)) {
        // all tied exactly (int8 mode): the earliest `need` in (source, cand) order
        int r = seg_excl_scan4(__popc(bmask), lane, seg, seg);
#pragma unroll
        for (int c = 0; c < C; ++c)
            if ((bmask >> c) & 1u) {
                if (r < need) mask |= 1u << c;
                ++r;
            }
        return mask;
    }
    // one survivor at a time by (full key desc, source asc, cand asc)
    for (int it = 0; it < need; ++it) {
        long long mine = LLONG_MIN;
        int mc = -1;
#pragma unroll
        for (int c = 0; c < C; ++c)
            if (((bmask >> c) & 1u) && key[c] > mine) {
                mine = key[c];
                mc = c;
            }
        const long long best = seg_max_ll(mine, seg);
        const int from = __ffs(__ballot_sync(seg, mc >= 0 && mine == best) & seg) - 1;
        if (lane == from) {
            mask |= 1u << mc;
            bmask &= ~(1u << mc);
        }
    }
    return mask;
}

// ------------------------------------------------------- materialisation

// word w (m >= 32) / the m-bit value (m < 32) of decision c of a path whose
// leaf data is (hard, lrb, flag); hw = the source path's hard words when the
// leaf is wider than one word
__device__ __forceinline__ uint32_t leaf_word(int kind, int m, int c, uint32_t hard, uint32_t l01, uint32_t l23,
                                              uint32_t flag, const uint32_t *hw, int w) {
    const uint32_t fullw = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
    if (kind == K_R0) return 0u;
    if (kind == K_REP) {
        const bool ones = flag ? (c == 0) : (c == 1);
        return ones ? fullw : 0u;
    }
    const uint32_t v0 = m > 32 ? hw[w * 32] : hard;
    uint32_t v = v0;
    const int fm = lk_flip_mask(kind, c, (int)flag);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if ((fm >> j) & 1) {
            const int pos = (int)(((j < 2 ? l01 : l23) >> ((j & 1) * 16)) & 0xffffu);
            if ((pos >> 5) == w) v ^= 1u << (pos & 31);
        }
    return v;
}

// The slot-sE row a leaf's chain of Combines produces (listdec.py:327-332):
// level by level dst[E - 2^(s+1), E - 2^s) = slot_s[row_s] ^ dst[E - 2^s, E),
// i.e. unrolled, bit j of the row is
//   leaf[j mod m] ^ XOR_{s in [t, sE), bit s of j clear} slot_s[j mod 2^s].
// The levels below 32 bits only depend on j mod 32: one register pattern R
// (computed level by level); the word levels make word w
//   base(w) ^ XOR_{s >= 5, bit (s-5) of w clear} slot_s[w mod 2^(s-5)]
// with base = R (leaf narrower than a word) or the leaf word w mod (m/32).
// No word depends on another, so a block's loads (every level) are in flight
// together instead of one memory round trip per level.  Words w0, w0 + step,
// ... of the row; ib = the path's beta rows.
template <typename T>
__device__ __forceinline__ void chain_row(const Fr<T> &F, int kind, int t, int sE, const uint32_t (&ib)[4],
                                          uint32_t *dst, const uint32_t *hw, int c, uint32_t hard, uint32_t l01,
                                          uint32_t l23, uint32_t flag, int w0, int step) {
    const int m = 1 << t, E = 1 << sE;
    uint32_t R = 0u;
    if (m < 32) {
        const int s_sub = sE < 5 ? sE : 5;
        const int W0 = E >= 32 ? E - 32 : 0;
        R = leaf_word(kind, m, c, hard, l01, l23, flag, hw, 0) << (E - m - W0);
        for (int s = t; s < s_sub; ++s) {
            const uint32_t sl = F.beta_row(s, get8(ib, s))[0];
            const int seg = 1 << s;
            R |= ((sl ^ (R >> (E - seg - W0))) & ((1u << seg) - 1u)) << (E - 2 * seg - W0);
        }
        if (E <= 32) {
            if (w0 == 0) dst[0] = E == 32 ? R : (R & ((1u << E) - 1u));
            return;
        }
    }
    const int s0 = t > 5 ? t : 5;
    const int nw = E >> 5, lw = m >= 32 ? (m >> 5) - 1 : 0;
    if (step == 1 && (nw < PB_CHAIN_CLOSED_MIN || sE - s0 > 6)) {
        // short rows (and very deep chains): level by level, each level's
        // words from the one below (the recursion as written)
        if (m >= 32) {
            for (int w = 0; w < (m >> 5); ++w)
                dst[((E - m) >> 5) + w] = leaf_word(kind, m, c, hard, l01, l23, flag, hw, w);
        } else {
            dst[nw - 1] = R;
        }
        for (int s = s0; s < sE; ++s) {
            const int seg = 1 << s, nws = seg >> 5;
            const uint32_t *sl = F.beta_row(s, get8(ib, s));
            uint32_t *da = dst + ((E - 2 * seg) >> 5);
            const uint32_t *db = dst + ((E - seg) >> 5);
            int w = 0;
            for (; w + 4 <= nws; w += 4) {
                uint32_t a[4], b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u] = sl[w + u];
                    b[u] = db[w + u];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) da[w + u] = a[u] ^ b[u];
            }
            for (; w < nws; ++w) da[w] = sl[w] ^ db[w];
        }
        return;
    }
    constexpr int NL = 6;  // word levels handled unrolled (N <= 2048: all of them)
    const uint32_t *sl[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) sl[i] = s0 + i < sE ? F.beta_row(s0 + i, get8(ib, s0 + i)) : nullptr;
    for (int wb = w0; wb < nw; wb += 8 * step) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int w = wb + u * step;
            v[u] = m >= 32 ? (w < nw ? leaf_word(kind, m, c, hard, l01, l23, flag, hw, w & lw) : 0u) : R;
        }
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            if (s0 + i < sE) {
                const int sh = s0 + i - 5, msk = (1 << sh) - 1;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int w = wb + u * step;
                    if (w < nw && !((w >> sh) & 1)) v[u] ^= sl[i][w & msk];
                }
            }
        }
        for (int s = s0 + NL; s < sE; ++s) {  // deeper chains (N > 2048, warp mode)
            const uint32_t *q = F.beta_row(s, get8(ib, s));
            const int sh = s - 5, msk = (1 << sh) - 1;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int w = wb + u * step;
                if (w < nw && !((w >> sh) & 1)) v[u] ^= q[w & msk];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (wb + u * step < nw) dst[wb + u * step] = v[u];
    }
}

// Leaf word of this lane's survivor and its chain into slot sE's own row
template <typename T, class OP>
__device__ __forceinline__ void write_chain(Fr<T> &F, const OP &o, int kind, uint32_t *dst, int p, int c,
                                            uint32_t hard, uint32_t l01, uint32_t l23, uint32_t flag) {
    chain_row(F, kind, o.stage(), o.aux(), F.ib, dst, F.hard_words() + p, c, hard, l01, l23, flag, 0, 1);
}

template <typename T, class OP>
__device__ __forceinline__ void leaf_op(Fr<T> &F, const OP &o) {
    const LParams &P = F.P;
    const int t = o.stage();
    int kind = o.kind();
    if (kind == K_R1 && t == 0) kind = K_REP;  // listdec.py:347
    const bool valid = F.slot() < o.pin();
    long long key[8];
    if (valid) leaf_phase_a(F, o, kind, key);
    __syncwarp();
    if ((o.flags() & LF_LAST) && o.src() == S_GL) F.discard_stage((o.flags() >> LF_FUSE_SHIFT) & 3 ? t + 1 : t);
    F.mark(0);
    const int sE = o.aux();
    if (kind == K_R0) {
        if (sE < LK_C(P, n) && valid) {
            uint32_t *dst = F.beta_row(sE, F.lane);
            write_chain(F, o, K_R0, dst, F.lane, 0, 0u, 0u, 0u, 0u);
            set8(F.ib, sE, F.lane);
        }
        F.dec = 0;
        return;
    }
    unsigned mask;
    const int C = o.ncand();
    if (!(o.flags() & LF_SELECT)) {
        mask = valid ? (1u << C) - 1u : 0u;
    } else if (C == 2) {
        mask = select_mask<2>(key, valid, LK_C(P, L), F.lane, F.slot(), F.seg());
    } else if (C == 4) {
        mask = select_mask<4>(key, valid, LK_C(P, L), F.lane, F.slot(), F.seg());
    } else {
        mask = select_mask<8>(key, valid, LK_C(P, L), F.lane, F.slot(), F.seg());
    }
    F.mark(1);
    // survivors in (source, cand) order: this lane's go to slots off ..
    uint8_t *asg = F.sm + LK_LAY(P).asg_off;
    double *met = reinterpret_cast<double *>(F.sm + LK_LAY(P).met_off);
    int k = F.base() + seg_excl_scan4(__popc(mask), F.lane, F.seg(), FULL_MASK);
#if PB_ASG_LOOP
    for (unsigned mk = mask; mk; mk &= mk - 1) {
        const int c = __ffs(mk) - 1;
        asg[k] = (uint8_t)((F.lane << 3) | c);
        met[k] = unkey(key[c]);
        ++k;
    }
#else
    // (static indices: a run-time key[c] would put the keys in local memory)
#pragma unroll
    for (int c = 0; c < 8; ++c)
        if (c < C && ((mask >> c) & 1u)) {
            const int kk = k + __popc(mask & ((1u << c) - 1u));  // no chain through k
            asg[kk] = (uint8_t)((F.lane << 3) | c);
            met[kk] = unkey(key[c]);
        }
#endif
    __syncwarp();
    const bool live = F.slot() < o.pout();
    int p = F.lane, c = 0;
    double pmn = F.pm;
    if (live) {
        const int v = asg[F.lane];
        p = v >> 3;
        c = v & 7;
        pmn = met[F.lane];
    }
    __syncwarp();
    // inherit the source's rows and leaf data (lazy copy, listdec.py:403-418)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        F.ia[j] = __shfl_sync(FULL_MASK, F.ia[j], p);
        F.ib[j] = __shfl_sync(FULL_MASK, F.ib[j], p);
    }
    const uint32_t hard = __shfl_sync(FULL_MASK, F.hard, p);
    const uint32_t l01 = __shfl_sync(FULL_MASK, F.lrb01, p);
    const uint32_t l23 = __shfl_sync(FULL_MASK, F.lrb23, p);
    const uint32_t flag = __shfl_sync(FULL_MASK, F.lflag, p);
    F.pm = pmn;
    F.hard = hard;
    F.lrb01 = l01;
    F.lrb23 = l23;
    F.lflag = flag;
    F.dec = (uint32_t)c;
    F.srcl = (uint32_t)p;
    F.mark(2);
    if (live && sE < LK_C(P, n)) {
        uint32_t *dst = F.beta_row(sE, F.lane);
        write_chain(F, o, kind, dst, p, c, hard, l01, l23, flag);
        set8(F.ib, sE, F.lane);
    }
}

// ------------------------------------------------------------ finalise

// Root codeword of survivor kk (listdec.py:275-287: the root row), built
// on demand from its final leaf decision and its beta rows; warp-parallel.
template <typename T>
__device__ __forceinline__ void build_root(const Fr<T> &F, int kk, uint32_t *x) {
    const LParams &P = F.P;
    const LOp fo = P.prog[LK_C(P, final_op)];
    const int n = LK_C(P, n), t = fo.stage, lane = F.lane;
    int kind = fo.kind;
    if (kind == K_R1 && t == 0) kind = K_REP;
    const int c = (int)__shfl_sync(FULL_MASK, F.dec, kk);
    const uint32_t hard = __shfl_sync(FULL_MASK, F.hard, kk);
    const uint32_t l01 = __shfl_sync(FULL_MASK, F.lrb01, kk);
    const uint32_t l23 = __shfl_sync(FULL_MASK, F.lrb23, kk);
    const uint32_t flag = __shfl_sync(FULL_MASK, F.lflag, kk);
    uint32_t ib[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ib[j] = __shfl_sync(FULL_MASK, F.ib[j], kk);
    // the final leaf's hard words (leaves wider than 32)
    const uint32_t *src = F.hard_words() + __shfl_sync(FULL_MASK, F.srcl, kk);
    // lanes over the root's words (the chain ends at the root: E = N)
    chain_row(F, kind, t, n, ib, x, src, c, hard, l01, l23, flag, lane, 32);
    __syncwarp();
}

__device__ __forceinline__ uint32_t syndrome(const LParams &P, const uint32_t *x, int lane) {
    const int N = LK_C(P, N), nw = N >= 32 ? N >> 5 : 1;
    uint32_t s = 0u;
    for (int w = lane; w < nw; w += 32) {
        uint32_t v = x[w];
        if (N < 32) v &= (1u << N) - 1u;
        const uint32_t *t = P.xsyn4 + (size_t)w * 128;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) s ^= __ldg(t + nb * 16 + ((v >> (4 * nb)) & 15u));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s ^= __shfl_xor_sync(FULL_MASK, s, d);
    return s;
}

// listdec.py:289-308: among CRC-passing survivors the strictly greater
// metric wins, earliest survivor on ties; with none passing, the best metric
// overall -- survivors visited by (metric desc, index asc), first pass wins.
// The whole warp works on the frame whose survivors are lanes b0 .. b0 + np - 1.
template <typename T>
__device__ __forceinline__ void finalize(Fr<T> &F, long long f, int np, int b0) {
    const LParams &P = F.P;
    const int lane = F.lane;
    const bool live = lane >= b0 && lane < b0 + np;
    const double pmk = live ? F.pm : -INFINITY;
    uint32_t *u = reinterpret_cast<uint32_t *>(F.sm + LK_LAY(P).root_off);
    const int rw = LK_C(P, N) >= 32 ? LK_C(P, N) >> 5 : 1;
    if (P.path_cw) {  // decode_paths: every survivor's codeword, metric and CRC flag
        for (int kk = 0; kk < np; ++kk) {
            uint32_t *dst = P.path_cw + ((size_t)f * LK_C(P, L) + kk) * rw;
            if (LK_C(P, N) < 32 && lane == 0) dst[0] = 0u;
            __syncwarp();
            build_root(F, b0 + kk, dst);
            const uint32_t syn = syndrome(P, dst, lane);
            if (lane == 0) P.path_crc[(size_t)f * LK_C(P, L) + kk] = LK_C(P, has_crc) && syn == LK_C(P, crc_const);
        }
        if (live) P.path_pm[(size_t)f * LK_C(P, L) + lane - b0] = pmk;
        __syncwarp();
    }
    unsigned tried = 0u;
    int first = -1, wnr = -1;
    double wpm = -INFINITY;
    for (int it = 0; it < np; ++it) {
        double bm = (live && !((tried >> lane) & 1u)) ? pmk : -INFINITY;
        int bk = (live && !((tried >> lane) & 1u)) ? lane : 64;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double om = __shfl_xor_sync(FULL_MASK, bm, d);
            const int ok2 = __shfl_xor_sync(FULL_MASK, bk, d);
            if (om > bm || (om == bm && ok2 < bk)) {
                bm = om;
                bk = ok2;
            }
        }
        if (first < 0) first = bk;
        tried |= 1u << bk;
        if (!LK_C(P, has_crc)) {
            wnr = bk;
            wpm = bm;
            break;
        }
        if (LK_C(P, N) < 32 && lane == 0) u[0] = 0u;
        __syncwarp();
        build_root(F, bk, u);
        if (syndrome(P, u, lane) == LK_C(P, crc_const)) {
            wnr = bk;
            wpm = bm;
            break;
        }
    }
    const bool wok = wnr >= 0 && LK_C(P, has_crc);
    if (wnr < 0) {
        wnr = first;
        wpm = __shfl_sync(FULL_MASK, pmk, first & 31);
    }
    if (P.info_out) {
        if (!wok) {
            if (LK_C(P, N) < 32 && lane == 0) u[0] = 0u;
            __syncwarp();
            build_root(F, wnr, u);
        }
        polar_transform_words(u, LK_C(P, N), lane);
        uint8_t *out = P.info_out + (size_t)f * LK_C(P, k);
        for (int i = lane; i < LK_C(P, k); i += 32) {
            const uint32_t pos = __ldg(P.info_pos + i);
            out[i] = (uint8_t)((u[pos >> 5] >> (pos & 31)) & 1u);
        }
    }
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[f] = wok;
        if (P.pm_out) P.pm_out[f] = wpm;
        if (P.paths_used) P.paths_used[f] = np;
    }
    __syncwarp();
}

// ------------------------------------------------------------- kernel

template <typename T>
__device__ __forceinline__ void load_channel_lane(const LParams &P, T *ch, long long f, int lane) {
    // ch: the frame's channel, quad x at ch + x * CQ (element i at che(ch, i))
    const int N = LK_C(P, N);
    if (P.in_type == PB_IN_I8) {
        const int8_t *src = reinterpret_cast<const int8_t *>(P.llr) + (size_t)f * N;
        for (int i = lane; i < N; i += 32) ch[(i >> 2) * CQ + (i & 3)] = (T)src[i];
        return;
    }
    const float *src = reinterpret_cast<const float *>(P.llr) + (size_t)f * N;
    if ((N & 3) == 0) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        for (int i = lane; i < (N >> 2); i += 32) {
            const float4 v = __ldcs(s4 + i);  // read once: evict-first
            float q[4] = {ingest<T>(v.x), ingest<T>(v.y), ingest<T>(v.z), ingest<T>(v.w)};
            V4<T>::st(ch + CQ * i, q);
        }
    } else {
        for (int i = lane; i < N; i += 32) Elem<T>::st(ch + (i >> 2) * CQ + (i & 3), ingest<T>(src[i]));
    }
}

// One op.  Compile-time kind (the specialised build): exactly the body the
// op needs is instantiated; run-time kind: a jump over the (F / G, source,
// destination) placements that occur and the leaf body.
template <typename T, int K, int S, int PI, int PO, int NC, int SR, int AX, int FL>
__device__ __forceinline__ void exec_op(Fr<T> &F, const Op<K, S, PI, PO, NC, SR, AX, FL> &o, int &np) {
    if constexpr (K >= 0) {
        if constexpr (K <= K_G) {
            static_assert(SR >= 0 && AX >= 0, "a compile-time F / G needs compile-time placements");
            fg_op<T, K == K_G, SR, AX == S_GL ? S_GL : S_SM>(F, o);
        } else if constexpr (K != K_NOP) {
            leaf_op(F, o);
            np = o.pout();
        }
    } else {
        const int sel = o.kind() <= K_G ? (o.kind() * 16 + o.src() * 2 + (o.aux() == S_GL ? 1 : 0)) : -1;
        switch (sel) {
            // F: (source, destination) placements that occur (channel and
            // stage n-1 sources only write stages read by a leaf)
            case 0 * 16 + S_CH * 2 + 1: fg_op<T, false, S_CH, S_GL>(F, o); break;
            case 1 * 16 + S_CH * 2 + 1: fg_op<T, true, S_CH, S_GL>(F, o); break;
            case 0 * 16 + S_SM * 2 + 0: fg_op<T, false, S_SM, S_SM>(F, o); break;
            case 0 * 16 + S_GL * 2 + 0: fg_op<T, false, S_GL, S_SM>(F, o); break;
            case 0 * 16 + S_GL * 2 + 1: fg_op<T, false, S_GL, S_GL>(F, o); break;
            case 0 * 16 + S_V1 * 2 + 0: fg_op<T, false, S_V1, S_SM>(F, o); break;
            case 0 * 16 + S_V1 * 2 + 1: fg_op<T, false, S_V1, S_GL>(F, o); break;
            case 0 * 16 + S_V2 * 2 + 0: fg_op<T, false, S_V2, S_SM>(F, o); break;
            case 0 * 16 + S_V2 * 2 + 1: fg_op<T, false, S_V2, S_GL>(F, o); break;
            case 1 * 16 + S_SM * 2 + 0: fg_op<T, true, S_SM, S_SM>(F, o); break;
            case 1 * 16 + S_GL * 2 + 0: fg_op<T, true, S_GL, S_SM>(F, o); break;
            case 1 * 16 + S_GL * 2 + 1: fg_op<T, true, S_GL, S_GL>(F, o); break;
            case 1 * 16 + S_V1 * 2 + 0: fg_op<T, true, S_V1, S_SM>(F, o); break;
            case 1 * 16 + S_V1 * 2 + 1: fg_op<T, true, S_V1, S_GL>(F, o); break;
            case 1 * 16 + S_V2 * 2 + 0: fg_op<T, true, S_V2, S_SM>(F, o); break;
            case 1 * 16 + S_V2 * 2 + 1: fg_op<T, true, S_V2, S_GL>(F, o); break;
            default:
                if (o.kind() != K_NOP) {
                    leaf_op(F, o);
                    np = o.pout();
                }
                break;
        }
    }
}

template <typename T>
__device__ __forceinline__ void run_ops(Fr<T> &F, int &np) {
    const LParams &P = F.P;
#if PB_PROFILE
    const bool prof = P.op_cycles && blockIdx.x == 0 && threadIdx.x == 0;
#endif
    for (int oi = 0; oi < LK_C(P, n_ops); ++oi) {
#if PB_PROFILE
        if (prof) P.op_cycles[oi] = clock64();
        F.marks = prof ? P.op_cycles + LK_C(P, n_ops) + 1 + 4 * oi : nullptr;
#endif
        LOp o;
        {
            const uint2 raw = reinterpret_cast<const uint2 *>(P.prog)[oi];  // one 8-byte constant load
            o = *reinterpret_cast<const LOp *>(&raw);
        }
#ifdef PB_JIT
        // the op's variant: its body with the schedule's constants folded in
        switch (P.vid[oi]) {
#define PB_JIT_CASE(id, K, S, PI, PO, NC, SR, AX, FL) \
    case id: exec_op<T>(F, Op<K, S, PI, PO, NC, SR, AX, FL>{o}, np); break;
            PB_JIT_OPS(PB_JIT_CASE)
#undef PB_JIT_CASE
            default: break;
        }
#else
        exec_op<T>(F, Op<>{o}, np);
#endif
        // (measured and dropped: the CTA's two halves regrouping separately, 5.18 against 5.17 Gbit/s)
        if (P.sync_mask >= 0 && (oi & P.sync_mask) == 0)
            __syncthreads();  // regroup the CTA's frames (shared instruction fetch)
        else
            __syncwarp();
    }
#if PB_PROFILE
    if (prof) P.op_cycles[LK_C(P, n_ops)] = clock64();
#endif
}

// Persistent frame loop: a CTA holds P.fpc frames (one warp each).
template <typename T>
__device__ __forceinline__ void lane_body(const LParams &P) {
    extern __shared__ __align__(16) unsigned char lk_smem[];
    constexpr int G = LK_G, LP = 32 / LK_G;  // frames per warp, path slots per frame
    const int grp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long slot = (long long)blockIdx.x * P.fpc + grp;
    unsigned char *gs = P.gscratch ? P.gscratch + (size_t)slot * LK_LAY(P).gbytes : nullptr;
    unsigned char *sm = lk_smem + (size_t)grp * LK_LAY(P).smem_bytes;
    const long long per_cta = (long long)P.fpc * G, stride = (long long)gridDim.x * per_cta;
    const long long batch = P.batch_dev ? (long long)*P.batch_dev : P.batch;
    // (measured and dropped: a second frame group per CTA started half a
    // program late, and CTAs started at staggered ops: +2 % / -2 % device
    // rate, both costing a throwaway half frame per launch)
    for (long long f0 = (long long)blockIdx.x * per_cta; f0 < batch; f0 += stride) {
        Fr<T> F(P, sm, gs);
        // tail: idle frame slots decode the last frame again and write nothing
        auto frame_of = [&](int g) {
            const long long fi = f0 + grp * G + g < batch ? f0 + grp * G + g : batch - 1;
            return P.frame_map ? (long long)P.frame_map[fi] : fi;
        };
#pragma unroll 1
        for (int g = 0; g < G; ++g)
            load_channel_lane<T>(P, reinterpret_cast<T *>((LK_LAY(P).ch_gl ? gs : sm) + LK_LAY(P).ch_off) + 4 * g,
                                 frame_of(g), lane);
        __syncwarp();
        int np = 1;
        run_ops(F, np);
#pragma unroll 1
        for (int g = 0; g < G; ++g)
            if (f0 + grp * G + g < batch) finalize(F, frame_of(g), np, g * LP);
        if (P.fpc > 1) __syncthreads();
    }
}

#ifndef PB_JIT
template <typename T>
__global__ void __launch_bounds__(512, 1) k_lane(const __grid_constant__ LParams P) {
    lane_body<T>(P);
}
#endif

#if !defined(__CUDACC_RTC__) && !defined(PB_JIT)
template <typename T>
cudaError_t lane_launch_t(const LParams *p, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_lane<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // a batch smaller than one CTA's frame slots runs only the warps it needs
    // (single-frame latency: the frame's warp does not share the SM)
    const int warps = grid == 1 && p->batch < p->fpc && !p->batch_dev ? (int)p->batch : p->fpc;
    k_lane<T><<<grid, 32 * warps, smem, st>>>(*p);
    return cudaGetLastError();
}
template <typename T>
cudaError_t lane_occ_t(size_t smem, int fpc, int *bps) {
    cudaError_t e = cudaFuncSetAttribute(k_lane<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k_lane<T>, 32 * fpc, smem);
}
#endif

}  // namespace lk
}  // namespace pb

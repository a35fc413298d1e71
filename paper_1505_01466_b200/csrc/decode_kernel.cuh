// decode_kernel.cuh -- Fast-SSC list-CRC decode kernel for sm_100a.
// Instantiated per (mode, W, PPW) by decode_inst.cu; dispatched in dispatch.cu.
//
// One CTA of W warps decodes one frame at a time (persistent loop over
// frames).  The L path slots are split across the warps, PPW per warp
// (compile-time, a power of two); a warp only synchronises with the others at
// leaves.  Per op:
//   F / G      element-parallel over the warp's (path, element) pairs: its A
//              active paths split 32 lanes into groups of G = 32/pow2(A)
//              (kernels.py:39-56, listdec.py:319-326).  In the steady state
//              (A = PPW) G is a compile-time constant and the loops address
//              shared memory with immediate offsets.
//   leaves     per-path scans of the node LLRs: numpy-pairwise-exact float sums
//              (Rate-0 / Rep, listdec.py:340-359), stable two / four least
//              reliable positions + hard decisions + parity (Rate-1 / SPC,
//              listdec.py:360-394)
//   selection  warp 0, lane = source path: candidate metrics as orderable
//              int64 keys, each lane's candidates a sorted column; the L-th
//              best key from a k-way merge of the columns (REDUX max / min,
//              select_phase_c), exact ties resolved by (source, cand) prefix
//              counts -- listdec.py:63-100
//   materialise survivors copy their source's row-index vectors (lazy copy,
//              listdec.py:103-143,397-434), write the leaf word and run the
//              leaf's chain of Combines in place (listdec.py:327-332)
//   finalise   CRC by per-path GF(2) syndrome == constant, strict-max pick
//              among CRC-passing paths (listdec.py:289-308), polar transform
//              of the winner and payload gather (encode.py:29-53,76-87)
#pragma once
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#else
#define INT_MAX 2147483647
#define INT_MIN (-2147483647 - 1)
#define LLONG_MIN (-9223372036854775807LL - 1)
#define LLONG_MAX 9223372036854775807LL
#define INFINITY __int_as_float(0x7f800000)
#endif

#include "decoder.cuh"

// Profiling build (-DPB_PROFILE=1, tools/op_cycles.py, PB_ABLATE): per-op
// clock64 phase marks and ablation switches; compiled out otherwise.
#ifndef PB_PROFILE
#define PB_PROFILE 0
#endif
#define PB_ABL(P, bit) (PB_PROFILE && ((P).ablate & (bit)))

#define PB_IN_F32 0
#define PB_IN_I8 1

// one frame per CTA: the frame's shared block is the whole dynamic smem
extern __shared__ __align__(16) unsigned char g_smem[];

namespace pb {

#define FULL_MASK 0xffffffffu

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static constexpr bool kInt = false;
    static __device__ __forceinline__ float ld(const float *p) { return *p; }
    static __device__ __forceinline__ float ldcs(const float *p) { return __ldcs(p); }
    static __device__ __forceinline__ void st(float *p, float v) { *p = v; }
};
template <>
struct Elem<int8_t> {
    static constexpr bool kInt = true;
    static __device__ __forceinline__ float ld(const int8_t *p) { return (float)*p; }
    static __device__ __forceinline__ float ldcs(const int8_t *p) {
        return (float)__ldcs(reinterpret_cast<const signed char *>(p));
    }
    static __device__ __forceinline__ void st(int8_t *p, float v) { *p = (int8_t)__float2int_rn(v); }
};

// min-sum F: sign(a) sign(b) min(|a|,|b|); a zero product comes out as a
// signed zero, numerically equal to the reference's 0 (kernels.py:39-48)
// (one instruction: FMNMX.XORSIGN |a|, |b|)
__device__ __forceinline__ float f_op(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// G: b + (1 - 2 beta) a -- one correctly rounded add (kernels.py:51-56);
// int8 mode saturates to [-127, 127]
template <typename T>
__device__ __forceinline__ float g_op(float a, float b, unsigned bit) {
    float v = __fadd_rn(b, __uint_as_float(__float_as_uint(a) ^ (bit << 31)));
    if (Elem<T>::kInt) v = fminf(fmaxf(v, -127.f), 127.f);
    return v;
}

template <typename T>
__device__ __forceinline__ float g_op_bits(float a, float b, unsigned bits, int j) {
    float v = __fadd_rn(b, __uint_as_float(__float_as_uint(a) ^ ((bits << (31 - j)) & 0x80000000u)));
    if (Elem<T>::kInt) v = fminf(fmaxf(v, -127.f), 127.f);
    return v;
}

__device__ __forceinline__ int log2ceil(int x) { return x <= 1 ? 0 : 32 - __clz(x - 1); }

// four consecutive elements (one 128-bit / 32-bit access)
template <typename T>
struct V4;
template <>
struct V4<float> {
    static __device__ __forceinline__ void ld(const float *p, float (&v)[4]) {
        const float4 x = *reinterpret_cast<const float4 *>(p);
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
    }
    static __device__ __forceinline__ void ldcs(const float *p, float (&v)[4]) {
        const float4 x = __ldcs(reinterpret_cast<const float4 *>(p));
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
    }
    static __device__ __forceinline__ void st(float *p, const float (&v)[4]) {
        *reinterpret_cast<float4 *>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct V4<int8_t> {
    static __device__ __forceinline__ void ld(const int8_t *p, float (&v)[4]) {
        const int x = *reinterpret_cast<const int *>(p);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (float)((x << (24 - 8 * j)) >> 24);
    }
    static __device__ __forceinline__ void ldcs(const int8_t *p, float (&v)[4]) {
        const int x = __ldcs(reinterpret_cast<const int *>(p));
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = (float)((x << (24 - 8 * j)) >> 24);
    }
    static __device__ __forceinline__ void st(int8_t *p, const float (&v)[4]) {
        unsigned x = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) x |= ((unsigned)__float2int_rn(v[j]) & 0xffu) << (8 * j);
        *reinterpret_cast<unsigned *>(p) = x;
    }
};

// ------------------------------------------------------------- sources
// Stored alpha rows (FrameLayout).  PPW >= 16 (one or two lanes per path in
// the steady state): quad-interleaved -- a block of PPW rows stores quad x
// (elements 4x .. 4x+3) of local row rl at quad index
// x * PPW + ((rl + c(x)) mod PPW), c(x) = (x mod GS) * 8 / GS (GS = 32 / PPW
// steady-state lanes per path: 0 for PPW = 32, 4 (x odd) for PPW = 16), so the
// steady-state lanes read their quads with 128-bit accesses from 512
// contiguous bytes, bank-conflict free, at addresses affine in x (immediate
// offsets in the unrolled loops).  PPW <= 8 (four or more lanes per path):
// element-interleaved, element i of local row rl at i * PPW + rl, the lanes
// of a path taking consecutive elements (conflict free).
template <int PPW>
struct Lay {
    static constexpr bool kQuad = PPW >= 16;
    static constexpr int GS = 32 / PPW;
    static __device__ __forceinline__ int q(int x, int rl) {
        const int c = (x & (GS - 1)) * (8 / GS);
        return (x * PPW + ((rl + c) & (PPW - 1))) * 4;
    }
    static __device__ __forceinline__ int e(int i, int rl) { return kQuad ? q(i >> 2, rl) + (i & 3) : i * PPW + rl; }
};
// LAST: the row's last read (a G or a leaf; F reads first) from global
// scratch -- evict-first loads, so the L2 keeps the rows still to be read
template <typename T, int PPW, bool LAST = false>
struct RowSrc {
    static constexpr bool kQuad = Lay<PPW>::kQuad;
    const T *blk;
    int rl;
    __device__ __forceinline__ float get(int i) const {
        return LAST ? Elem<T>::ldcs(blk + Lay<PPW>::e(i, rl)) : Elem<T>::ld(blk + Lay<PPW>::e(i, rl));
    }
    __device__ __forceinline__ void get4(int x, float (&v)[4]) const {
        if (kQuad) {
            if (LAST)
                V4<T>::ldcs(blk + Lay<PPW>::q(x, rl), v);
            else
                V4<T>::ld(blk + Lay<PPW>::q(x, rl), v);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[j] = get(4 * x + j);
        }
    }
    __device__ __forceinline__ unsigned bits_word(int) const { return 0u; }
    __device__ __forceinline__ void get4w(int x, float (&v)[4], unsigned) const { get4(x, v); }
};
template <typename T, int PPW>
struct RowDst {
    T *blk;
    int rl;
    __device__ __forceinline__ void put(int i, float v) const { Elem<T>::st(blk + Lay<PPW>::e(i, rl), v); }
    __device__ __forceinline__ void put4(int x, const float (&v)[4]) const {
        if (Lay<PPW>::kQuad) {
            V4<T>::st(blk + Lay<PPW>::q(x, rl), v);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) put(4 * x + j, v[j]);
        }
    }
};
// stage n-1 in the left half of the tree: f(channel halves)
template <typename T>
struct VirtF {
    static constexpr bool kQuad = true;
    const T *ch;
    int half;
    __device__ __forceinline__ float get(int i) const {
        return f_op(Elem<T>::ld(ch + i), Elem<T>::ld(ch + i + half));
    }
    __device__ __forceinline__ void get4(int x, float (&v)[4]) const {
        float a[4], b[4];
        V4<T>::ld(ch + 4 * x, a);
        V4<T>::ld(ch + 4 * x + half, b);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = f_op(a[j], b[j]);
    }
    __device__ __forceinline__ unsigned bits_word(int) const { return 0u; }
    __device__ __forceinline__ void get4w(int x, float (&v)[4], unsigned) const { get4(x, v); }
};
// stage n-1 in the right half: g(channel halves, the path's left-half bits)
template <typename T>
struct VirtG {
    static constexpr bool kQuad = true;
    const T *ch;
    const uint32_t *bw;
    int half;
    __device__ __forceinline__ float get(int i) const {
        return g_op<T>(Elem<T>::ld(ch + i), Elem<T>::ld(ch + i + half), (bw[i >> 5] >> (i & 31)) & 1u);
    }
    __device__ __forceinline__ void get4(int x, float (&v)[4]) const {
        float a[4], b[4];
        V4<T>::ld(ch + 4 * x, a);
        V4<T>::ld(ch + 4 * x + half, b);
        const unsigned bits = bw[x >> 3] >> ((x & 7) * 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(a[j], b[j], bits, j);
    }
    // the beta word of quad x, and get4 with it preloaded (x in that word)
    __device__ __forceinline__ unsigned bits_word(int x) const { return bw[x >> 3]; }
    __device__ __forceinline__ void get4w(int x, float (&v)[4], unsigned wd) const {
        float a[4], b[4];
        V4<T>::ld(ch + 4 * x, a);
        V4<T>::ld(ch + 4 * x + half, b);
        const unsigned bits = wd >> ((x & 7) * 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = g_op_bits<T>(a[j], b[j], bits, j);
    }
};
// Leaf fusion (DOp::fuse) is compiled for the int8 shapes only: measured
// +3.5 % on c4 int8 L=32, while in the float32 shapes the extra leaf
// instantiations cost registers / spills and lost 2.5-5 % (c3 L=32).
template <typename T>
constexpr bool kFuseLeaf = Elem<T>::kInt;

// f / g of a stored parent row's halves (a leaf fused with the F / G that
// would have stored its LLRs, DOp::fuse); g with the path's left-sibling bits
template <typename T, bool IS_G, class S>
struct FusedSrc {
    static constexpr bool kQuad = true;
    S in;
    const uint32_t *bw;
    int half;  // the leaf's size
    __device__ __forceinline__ float get(int i) const {
        const float a = in.get(i), b = in.get(i + half);
        return IS_G ? g_op<T>(a, b, (bw[i >> 5] >> (i & 31)) & 1u) : f_op(a, b);
    }
    __device__ __forceinline__ void get4(int x, float (&v)[4]) const {
        float a[4], b[4];
        in.get4(x, a);
        in.get4(x + (half >> 2), b);
        const unsigned bits = IS_G ? bw[x >> 3] >> ((x & 7) * 4) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = IS_G ? g_op_bits<T>(a[j], b[j], bits, j) : f_op(a[j], b[j]);
    }
    __device__ __forceinline__ unsigned bits_word(int) const { return 0u; }
    __device__ __forceinline__ void get4w(int x, float (&v)[4], unsigned) const { get4(x, v); }
};
// the channel itself (a root leaf)
template <typename T>
struct ChanSrc {
    static constexpr bool kQuad = true;
    const T *ch;
    __device__ __forceinline__ float get(int i) const { return Elem<T>::ld(ch + i); }
    __device__ __forceinline__ void get4(int x, float (&v)[4]) const { V4<T>::ld(ch + 4 * x, v); }
    __device__ __forceinline__ unsigned bits_word(int) const { return 0u; }
    __device__ __forceinline__ void get4w(int x, float (&v)[4], unsigned) const { get4(x, v); }
};

// ------------------------------------------------------- configuration
// Code / layout constants, read from the launch parameters; where the
// channel lives (shared memory or global scratch) is compile-time.
template <bool CHG>
struct RtCfg {
    static constexpr bool kChGlobal = CHG;  // channel in global scratch
    const Params *p;
    __device__ __forceinline__ int N() const { return p->N; }
    __device__ __forceinline__ int n() const { return p->n; }
    __device__ __forceinline__ int L() const { return p->L; }
    __device__ __forceinline__ int k() const { return p->k; }
    __device__ __forceinline__ int has_crc() const { return p->has_crc; }
    __device__ __forceinline__ uint32_t crc_const() const { return p->crc_const; }
    __device__ __forceinline__ int ch_off() const { return p->lay.ch_off; }
    __device__ __forceinline__ int a_off(int s) const { return p->lay.a_off[s]; }
    __device__ __forceinline__ int a_gfrom() const { return p->lay.a_gfrom; }
    __device__ __forceinline__ int b_off(int s) const { return p->lay.b_off[s]; }
    __device__ __forceinline__ int b_gfrom() const { return p->lay.b_gfrom; }
    __device__ __forceinline__ int b_stride(int s) const { return p->lay.b_stride[s]; }
    __device__ __forceinline__ int pm_off() const { return p->lay.pm_off; }
    __device__ __forceinline__ int ia_off() const { return p->lay.ia_off; }
    __device__ __forceinline__ int ib_off() const { return p->lay.ib_off; }
    __device__ __forceinline__ int idx_stride() const { return p->lay.idx_stride; }
    __device__ __forceinline__ int cd_off() const { return p->lay.cd_off; }
    __device__ __forceinline__ int clrb_off() const { return p->lay.clrb_off; }
    __device__ __forceinline__ int cflag_off() const { return p->lay.cflag_off; }
    __device__ __forceinline__ int asg_off() const { return p->lay.asg_off; }
    __device__ __forceinline__ int hard_off() const { return p->lay.hard_off; }
    __device__ __forceinline__ int hard_words() const { return p->lay.hard_words; }
    __device__ __forceinline__ int root_off() const { return p->lay.root_off; }
    __device__ __forceinline__ int root_words() const { return p->lay.root_words; }
    __device__ __forceinline__ int gbytes() const { return p->lay.gbytes; }
    __device__ __forceinline__ int smem_bytes() const { return p->lay.smem_bytes; }
};

// ------------------------------------------------------- frame state

template <typename T, int W, int PPW, class CFG>
struct Dec {
    static constexpr int LP = ilog2(PPW);
    static constexpr int GSS = 32 / PPW;           // steady-state lanes per path
    static constexpr int NBUF = W > 1 ? 2 : 1;     // candidate buffers
    static constexpr int RW = PPW * W;              // path rows (>= L): the per-path arrays' stride
    static constexpr int IW = (kMaxLog + 3) / 4;    // index words per path (4 stages each)
    const Params &P;
    CFG cfg;
    unsigned char *sm;  // this frame's shared-memory block
    unsigned char *gs;  // this frame's global scratch block
    int lane, warp;
    int cur;            // live half of the double-buffered path state
    int par;            // candidate-buffer parity (toggles at forking leaves)
    int lpar;           // parity used by the last forking leaf
    long long *ph;      // debug: phase timestamps of the current op (or null)
    const DOp *prog;    // the op program (shared-memory copy when staged)

    __device__ Dec(const Params &p, CFG c, unsigned char *s, unsigned char *g)
        : P(p), cfg(c), sm(s), gs(g), lane(threadIdx.x & 31), warp((threadIdx.x >> 5) & (W - 1)), cur(0), par(0),
          lpar(0), ph(nullptr), prog(p.prog) {}
    __device__ __forceinline__ void mark(int i) const {
        if (PB_PROFILE && ph && lane == 0) ph[i] = clock64();
    }

    // row r of stage s: its PPW-row block (quad-interleaved, FrameLayout)
    // and its local row index
    __device__ __forceinline__ int blkoff(int s, int r) const { return (r >> LP) * (PPW << (s < 2 ? 2 : s)); }
    __device__ __forceinline__ T *a_sm(int s) const { return reinterpret_cast<T *>(sm + cfg.a_off(s)); }
    __device__ __forceinline__ T *a_gl(int s) const { return reinterpret_cast<T *>(gs + cfg.a_off(s)); }
    __device__ __forceinline__ uint32_t *beta_row(int s, int row) const {
        return reinterpret_cast<uint32_t *>((s >= cfg.b_gfrom() ? gs : sm) + cfg.b_off(s)) + row * cfg.b_stride(s);
    }
    __device__ __forceinline__ T *channel() const {
        return reinterpret_cast<T *>((CFG::kChGlobal ? gs : sm) + cfg.ch_off());
    }
    __device__ __forceinline__ double *pm(int b) const {
        return reinterpret_cast<double *>(sm + cfg.pm_off()) + b * RW;
    }
    // alpha / beta row index of path q at stage / slot s, four stages per
    // word: byte (s & 3) of word [buf][s >> 2][path]
    __device__ __forceinline__ uint8_t &ia(int b, int s, int q) const {
        return sm[cfg.ia_off() + ((b * IW + (s >> 2)) * RW + q) * 4 + (s & 3)];
    }
    __device__ __forceinline__ uint8_t &ib(int b, int s, int q) const {
        return sm[cfg.ib_off() + ((b * IW + (s >> 2)) * RW + q) * 4 + (s & 3)];
    }
    __device__ __forceinline__ uint32_t &iaw(int b, int x, int q) const {
        return reinterpret_cast<uint32_t *>(sm + cfg.ia_off())[(b * IW + x) * RW + q];
    }
    __device__ __forceinline__ uint32_t &ibw(int b, int x, int q) const {
        return reinterpret_cast<uint32_t *>(sm + cfg.ib_off())[(b * IW + x) * RW + q];
    }
    __device__ __forceinline__ int bsel(int b) const { return NBUF > 1 ? b : 0; }
    // candidate data: [buf][entry][source path]
    __device__ __forceinline__ double &cd(int b, int c, int q) const {
        return reinterpret_cast<double *>(sm + cfg.cd_off())[(bsel(b) * kMaxCand + c) * RW + q];
    }
    __device__ __forceinline__ uint16_t &clrb(int b, int j, int q) const {
        return reinterpret_cast<uint16_t *>(sm + cfg.clrb_off())[(bsel(b) * 4 + j) * RW + q];
    }
    __device__ __forceinline__ uint8_t *cflag(int b) const { return sm + cfg.cflag_off() + bsel(b) * RW; }
    __device__ __forceinline__ uint8_t *asg(int b) const { return sm + cfg.asg_off() + bsel(b) * 2 * RW; }
    __device__ __forceinline__ uint32_t &hard(int b, int w, int q) const {
        return reinterpret_cast<uint32_t *>(sm + cfg.hard_off())[(bsel(b) * cfg.hard_words() + w) * RW + q];
    }
    __device__ __forceinline__ uint32_t *root() const { return reinterpret_cast<uint32_t *>(sm + cfg.root_off()); }

    // the frame's W warps (named barrier per frame slot; the CTA may hold several frames)
    __device__ __forceinline__ void sync() const {
        if (W > 1)
            asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / (32 * W))), "r"(32 * W) : "memory");
        else
            __syncwarp();
    }

    // lane -> (path, sub-lane) for this warp when np paths are active
    struct Map {
        int q, sub, G, lg;
        bool active;
    };
    __device__ __forceinline__ Map map(int np) const {
        Map m;
        int act = np - warp * PPW;
        act = act < 0 ? 0 : (act > PPW ? PPW : act);
        m.lg = 5 - log2ceil(act > 0 ? act : 1);
        m.G = 1 << m.lg;
        const int ql = lane >> m.lg;
        m.sub = lane & (m.G - 1);
        m.active = ql < act;
        m.q = warp * PPW + ql;
        return m;
    }
    // the same with log2 lanes per path precomputed on the host (DOp::lgi /
    // lgo; one warp per frame, where every path is this warp's)
    __device__ __forceinline__ Map map(int np, int lgp) const {
        if (W > 1) return map(np);
        Map m;
        m.lg = lgp;
        m.G = 1 << lgp;
        const int ql = lane >> lgp;
        m.sub = lane & (m.G - 1);
        m.active = ql < np;
        m.q = ql;
        return m;
    }
};

// ---------------------------------------------------------------- F / G

// One path's F / G: h outputs, G lanes per path (GC > 0: known at compile
// time, the steady state), this lane = sub.  h >= 4: the lane's quads
// x = sub, sub + G, ... in unrolled blocks of UQ whose loads all issue before
// the stores (UQ = 8 for L2-latency global sources); h < 4: scalar.
template <typename T, bool IS_G, int GC, int UQ, class S, class D>
__device__ __forceinline__ void fg_row(const S &src, const D &dst, const uint32_t *bw, int h, int Grt, int sub) {
    const int G = GC > 0 ? GC : Grt;
    if (h < 4) {
        for (int i = sub; i < h; i += G)
            dst.put(i, IS_G ? g_op<T>(src.get(i), src.get(i + h), (bw[0] >> i) & 1u) : f_op(src.get(i), src.get(i + h)));
        return;
    }
    const int nq = h >> 2;
    int x0 = sub;
    // G lanes x UQ quads of a block within one 32-element beta word (the
    // steady state): that word is loaded once per block
    constexpr bool ONE_WORD = GC > 0 && GC * UQ <= 8;
    for (; x0 + (UQ - 1) * G < nq; x0 += G * UQ) {  // whole blocks: no guards
        float a[UQ][4], b[UQ][4];
        unsigned bits[UQ];
        const unsigned wd = IS_G && ONE_WORD ? bw[x0 >> 3] : 0u;
        const unsigned swa = ONE_WORD ? src.bits_word(x0) : 0u, swb = ONE_WORD ? src.bits_word(x0 + nq) : 0u;
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
            const int x = x0 + u * G;
            if (ONE_WORD) {
                src.get4w(x, a[u], swa);
                src.get4w(x + nq, b[u], swb);
            } else {
                src.get4(x, a[u]);
                src.get4(x + nq, b[u]);
            }
            bits[u] = IS_G ? (ONE_WORD ? wd : bw[x >> 3]) >> ((x & 7) * 4) : 0u;
        }
#pragma unroll
        for (int u = 0; u < UQ; ++u) {
            float o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) o[j] = IS_G ? g_op_bits<T>(a[u][j], b[u][j], bits[u], j) : f_op(a[u][j], b[u][j]);
            dst.put4(x0 + u * G, o);
        }
    }
    for (; x0 < nq; x0 += G) {  // the rest, one quad at a time
        float a[4], b[4], o[4];
        src.get4(x0, a);
        src.get4(x0 + nq, b);
        const unsigned bits = IS_G ? bw[x0 >> 3] >> ((x0 & 7) * 4) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = IS_G ? g_op_bits<T>(a[j], b[j], bits, j) : f_op(a[j], b[j]);
        dst.put4(x0, o);
    }
}

// evict-first loads for the last read of a global-scratch row (RowSrc LAST)
#ifndef PB_LAST_CS
#define PB_LAST_CS 1
#endif

// quads in flight per lane (global-scratch / shared-memory sources)
#ifndef PB_UQ_GL
#define PB_UQ_GL 8
#endif
#ifndef PB_UQ_SM
#define PB_UQ_SM 4
#endif

// Element-interleaved layout (PPW <= 8): the G lanes of a path take
// consecutive elements.  fg_loop: any G (GC > 0: compile-time); fg_chunks:
// steady state with h >= 32, 32-element chunks whose loads all issue before
// the stores (immediate offsets, beta word loaded once).
template <typename T, bool IS_G, int GC, class S, class D>
__device__ __forceinline__ void fg_loop(const S &src, const D &dst, const uint32_t *bw, int h, int Grt, int sub) {
    const int G = GC > 0 ? GC : Grt;
    if (!IS_G) {
#pragma unroll 4
        for (int i = sub; i < h; i += G) dst.put(i, f_op(src.get(i), src.get(i + h)));
    } else {
        const int lim = h < 32 ? h : 32;
        for (int c0 = 0; c0 < h; c0 += 32) {
            const uint32_t word = bw[c0 >> 5];
#pragma unroll 4
            for (int j = sub; j < lim; j += G)
                dst.put(c0 + j, g_op<T>(src.get(c0 + j), src.get(c0 + j + h), (word >> j) & 1u));
        }
    }
}
template <typename T, bool IS_G, int GC, int PPW, int UMAX, class S>
__device__ __forceinline__ void fg_chunks(const S &src, T *dst, const uint32_t *bw, int h, int sub) {
    constexpr int PER = 32 / GC;                // this lane's elements per chunk
    constexpr int U = PER < UMAX ? PER : UMAX;  // unrolled block (loads in flight)
    for (int c0 = 0; c0 < h; c0 += 32) {
        const uint32_t wsh = IS_G ? (bw[c0 >> 5] >> sub) : 0u;
        T *d = dst + (c0 + sub) * PPW;
#pragma unroll
        for (int blk = 0; blk < PER; blk += U) {
            float a[U], b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = c0 + sub + (blk + u) * GC;
                a[u] = src.get(i);
                b[u] = src.get(i + h);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float v = IS_G ? g_op<T>(a[u], b[u], (wsh >> ((blk + u) * GC)) & 1u) : f_op(a[u], b[u]);
                Elem<T>::st(d + (blk + u) * GC * PPW, v);
            }
        }
    }
}

// SRC_GL: the source rows are in global scratch (L2 latency: more loads in flight)
template <typename T, int W, int PPW, class CFG, bool IS_G, bool SRC_GL = false, class S>
__device__ __forceinline__ void fg_to_dst(const Dec<T, W, PPW, CFG> &F, const S &src, int s, int q, const uint32_t *bw,
                                          int h, int G, int sub) {
    constexpr int GS = Dec<T, W, PPW, CFG>::GSS;
    const int off = F.blkoff(s - 1, q), rl = q & (PPW - 1);
    T *d = (s - 1 < F.cfg.a_gfrom() ? F.a_sm(s - 1) : F.a_gl(s - 1)) + off;
    if (Lay<PPW>::kQuad) {
        constexpr int UQ = SRC_GL ? PB_UQ_GL : PB_UQ_SM;
        if (G == GS)
            fg_row<T, IS_G, GS, UQ>(src, RowDst<T, PPW>{d, rl}, bw, h, G, sub);
        else
            fg_row<T, IS_G, 0, UQ>(src, RowDst<T, PPW>{d, rl}, bw, h, G, sub);
    } else {
        constexpr int UM = SRC_GL ? 32 : 8;
        if (G == GS && h >= 32)
            fg_chunks<T, IS_G, GS, PPW, UM>(src, d + rl, bw, h, sub);
        else
            fg_loop<T, IS_G, 0>(src, RowDst<T, PPW>{d, rl}, bw, h, G, sub);
    }
}

// F / G whose source is the never-stored stage n-1 (recomputed from the
// channel) or a global-scratch stage: few ops per frame, each long
// (PB_FAR=1 keeps them out of line; measured slower, so inlined by default)
#ifndef PB_FAR
#define PB_FAR 0
#endif
template <typename T, int W, int PPW, class CFG, bool IS_G>
__device__ __forceinline__ void fg_far_body(Dec<T, W, PPW, CFG> &F, const DOp &o, int q, int G, int sub) {
    const CFG &cfg = F.cfg;
    const int s = o.stage, h = 1 << (s - 1);
    const uint32_t *bw = IS_G ? F.beta_row(s - 1, F.ib(F.cur, s - 1, q)) : nullptr;
    if (s == cfg.n() - 1) {
        if (o.vmode == VM_F)
            fg_to_dst<T, W, PPW, CFG, IS_G>(F, VirtF<T>{F.channel(), cfg.N() >> 1}, s, q, bw, h, G, sub);
        else
            fg_to_dst<T, W, PPW, CFG, IS_G>(
                F, VirtG<T>{F.channel(), F.beta_row(cfg.n() - 1, F.ib(F.cur, cfg.n() - 1, q)), cfg.N() >> 1}, s, q, bw, h,
                G, sub);
    } else {
        const int r = F.ia(F.cur, s, q);
        fg_to_dst<T, W, PPW, CFG, IS_G, true>(F, RowSrc<T, PPW, IS_G && PB_LAST_CS>{F.a_gl(s) + F.blkoff(s, r), r & (PPW - 1)}, s, q, bw,
                                             h, G, sub);
    }
}
template <typename T, int W, int PPW, class CFG, bool IS_G>
__device__ __noinline__ void fg_far(const Params &P, unsigned char *sm, unsigned char *gs, int cur, DOp o, int q, int G,
                                    int sub) {
    Dec<T, W, PPW, CFG> F(P, CFG{&P}, sm, gs);
    F.cur = cur;
    fg_far_body<T, W, PPW, CFG, IS_G>(F, o, q, G, sub);
}

template <typename T, int W, int PPW, class CFG, bool IS_G>
__device__ __forceinline__ void fg_op(Dec<T, W, PPW, CFG> &F, const DOp &o) {
    if (kFuseLeaf<T> && o.fuse < 0) return;  // fused into the next leaf (it reads this op's source)
    const auto mp = F.map(o.pin, o.lgi);
    if (!mp.active || PB_ABL(F.P, 8)) return;
    const CFG &cfg = F.cfg;
    const int s = o.stage, h = 1 << (s - 1), q = mp.q;
    if (s == cfg.n() - 1 || s >= cfg.a_gfrom()) {
        if (PB_FAR)
            fg_far<T, W, PPW, CFG, IS_G>(F.P, F.sm, F.gs, F.cur, o, q, mp.G, mp.sub);
        else
            fg_far_body<T, W, PPW, CFG, IS_G>(F, o, q, mp.G, mp.sub);
    } else {
        const uint32_t *bw = IS_G ? F.beta_row(s - 1, F.ib(F.cur, s - 1, q)) : nullptr;
        const int r = F.ia(F.cur, s, q);
        fg_to_dst<T, W, PPW, CFG, IS_G>(F, RowSrc<T, PPW>{F.a_sm(s) + F.blkoff(s, r), r & (PPW - 1)}, s, q, bw, h,
                                        mp.G, mp.sub);
    }
    if (mp.sub == 0) F.ia(F.cur, s - 1, q) = (uint8_t)q;
}

// ------------------------------------------------- pairwise-exact sums
// numpy float32 pairwise summation (what the reference's sum(axis=1) runs):
// n < 8 sequential from 0; 8 <= n <= 128 eight strided accumulators combined
// ((0+1)+(2+3))+((4+5)+(6+7)); larger n halves recursively.  For power-of-
// two node sizes that is a perfect binary tree over 8*nb accumulators
// (nb = max(1, n/128)), each a sequential sum of min(n,128)/8 elements.
// GS lanes of a group share the 8 accumulator columns, lane sub owning the
// contiguous columns [sub*NA, sub*NA + NA) (NA = 8/GS): the low tree levels
// add in registers, the rest shuffle; the columns of a row of 8 elements are
// one or two quads (128-bit loads) for NA >= 4.

template <int NS>
__device__ __forceinline__ void acc_add(float *acc, float a) {
    acc[0] = __fadd_rn(acc[0], fminf(a, 0.f));
    if (NS == 3) {
        acc[1] = __fadd_rn(acc[1], fmaxf(a, 0.f));
        acc[2] = __fadd_rn(acc[2], a);
    }
}
template <int NS>
__device__ __forceinline__ void acc_init(float *acc, float a) {
    acc[0] = fminf(a, 0.f);
    if (NS == 3) {
        acc[1] = fmaxf(a, 0.f);
        acc[2] = a;
    }
}

// the NA elements e0 .. e0+NA-1 (e0 a multiple of NA)
template <int NA, class S>
__device__ __forceinline__ void load_cols(const S &src, int e0, float (&v)[NA]) {
    if (NA == 8) {
        float q0[4], q1[4];
        src.get4(e0 >> 2, q0);
        src.get4((e0 >> 2) + 1, q1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = q0[j];
            v[(j + 4) & (NA - 1)] = q1[j];
        }
    } else if (NA == 4) {
        float q0[4];
        src.get4(e0 >> 2, q0);
#pragma unroll
        for (int j = 0; j < NA; ++j) v[j] = q0[j];
    } else {
#pragma unroll
        for (int j = 0; j < NA; ++j) v[j] = src.get(e0 + j);
    }
}

// NS = 1: sum min(a,0); NS = 3: (sum min(a,0), sum max(a,0), sum a).
// Valid in the group leader lane.
template <int NS, int GS, class S>
__device__ __forceinline__ void pw_sums(const S &src, int m, bool active, int sub, int lead, float (&out)[NS]) {
    if (m < 8) {
        float r[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) r[t] = 0.f;
        if (active && sub == 0)
            for (int i = 0; i < m; ++i) acc_add<NS>(r, src.get(i));
#pragma unroll
        for (int t = 0; t < NS; ++t) out[t] = r[t];
        return;
    }
    constexpr int NA = 8 / GS;  // accumulator columns per lane
    constexpr int LNA = ilog2(NA);
    constexpr int LG = ilog2(GS);
    // quad-readable sources: lane sub owns the contiguous columns
    // [sub*NA, sub*NA + NA); element-interleaved rows: columns sub + a*GS
    constexpr bool CONTIG = S::kQuad;
    const int blk = m < 128 ? m : 128;
    const int nb = m / blk;
    const int per = blk >> 3;
    const bool act = active && sub < GS;
    float stk[7][NS];
    float carry[NS];
    for (int b = 0; b < nb; ++b) {
        float acc[NA][NS];
        // the NA column chains are independent: interleave them (ILP)
        const int base = b * blk + (CONTIG ? sub * NA : sub);
        if (act) {
            float v[NA];
            if (CONTIG) {
                load_cols<NA>(src, base, v);
            } else {
#pragma unroll
                for (int a = 0; a < NA; ++a) v[a] = src.get(base + a * GS);
            }
#pragma unroll
            for (int a = 0; a < NA; ++a) acc_init<NS>(acc[a], v[a]);
            for (int r = 1; r < per; ++r) {
                if (CONTIG) {
                    load_cols<NA>(src, base + 8 * r, v);
                } else {
#pragma unroll
                    for (int a = 0; a < NA; ++a) v[a] = src.get(base + a * GS + 8 * r);
                }
#pragma unroll
                for (int a = 0; a < NA; ++a) acc_add<NS>(acc[a], v[a]);
            }
        } else {
#pragma unroll
            for (int a = 0; a < NA; ++a)
#pragma unroll
                for (int t = 0; t < NS; ++t) acc[a][t] = 0.f;
        }
        // levels 0..2 of the column tree (column index bits: register bits
        // add in registers, lane bits shuffle)
#pragma unroll
        for (int lv = 0; lv < 3; ++lv) {
            const bool reg = CONTIG ? lv < LNA : lv >= LG;
            if (reg) {
                const int step = CONTIG ? 1 << lv : 1 << (lv - LG);
#pragma unroll
                for (int a = 0; a < NA; a += 2 * step)
#pragma unroll
                    for (int t = 0; t < NS; ++t) acc[a][t] = __fadd_rn(acc[a][t], acc[a + step][t]);
            } else {
                const int d = CONTIG ? 1 << (lv - LNA) : 1 << lv;
#pragma unroll
                for (int a = 0; a < (CONTIG ? 1 : NA); ++a)
#pragma unroll
                    for (int t = 0; t < NS; ++t)
                        acc[a][t] = __fadd_rn(acc[a][t], __shfl_xor_sync(FULL_MASK, acc[a][t], d));
            }
        }
        // combine block sums in numpy's halving order: registers for the
        // common nb <= 2, a binary-counter stack (local memory) beyond
        if (nb <= 2) {
#pragma unroll
            for (int t = 0; t < NS; ++t) carry[t] = b == 0 ? acc[0][t] : __fadd_rn(carry[t], acc[0][t]);
        } else {
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
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) out[t] = carry[t];
}

template <int NS, class S>
__device__ __forceinline__ void pw_sums_rt(const S &src, int m, bool active, int G, int sub, int lead,
                                           float (&out)[NS]) {
    if (G == 1)
        pw_sums<NS, 1>(src, m, active, sub, lead, out);
    else if (G == 2)
        pw_sums<NS, 2>(src, m, active, sub, lead, out);
    else if (G == 4)
        pw_sums<NS, 4>(src, m, active, sub, lead, out);
    else
        pw_sums<NS, 8>(src, m, active, sub, lead, out);
}

// ------------------------------------------------ least reliable positions

template <int K>
struct TopK {
    float m[K];
    int i[K];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            m[k] = INFINITY;
            i[k] = 0x7fffffff;
        }
    }
    __device__ __forceinline__ void insert(float v, int idx) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const bool lt = v < m[k] || (v == m[k] && idx < i[k]);
            const float tm = m[k];
            const int ti = i[k];
            if (lt) {
                m[k] = v;
                i[k] = idx;
                v = tm;
                idx = ti;
            }
        }
    }
    // ascending index scan: only strictly smaller values enter (stable argsort);
    // once placed, the displaced entries shift down unconditionally
    __device__ __forceinline__ void push_scan(float v, int idx) {
        if (K == 2) {  // branch-free
            const bool lt0 = v < m[0], lt1 = v < m[K - 1];
            m[K - 1] = lt0 ? m[0] : (lt1 ? v : m[K - 1]);
            i[K - 1] = lt0 ? i[0] : (lt1 ? idx : i[K - 1]);
            m[0] = lt0 ? v : m[0];
            i[0] = lt0 ? idx : i[0];
            return;
        }
        if (v < m[K - 1]) {
            bool placed = false;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const bool lt = placed || v < m[k];
                placed = lt;
                const float tm = m[k];
                const int ti = i[k];
                if (lt) {
                    m[k] = v;
                    i[k] = idx;
                    v = tm;
                    idx = ti;
                }
            }
        }
    }
};

// ------------------------------------------------------------ selection

// total order of float64 metrics as int64 (-0.0 folded onto +0.0)
__device__ __forceinline__ long long okey(double x) {
    const long long b = __double_as_longlong(x + 0.0);
    return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ long long shfl_xor_ll(long long v, int j) {
    const int lo = __shfl_xor_sync(FULL_MASK, (int)(v & 0xffffffff), j);
    const int hi = __shfl_xor_sync(FULL_MASK, (int)(v >> 32), j);
    return ((long long)hi << 32) | (unsigned)lo;
}
__device__ __forceinline__ long long shfl_ll(long long v, int src) {
    const int lo = __shfl_sync(FULL_MASK, (int)(v & 0xffffffff), src);
    const int hi = __shfl_sync(FULL_MASK, (int)(v >> 32), src);
    return ((long long)hi << 32) | (unsigned)lo;
}
// exclusive warp prefix sum of v in [0, 15]: one ballot per bit, independent
__device__ __forceinline__ int excl_scan4(int v, int lane) {
    const unsigned below = (1u << lane) - 1u;
    int r = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) r += __popc(__ballot_sync(FULL_MASK, (v >> b) & 1) & below) << b;
    return r;
}

// SPC flip sets relative to the ML word over the four LRB slots, emission
// order of listdec.py:157 (_SPC_PAIRS)
__device__ __constant__ uint8_t kSpcPairs[7] = {0x3, 0x5, 0x9, 0x6, 0xA, 0xC, 0xF};

__device__ __forceinline__ int flip_mask(int kind, int c, int odd) {
    if (kind == DK_R1) return c;  // (), (b1), (b2), (b1, b2)
    const int ml = odd ? 1 : 0;
    return c == 0 ? ml : (kSpcPairs[c - 1] ^ ml);
}

// warp-wide max / min of an int64 key via two REDUX steps on its halves
__device__ __forceinline__ long long warp_max_ll(long long v) {
    const int hi = (int)(v >> 32);
    const int mh = __reduce_max_sync(FULL_MASK, hi);
    const unsigned ml = __reduce_max_sync(FULL_MASK, hi == mh ? (unsigned)v : 0u);
    return ((long long)mh << 32) | ml;
}
__device__ __forceinline__ long long warp_min_ll(long long v) {
    const int hi = (int)(v >> 32);
    const int mh = __reduce_min_sync(FULL_MASK, hi);
    const unsigned ml = __reduce_min_sync(FULL_MASK, hi == mh ? (unsigned)v : 0xffffffffu);
    return ((long long)mh << 32) | ml;
}

// Phase B (warp 0, lane = source): survivors -> asg[k] = (source, cand) in
// (source, cand) order.  The L best by (metric desc, source asc, cand asc)
// == listdec.py:63-100 (bounded heap == full sort, tests/oracles.py:74-89).
//
// The L-th best key Tk comes from a k-way merge: slot r of the kept set
// lives in lane r (lanes < L), each source lane exposes its best unconsumed
// candidate (candidates sorted best-first per lane); while the best exposed
// candidate beats the worst kept key it replaces it (REDUX max / min).  Then
// every key > Tk survives, plus the earliest ties == Tk in (source, cand)
// order until L are kept.
template <typename T, int W, int PPW, class CFG, int NC>
__device__ __forceinline__ void select_phase_c(const Dec<T, W, PPW, CFG> &F, const DOp &o) {
    const int lane = F.lane, np = o.pin, L = F.cfg.L();
    constexpr int C = NC;  // candidates per source (compile-time: 2 / 4 / 8)
    const bool vl = lane < np;
    const double pm = vl ? F.pm(F.cur)[lane] : 0.0;
    long long key[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) key[c] = (vl && c < C) ? okey(pm + F.cd(F.par, c, lane)) : LLONG_MIN;
    unsigned mask;
    if (!o.select) {
        mask = vl ? (1u << C) - 1u : 0u;
    } else {
        long long srt[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) srt[c] = key[c];
        // best-first column per lane (Rate-1 columns already are:
        // 0 >= -m1 >= -m2 >= -(m1+m2), monotone under rounding)
        auto cswap = [&](int a, int b) {
            const long long x = srt[a], y = srt[b];
            srt[a] = x > y ? x : y;
            srt[b] = x > y ? y : x;
        };
        if (C == 2) {
            cswap(0, 1);
        } else if (C == 8) {  // Batcher odd-even merge sort, 19 comparators, depth 6
            cswap(0, 1); cswap(2, 3); cswap(4, 5); cswap(6, 7);
            cswap(0, 2); cswap(1, 3); cswap(4, 6); cswap(5, 7);
            cswap(1, 2); cswap(5, 6);
            cswap(0, 4); cswap(1, 5); cswap(2, 6); cswap(3, 7);
            cswap(2, 4); cswap(3, 5);
            cswap(1, 2); cswap(3, 4); cswap(5, 6);
        }
        F.mark(4);
        // kept set: slot = lane (< L); start from every source's best.  The
        // lane's exposed candidate is srt[0] of its shifted column.
        long long kept = lane < L ? srt[0] : LLONG_MAX;
#pragma unroll
        for (int c = 0; c < NC; ++c) srt[c] = c + 1 < C ? srt[c + 1 < NC ? c + 1 : c] : LLONG_MIN;
        long long worst;
        for (;;) {
            const long long cand = srt[0];
            const long long best = warp_max_ll(cand);
            worst = warp_min_ll(kept);
            if (best <= worst) break;
            const int from = __ffs(__ballot_sync(FULL_MASK, cand == best)) - 1;
            const int into = __ffs(__ballot_sync(FULL_MASK, kept == worst)) - 1;
            if (lane == from) {
#pragma unroll
                for (int c = 0; c < NC; ++c) srt[c] = c + 1 < NC ? srt[c + 1] : LLONG_MIN;
            }
            if (lane == into) kept = best;
        }
        const long long Tk = worst;  // kept is unchanged since the exit test
        F.mark(5);
        // Tk = the L-th best key; keep all better, then the earliest ties
        int gt = 0, eq = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            gt += key[c] > Tk;
            eq += key[c] == Tk;
        }
        const int need = L - (int)__reduce_add_sync(FULL_MASK, (unsigned)gt);
        // ties at Tk: the earliest `need` in (source, cand) order; with no
        // surplus tie (the usual case) every tie survives and no scan is needed
        const int eqt = (int)__reduce_add_sync(FULL_MASK, (unsigned)eq);
        int r = eqt <= need ? 0 : excl_scan4(eq, lane);
        mask = 0u;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            if (key[c] > Tk) {
                mask |= 1u << c;
            } else if (key[c] == Tk) {
                if (r < need) mask |= 1u << c;
                ++r;
            }
        }
    }
    F.mark(6);
    int k = excl_scan4(__popc(mask), lane);
    uint8_t *asg = F.asg(F.par);
    while (mask) {
        const int c = __ffs(mask) - 1;
        mask &= mask - 1;
        asg[2 * k] = (uint8_t)lane;
        asg[2 * k + 1] = (uint8_t)c;
        ++k;
    }
}

template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void select_phase(const Dec<T, W, PPW, CFG> &F, const DOp &o) {
    if (o.ncand == 2)
        select_phase_c<T, W, PPW, CFG, 2>(F, o);
    else if (o.ncand == 4)
        select_phase_c<T, W, PPW, CFG, 4>(F, o);
    else
        select_phase_c<T, W, PPW, CFG, 8>(F, o);
}

// ----------------------------------------------------- leaf word + chain

// 32-bit word w of the leaf word of decision (p, c) (m < 32: the m-bit value)
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ uint32_t leaf_word(const Dec<T, W, PPW, CFG> &F, int b, int kind, int m, int p, int c,
                                              int w) {
    const uint32_t fullw = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
    if (kind == DK_R0) return 0u;
    if (kind == DK_REP) {
        const bool ones = F.cflag(b)[p] ? (c == 0) : (c == 1);
        return ones ? fullw : 0u;
    }
    uint32_t v = F.hard(b, w, p);
    const int fm = flip_mask(kind, c, F.cflag(b)[p]);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if ((fm >> j) & 1) {
            const int pos = F.clrb(b, j, p);
            if ((pos >> 5) == w) v ^= 1u << (pos & 31);
        }
    return v;
}

__device__ __forceinline__ uint32_t bits_get(const uint32_t *row, int off, int len) {
    const uint32_t msk = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    return (row[off >> 5] >> (off & 31)) & msk;
}
__device__ __forceinline__ void bits_put(uint32_t *row, int off, int len, uint32_t v) {
    const uint32_t msk = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    uint32_t &w = row[off >> 5];
    w = (w & ~(msk << (off & 31))) | ((v & msk) << (off & 31));
}

// Leaf word of path k (decision (p, c)) into dst[E - m, E), then the leaf's
// chain of Combines t .. sE-1 in place:
//   dst[E - 2^(s+1), E - 2^s) = slot_s[row_s] ^ dst[E - 2^s, E)
// (listdec.py:327-332 with the right child's bits kept where they are).
// The levels below 32 bits all land in the node's last word: they run in a
// register from prefetched slot words, one store; wider levels go word-
// parallel over the group's lanes.  Called by all lanes of a warp.
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void word_and_chain(const Dec<T, W, PPW, CFG> &F, int b, const DOp &o, int kind, bool active,
                                               int G, int sub, int p, int c, int ibuf, int ipath, uint32_t *dst,
                                               int sE) {
    const int t = o.stage, m = 1 << t, E = 1 << sE;
    if (active) {
        if (m >= 32) {
            for (int w = sub; w < (m >> 5); w += G) dst[((E - m) >> 5) + w] = leaf_word(F, b, kind, m, p, c, w);
        } else if (sub == 0) {
            const int s_sub = sE < 5 ? sE : 5;
            const int W0 = E >= 32 ? E - 32 : 0;
            uint32_t slw[5];
#pragma unroll
            for (int s = 0; s < 5; ++s)
                slw[s] = (s >= t && s < s_sub) ? F.beta_row(s, F.ib(ibuf, s, ipath))[0] : 0u;
            uint32_t R = leaf_word(F, b, kind, m, p, c, 0) << (E - m - W0);
#pragma unroll
            for (int s = 0; s < 5; ++s)
                if (s >= t && s < s_sub) {
                    const int seg = 1 << s;
                    const uint32_t msk = (1u << seg) - 1u;
                    R |= ((slw[s] ^ (R >> (E - seg - W0))) & msk) << (E - 2 * seg - W0);
                }
            if (E >= 32)
                dst[(E >> 5) - 1] = R;
            else
                bits_put(dst, 0, E, R);
        }
    }
    __syncwarp();
    for (int s = t > 5 ? t : 5; s < sE; ++s) {
        const int seg = 1 << s;
        if (active) {
            const uint32_t *sl = F.beta_row(s, F.ib(ibuf, s, ipath));
            const int a = (E - 2 * seg) >> 5, bb = (E - seg) >> 5;
            for (int w = sub; w < (seg >> 5); w += G) dst[a + w] = sl[w] ^ dst[bb + w];
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------- leaves

template <typename T, int W, int PPW, class CFG, class S>
__device__ __forceinline__ void leaf_sums(Dec<T, W, PPW, CFG> &F, const DOp &o, int kind, const S &src, int q, bool active,
                                          int G, int sub) {
    const int m = 1 << o.stage;
    const int lead = F.lane - sub;
    if (kind == DK_R0) {
        float r[1];
        pw_sums_rt<1>(src, m, active, G, sub, lead, r);
        if (active && sub == 0) F.pm(F.cur)[q] += (double)r[0];  // listdec.py:341-343
    } else {
        float r[3];
        pw_sums_rt<3>(src, m, active, G, sub, lead, r);
        if (active && sub == 0) {  // listdec.py:348-358
            const bool ones_first = r[2] < 0.f;
            const double neg = (double)r[0], pos = (double)r[1];
            F.cd(F.par, 0, q) = ones_first ? -pos : neg;
            F.cd(F.par, 1, q) = ones_first ? neg : -pos;
            F.cflag(F.par)[q] = ones_first;
        }
    }
}


// Rate-1 / SPC scan: stable K least reliable positions, hard decisions,
// parity and syndrome of the hard word.  Gl (<= G) lanes of the path's group
// scan (one lane unless the node is large); the rest idle.
template <typename T, int W, int PPW, class CFG, int K, class S>
__device__ __forceinline__ void leaf_scan(Dec<T, W, PPW, CFG> &F, const DOp &o, int kind, const S &src, int q,
                                          bool active, int G, int sub) {
    const Params &P = F.P;
    const CFG &cfg = F.cfg;
    const int m = 1 << o.stage;
    int Gl = m >> 4;
    Gl = Gl < 1 ? 1 : (Gl > G ? G : Gl);
    TopK<K> tk;
    tk.init();
    int par = 0;
    float mag4[4] = {0.f, 0.f, 0.f, 0.f};  // SPC of size 4: |a| by position
    if (Gl == 1) {
        if (active && sub == 0 && m >= 32) {
            // whole 32-element blocks: all (quad) loads in flight, then NCH
            // independent scan chains (element j in chain j % NCH, ascending
            // within a chain), merged by (magnitude, index) at the end
            constexpr int NCH = K == 2 ? 4 : 2;
            TopK<K> tc[NCH];
#pragma unroll
            for (int h = 0; h < NCH; ++h) tc[h].init();
            for (int w0 = 0; w0 < m; w0 += 32) {
                float v[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float qv[4];
                    src.get4((w0 >> 2) + j, qv);
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[4 * j + e] = qv[e];
                }
                uint32_t word = 0u;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    word |= (v[j] < 0.f ? 1u : 0u) << j;
                    tc[j % NCH].push_scan(fabsf(v[j]), w0 + j);
                }
                F.hard(F.par, w0 >> 5, q) = word;
                par ^= __popc(word);
            }
            tk = tc[0];
#pragma unroll
            for (int h = 1; h < NCH; ++h)
#pragma unroll
                for (int e = 0; e < K; ++e) tk.insert(tc[h].m[e], tc[h].i[e]);
        } else if (K == 4 && active && sub == 0 && m == 4) {
            // SPC of size 4 (the default cap): every position is a least
            // reliable one -- a stable 5-comparator sort of (|a|, index)
            float qv[4];
            src.get4(0, qv);
            uint32_t word = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                word |= (qv[e] < 0.f ? 1u : 0u) << e;
                mag4[e] = fabsf(qv[e]);
                tk.m[e] = mag4[e];
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
            F.hard(F.par, 0, q) = word;
            par ^= __popc(word);
        } else if (S::kQuad && active && sub == 0 && m >= 4) {
            // m = 4, 8, 16: quads, loads first
            float v[16];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (4 * j < m) {
                    float qv[4];
                    src.get4(j, qv);
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[4 * j + e] = qv[e];
                }
            uint32_t word = 0u;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < m) {
                    word |= (v[j] < 0.f ? 1u : 0u) << j;
                    tk.push_scan(fabsf(v[j]), j);
                }
            F.hard(F.par, 0, q) = word;
            par ^= __popc(word);
        } else if (active && sub == 0) {
            uint32_t word = 0u;
            for (int j = 0; j < m; ++j) {
                const float a = src.get(j);
                word |= (a < 0.f ? 1u : 0u) << j;
                tk.push_scan(fabsf(a), j);
            }
            F.hard(F.par, 0, q) = word;
            par ^= __popc(word);
        }
        F.mark(2);
    } else {
        const int lgl = 31 - __clz(Gl);
        const bool scan = active && sub < Gl;
        uint32_t hword = 0u;
        const int iters = (m + Gl - 1) >> lgl;
        const int hq = active ? q : F.warp * PPW;
        const int gshift = F.lane - sub;  // group leader lane
        const uint32_t gmask = Gl == 32 ? 0xffffffffu : ((1u << Gl) - 1u);
        for (int it = 0; it < iters; ++it) {
            const int i = (it << lgl) + sub;
            const bool valid = scan && i < m;
            const float a = valid ? src.get(i) : 0.f;
            const bool neg = valid && a < 0.f;
            if (valid) tk.push_scan(fabsf(a), i);
            const uint32_t gb = (__ballot_sync(FULL_MASK, neg) >> gshift) & gmask;
            const int base = it << lgl;
            hword |= gb << (base & 31);
            if (((base + Gl) & 31) == 0 || it == iters - 1) {
                if (scan && sub == 0) F.hard(F.par, base >> 5, hq) = hword;
                par ^= __popc(hword);
                hword = 0u;
            }
        }
        for (int d = 1; d < Gl; d <<= 1) {
            float om[K];
            int oi[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                om[k] = __shfl_xor_sync(FULL_MASK, tk.m[k], d);
                oi[k] = __shfl_xor_sync(FULL_MASK, tk.i[k], d);
            }
#pragma unroll
            for (int k = 0; k < K; ++k) tk.insert(om[k], oi[k]);
        }
    }
    if (!(active && sub == 0)) return;
#pragma unroll
    for (int k = 0; k < K; ++k) F.clrb(F.par, k, q) = (uint16_t)(tk.i[k] < m ? tk.i[k] : 0);
    if (kind == DK_R1) {  // listdec.py:360-372
        const double w1 = (double)tk.m[0], w2 = (double)tk.m[1];
        F.cd(F.par, 0, q) = 0.0;
        F.cd(F.par, 1, q) = -w1;
        F.cd(F.par, 2, q) = -w2;
        F.cd(F.par, 3, q) = -(w1 + w2);
        F.cflag(F.par)[q] = 0;
        return;
    }
    // SPC, listdec.py:373-394: deltas sum the net flips in ascending position
    const int odd = par & 1;
    F.cflag(F.par)[q] = (uint8_t)odd;
    // rank of each LRB slot by position (the reference sums net flips in
    // ascending position order); all indices static
    int rk[4];
    double wr[4];  // magnitudes by position rank
    if (m == 4 && Gl == 1) {  // the four positions are 0..3: rank = position
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            rk[x] = tk.i[x & (K - 1)];
            wr[x] = (double)mag4[x];
        }
    } else {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            rk[x] = 0;
#pragma unroll
            for (int y = 0; y < 4; ++y) rk[x] += tk.i[y & (K - 1)] < tk.i[x & (K - 1)] ? 1 : 0;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double v = 0.0;
#pragma unroll
            for (int x = 0; x < 4; ++x) v = rk[x] == r ? (double)tk.m[x & (K - 1)] : v;
            wr[r] = v;
        }
    }
#pragma unroll
    for (int c = 0; c < kMaxCand; ++c) {
        if (c < o.ncand) {
            const int fm = flip_mask(DK_SPC, c, odd);
            int fr = 0;  // flip set in rank order
#pragma unroll
            for (int x = 0; x < 4; ++x) fr |= ((fm >> x) & 1) << rk[x];
            double accd = 0.0;
            bool any = false;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if ((fr >> r) & 1) {
                    accd = any ? accd + wr[r] : wr[r];
                    any = true;
                }
            F.cd(F.par, c, q) = any ? -accd : 0.0;
        }
    }
}

template <typename T, int W, int PPW, class CFG, class S>
__device__ __forceinline__ void leaf_phase_a(Dec<T, W, PPW, CFG> &F, const DOp &o, int kind, const S &src, int q,
                                             bool active, int G, int sub) {
    if (kind == DK_R0 || kind == DK_REP)
        leaf_sums(F, o, kind, src, q, active, G, sub);
    else if (kind == DK_R1)
        leaf_scan<T, W, PPW, CFG, 2>(F, o, kind, src, q, active, G, sub);
    else
        leaf_scan<T, W, PPW, CFG, 4>(F, o, kind, src, q, active, G, sub);
}

// leaves reading the channel, the recomputed stage n-1 or a global-scratch
// stage: rare, kept out of line (see fg_far)
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void leaf_read_far_body(Dec<T, W, PPW, CFG> &F, const DOp &o, int kind, int q, bool active,
                                                   int G, int sub) {
    const CFG &cfg = F.cfg;
    const int t = o.stage;
    const int qq = active ? q : F.warp * PPW;
    if (t == cfg.n()) {
        leaf_phase_a(F, o, kind, ChanSrc<T>{F.channel()}, q, active, G, sub);
    } else if (t == cfg.n() - 1) {
        if (o.vmode == VM_F)
            leaf_phase_a(F, o, kind, VirtF<T>{F.channel(), cfg.N() >> 1}, q, active, G, sub);
        else
            leaf_phase_a(F, o, kind, VirtG<T>{F.channel(), F.beta_row(cfg.n() - 1, F.ib(F.cur, cfg.n() - 1, qq)), cfg.N() >> 1}, q,
                         active, G, sub);
    } else {
        const int r = F.ia(F.cur, t, qq);
        leaf_phase_a(F, o, kind, RowSrc<T, PPW, PB_LAST_CS>{F.a_gl(t) + F.blkoff(t, r), r & (PPW - 1)}, q, active, G, sub);
    }
}
template <typename T, int W, int PPW, class CFG>
__device__ __noinline__ void leaf_read_far(const Params &P, unsigned char *sm, unsigned char *gs, int cur, int par,
                                           DOp o, int kind, int q, bool active, int G, int sub) {
    Dec<T, W, PPW, CFG> F(P, CFG{&P}, sm, gs);
    F.cur = cur;
    F.par = par;
    leaf_read_far_body(F, o, kind, q, active, G, sub);
}

// dispatch on where the node's LLRs live
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void leaf_read(Dec<T, W, PPW, CFG> &F, const DOp &o, int kind, int q, bool active, int G,
                                          int sub) {
    const CFG &cfg = F.cfg;
    const int t = o.stage;
    if constexpr (kFuseLeaf<T>) {
        if (o.fuse > 0) {  // f / g of the parent's shared-memory row (DOp::fuse)
            const int qq = active ? q : F.warp * PPW;
            const int r = F.ia(F.cur, t + 1, qq);
            const RowSrc<T, PPW> in{F.a_sm(t + 1) + F.blkoff(t + 1, r), r & (PPW - 1)};
            if (o.fuse == 1)
                leaf_phase_a(F, o, kind, FusedSrc<T, false, RowSrc<T, PPW>>{in, nullptr, 1 << t}, q, active, G, sub);
            else
                leaf_phase_a(F, o, kind, FusedSrc<T, true, RowSrc<T, PPW>>{in, F.beta_row(t, F.ib(F.cur, t, qq)), 1 << t},
                             q, active, G, sub);
            return;
        }
    }
    if (t >= cfg.n() - 1 || t >= cfg.a_gfrom()) {
        if (PB_FAR && !PB_PROFILE)
            leaf_read_far<T, W, PPW, CFG>(F.P, F.sm, F.gs, F.cur, F.par, o, kind, q, active, G, sub);
        else
            leaf_read_far_body(F, o, kind, q, active, G, sub);
    } else {
        const int qq = active ? q : F.warp * PPW;
        const int r = F.ia(F.cur, t, qq);
        leaf_phase_a(F, o, kind, RowSrc<T, PPW>{F.a_sm(t) + F.blkoff(t, r), r & (PPW - 1)}, q, active, G, sub);
    }
}

template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void leaf_op(Dec<T, W, PPW, CFG> &F, const DOp &o) {
    const Params &P = F.P;
    const CFG &cfg = F.cfg;
    int kind = o.kind;
    if (kind == DK_R1 && o.stage == 0) kind = DK_REP;  // listdec.py:347

    // Phase A: per-source sums / scans, this warp's sources
    if (!PB_ABL(P, 1)) {
        const auto mp = F.map(o.pin, o.lgi);
        leaf_read(F, o, kind, mp.q, mp.active, mp.G, mp.sub);
    }
    F.sync();
    F.mark(0);

    const bool fork = kind != DK_R0;
    if (fork) {
        if (F.warp == 0 && !PB_ABL(P, 2)) select_phase(F, o);
        if (F.warp == 0 && PB_ABL(P, 2) && F.lane < o.pout) {  // timing only: a valid dummy choice
            F.asg(F.par)[2 * F.lane] = (uint8_t)(F.lane % o.pin);
            F.asg(F.par)[2 * F.lane + 1] = 0;
        }
        F.sync();
    }
    F.mark(1);

    // Phase C: materialise survivors k < pout (this warp's)
    const auto mp = F.map(o.pout, o.lgo);
    const int k = mp.q;
    const int nxt = fork ? F.cur ^ 1 : F.cur;
    const int b = F.par;
    int p = k, c = 0;
    if (fork && mp.active) {
        p = F.asg(b)[2 * k];
        c = F.asg(b)[2 * k + 1];
    }
    if (fork && mp.active && mp.sub == 0) {
        F.pm(nxt)[k] = F.pm(F.cur)[p] + F.cd(b, c, p);  // listdec.py:415
        for (int x = 0; x < cfg.idx_stride(); ++x) {  // lazy copy: inherit the source's rows
            F.iaw(nxt, x, k) = F.iaw(F.cur, x, p);
            F.ibw(nxt, x, k) = F.ibw(F.cur, x, p);
        }
    }
    F.mark(7);
    const int sE = o.target;
    if (sE < cfg.n() && !PB_ABL(P, 4)) {
        word_and_chain(F, b, o, kind, mp.active, mp.G, mp.sub, p, c, F.cur, mp.active ? p : 0, F.beta_row(sE, k), sE);
        if (mp.active && mp.sub == 0) F.ib(nxt, sE, k) = (uint8_t)k;
    }
    __syncwarp();
    F.cur = nxt;
    if (fork) {
        F.lpar = F.par;
        F.par ^= 1;
    }
}

// ------------------------------------------------------------ finalise

__device__ __forceinline__ void polar_transform_words(uint32_t *x, int N, int lane) {
    const int nw = N >= 32 ? N >> 5 : 1;
    const int hin = N < 32 ? N : 32;
    const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    for (int w = lane; w < nw; w += 32) {
        uint32_t v = x[w];
#pragma unroll
        for (int b = 0; b < 5; ++b)
            if ((1 << b) < hin) v ^= (v >> (1 << b)) & masks[b];
        x[w] = v;
    }
    __syncwarp();
    for (int H = 1; H < nw; H <<= 1) {
        for (int w = lane; w < nw; w += 32)
            if ((w & H) == 0) x[w] ^= x[w + H];
        __syncwarp();
    }
}

template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void build_root(const Dec<T, W, PPW, CFG> &F, const DOp &fo, int k, uint32_t *dst) {
    int kind = fo.kind;
    if (kind == DK_R1 && fo.stage == 0) kind = DK_REP;
    int p = k, c = 0;
    const int b = F.lpar;
    if (kind != DK_R0) {
        p = F.asg(b)[2 * k];
        c = F.asg(b)[2 * k + 1];
    }
    if (F.cfg.N() < 32 && F.lane == 0) dst[0] = 0u;
    __syncwarp();
    word_and_chain(F, b, fo, kind, true, 32, F.lane, p, c, F.cur, k, dst, F.cfg.n());
    __syncwarp();
}

// CRC syndrome of codeword x (N bits, packed) in the codeword domain:
// XOR of the syndrome rows of its set bits by nibble tables, warp-parallel;
// equal to the u-domain check of extract_payload + crc_check
// (encode.py:76-87, codes.py:150-156) because u = x G_N (G_N involution).
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ uint32_t codeword_syndrome(const Dec<T, W, PPW, CFG> &F, const uint32_t *x) {
    const int N = F.cfg.N(), nw = N >= 32 ? N >> 5 : 1;
    uint32_t s = 0u;
    for (int w = F.lane; w < nw; w += 32) {
        uint32_t v = x[w];
        if (N < 32) v &= (1u << N) - 1u;
        const uint32_t *t = F.P.xsyn4 + (size_t)w * 128;  // 8 nibbles x 16 entries per word
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) s ^= __ldg(t + nb * 16 + ((v >> (4 * nb)) & 15u));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) s ^= __shfl_xor_sync(FULL_MASK, s, d);
    return s;
}

// listdec.py:289-308: among CRC-passing survivors the strictly greater
// metric wins, earliest survivor on ties; with none passing, the best metric
// overall.  Equivalently: visit survivors by (metric desc, index asc) and
// take the first that passes -- normally the very first, so only one or two
// codewords are built and checked per frame.
template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void finalize(Dec<T, W, PPW, CFG> &F, long long f, int np) {
    const Params &P = F.P;
    const CFG &cfg = F.cfg;
    const int lane = F.lane;
    const DOp fo = P.prog[P.final_op];
    const bool live = lane < np;
    const double pmk = live ? F.pm(F.cur)[lane] : -INFINITY;
    const int rw = cfg.root_words();
    uint32_t *u = F.root();
    if (P.path_cw) {  // decode_paths: every survivor's codeword, metric and CRC flag
        for (int kk = 0; kk < np; ++kk) {
            uint32_t *dst = P.path_cw + ((size_t)f * cfg.L() + kk) * rw;
            build_root(F, fo, kk, dst);
            const uint32_t syn = codeword_syndrome(F, dst);
            if (lane == 0) P.path_crc[(size_t)f * cfg.L() + kk] = cfg.has_crc() && syn == cfg.crc_const();
        }
        if (live) P.path_pm[(size_t)f * cfg.L() + lane] = pmk;
        __syncwarp();
    }
    unsigned tried = 0u;
    int first = -1, wnr = -1;
    double wpm = -INFINITY;
    for (int it = 0; it < np; ++it) {
        // best untried survivor: max metric, lowest index
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
        if (!cfg.has_crc() || PB_ABL(P, 16)) {
            wnr = bk;
            wpm = bm;
            break;
        }
        build_root(F, fo, bk, u);
        if (codeword_syndrome(F, u) == cfg.crc_const()) {
            wnr = bk;
            wpm = bm;
            break;
        }
    }
    const bool wok = wnr >= 0 && cfg.has_crc();
    if (wnr < 0) {
        wnr = first;
        wpm = __shfl_sync(FULL_MASK, pmk, first & 31);
    }
    if (P.info_out) {
        if (!wok) build_root(F, fo, wnr, u);  // the passing winner's codeword is already in u
        polar_transform_words(u, cfg.N(), lane);
        uint8_t *out = P.info_out + (size_t)f * cfg.k();
        for (int i = lane; i < cfg.k(); i += 32) {
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
__device__ __forceinline__ float ingest(float a) {
    if (Elem<T>::kInt) return fminf(fmaxf(rintf(a * 4.f), -127.f), 127.f);  // clip(rint(4x)), half-even
    return fminf(fmaxf(a, -1048576.f), 1048576.f);                             // clamp_llr (kernels.py:34-36)
}

template <typename T, int W, int PPW, class CFG>
__device__ __forceinline__ void load_channel(const Dec<T, W, PPW, CFG> &F, long long f) {
    const Params &P = F.P;
    const CFG &cfg = F.cfg;
    T *ch = F.channel();
    const int N = cfg.N(), tid = threadIdx.x & (32 * W - 1);
    if (P.in_type == PB_IN_I8) {
        const int8_t *src = reinterpret_cast<const int8_t *>(P.llr) + (size_t)f * N;
        for (int i = tid; i < N; i += 32 * W) ch[i] = (T)src[i];
        return;
    }
    const float *src = reinterpret_cast<const float *>(P.llr) + (size_t)f * N;
    if ((N & 3) == 0) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        for (int i = tid; i < (N >> 2); i += 32 * W) {
            const float4 v = __ldcs(s4 + i);  // read once: evict-first
            Elem<T>::st(ch + 4 * i + 0, ingest<T>(v.x));
            Elem<T>::st(ch + 4 * i + 1, ingest<T>(v.y));
            Elem<T>::st(ch + 4 * i + 2, ingest<T>(v.z));
            Elem<T>::st(ch + 4 * i + 3, ingest<T>(v.w));
        }
    } else {
        for (int i = tid; i < N; i += 32 * W) Elem<T>::st(ch + i, ingest<T>(src[i]));
    }
}

#ifndef PB_OP_PREFETCH
#define PB_OP_PREFETCH 0
#endif
// The op program interpreted from the schedule (runtime configuration).
struct RtOps {
    template <typename T, int W, int PPW, class CFG>
    __device__ __forceinline__ static void run(Dec<T, W, PPW, CFG> &F, int &np, bool prof) {
        const Params &P = F.P;
        const DOp *prog = F.prog;
#if PB_OP_PREFETCH
        DOp onext = prog[0];
#endif
        for (int oi = 0; oi < P.n_ops; ++oi) {
            const long long t0 = prof ? clock64() : 0;
#if PB_OP_PREFETCH
            const DOp o = onext;
            if (oi + 1 < P.n_ops) onext = prog[oi + 1];
#else
            // loaded at the top of the op (constant bank, or an L1 / shared
            // hit): a prefetched next op stays live across the whole op body
            // and was spilled and reloaded around every op (~15 local
            // accesses per op)
            const DOp o = P.prog_inline ? P.iprog[oi] : prog[oi];
#endif
            switch (o.kind) {
                case DK_F:
                    fg_op<T, W, PPW, CFG, false>(F, o);
                    break;
                case DK_G:
                    fg_op<T, W, PPW, CFG, true>(F, o);
                    break;
                case DK_NOP:
                    break;
                default:
                    leaf_op(F, o);
                    np = o.pout;
                    break;
            }
            if (P.sync_mask >= 0 && (oi & P.sync_mask) == 0)
                __syncthreads();  // regroup the CTA's frames (shared instruction fetch)
            else
                __syncwarp();
            if (prof) {
                const long long t1 = clock64();
                long long *oc = P.op_cycles + oi * 12;
                oc[0] = t1 - t0;
                oc[1] = t0;
                for (int x = 0; x < 10; ++x) {
                    oc[2 + x] = F.ph[x];
                    F.ph[x] = 0;
                }
            }
        }
    }
};

// Persistent frame loop.  A CTA holds P.fpc frames of W warps each; all of
// them step through the same op program (the schedule is per code, not per
// frame) and start together, so the SM's warps share instruction fetch.
template <typename T, int W, int PPW, class CFG, class OPS>
__device__ __forceinline__ void decode_frames(const Params &P, const CFG &cfg) {
    const int grp = threadIdx.x / (32 * W);
    const long long slot = (long long)blockIdx.x * P.fpc + grp;
    unsigned char *gs = P.gscratch ? P.gscratch + (size_t)slot * cfg.gbytes() : nullptr;
    unsigned char *sm = g_smem + (size_t)grp * cfg.smem_bytes();
    const long long stride = (long long)gridDim.x * P.fpc;
    // the op program, read by every frame once per op: staged in shared memory
    const DOp *prog = P.prog;
    if (P.prog_smem) {
        DOp *sp = reinterpret_cast<DOp *>(g_smem + (size_t)P.fpc * cfg.smem_bytes());
        for (int i = threadIdx.x; i < P.n_ops; i += blockDim.x) sp[i] = P.prog[i];
        __syncthreads();
        prog = sp;
    }
    // adaptive pass: the frames the single-path pass could not settle
    // (count and row map on the device, written by k_ssc)
    const long long batch = P.batch_dev ? (long long)*P.batch_dev : P.batch;
    for (long long f0 = (long long)blockIdx.x * P.fpc; f0 < batch; f0 += stride) {
        // tail: idle slots decode the last frame again and write nothing
        const long long fi = f0 + grp < batch ? f0 + grp : batch - 1;
        const long long f = P.frame_map ? (long long)P.frame_map[fi] : fi;
        const bool own = f0 + grp < batch;
        Dec<T, W, PPW, CFG> F(P, cfg, sm, gs);
        F.prog = prog;
        load_channel(F, f);
        if ((threadIdx.x & (32 * W - 1)) == 0) F.pm(0)[0] = 0.0;
        F.sync();
        int np = 1;
        const bool prof = PB_PROFILE && P.op_cycles && blockIdx.x == 0 && f == 0 && threadIdx.x == 0;
        long long phbuf[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (prof) F.ph = phbuf;
        OPS::run(F, np, prof);
        F.sync();
        if (F.warp == 0 && own) finalize(F, f, np);
        if (P.fpc > 1)
            __syncthreads();
        else
            F.sync();
    }
}

template <typename T, int W, int PPW, bool CHG>
__global__ void __launch_bounds__(shape_max_threads(W, PPW), 1) k_decode(const __grid_constant__ Params P) {
    decode_frames<T, W, PPW, RtCfg<CHG>, RtOps>(P, RtCfg<CHG>{&P});
}

#ifndef __CUDACC_RTC__
template <typename T, int W, int PPW, bool CHG>
cudaError_t launch_t(const Params *p, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e =
        cudaFuncSetAttribute(k_decode<T, W, PPW, CHG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_decode<T, W, PPW, CHG><<<grid, 32 * W * p->fpc, smem, st>>>(*p);
    return cudaGetLastError();
}
template <typename T, int W, int PPW, bool CHG>
cudaError_t occ_t(size_t smem, int fpc, int *bps) {
    cudaError_t e =
        cudaFuncSetAttribute(k_decode<T, W, PPW, CHG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k_decode<T, W, PPW, CHG>, 32 * W * fpc, smem);
}

#endif

}  // namespace pb


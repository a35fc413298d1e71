// decode_kernel.cu -- Fast-SSC list-CRC decode kernel for sm_100a.
//
// One warp decodes one frame at a time (persistent loop over frames); the
// L path slots of the list live on the warp's lanes.  Per op:
//   F / G      element-parallel over (path, element): P active paths split the
//              32 lanes into groups of G = 32/pow2(P) lanes per path
//              (kernels.py:39-56, listdec.py:319-326)
//   leaves     group scans of the node LLRs: pairwise-exact float sums
//              (Rate-0 / Rep, listdec.py:340-359), stable two/four least
//              reliable positions + hard decisions + parity (Rate-1 / SPC,
//              listdec.py:360-394)
//   selection  lane = source path; each lane's candidates are a sorted
//              column, the L best are found by warp-shuffle bitonic sorts of
//              the columns with early exit (listdec.py:63-100)
//   materialise survivors copy the source's row-index vectors (lazy copy,
//              listdec.py:103-143,397-434), write their leaf word and run the
//              leaf's chain of Combines in place (listdec.py:327-332)
//   finalise   CRC by per-path GF(2) syndrome == constant, strict-max pick
//              among CRC-passing paths (listdec.py:289-308), polar transform
//              of the winner and payload gather (encode.py:29-53,76-87).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "decoder.cuh"

#define PB_IN_F32 0
#define PB_IN_I8 1

namespace pb {

#define FULL_MASK 0xffffffffu

template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static constexpr bool kInt = false;
    static __device__ __forceinline__ float ld(const float *p) { return *p; }
    static __device__ __forceinline__ void st(float *p, float v) { *p = v; }
};
template <>
struct Elem<int8_t> {
    static constexpr bool kInt = true;
    static __device__ __forceinline__ float ld(const int8_t *p) { return (float)*p; }
    static __device__ __forceinline__ void st(int8_t *p, float v) { *p = (int8_t)__float2int_rn(v); }
};

// min-sum F: sign(a) sign(b) min(|a|,|b|); zero products give a signed zero,
// numerically equal to the reference's 0 (kernels.py:39-48)
__device__ __forceinline__ float f_op(float a, float b) {
    unsigned s = (__float_as_uint(a) ^ __float_as_uint(b)) & 0x80000000u;
    return __uint_as_float(__float_as_uint(fminf(fabsf(a), fabsf(b))) | s);
}

// G: b + (1 - 2 beta) a, one correctly rounded add (kernels.py:51-56);
// int8 mode saturates to [-127, 127]
template <typename T>
__device__ __forceinline__ float g_op(float a, float b, unsigned bit) {
    float v = __fadd_rn(b, __uint_as_float(__float_as_uint(a) ^ (bit << 31)));
    if (Elem<T>::kInt) v = fminf(fmaxf(v, -127.f), 127.f);
    return v;
}

__device__ __forceinline__ int pow2ceil(int x) { return x <= 1 ? 1 : 1 << (32 - __clz(x - 1)); }

// Reads the LLRs of one node for one path: a stored alpha row, the channel
// (root leaf) or the never-stored stage n-1, recomputed from the channel.
template <typename T>
struct Src {
    const T *p;
    const T *ch;
    const uint32_t *bw;
    int half;
    int mode;
    __device__ __forceinline__ float get(int i) const {
        if (mode == VM_NONE) return Elem<T>::ld(p + i);
        float a = Elem<T>::ld(ch + i), b = Elem<T>::ld(ch + i + half);
        if (mode == VM_F) return f_op(a, b);
        unsigned bit = (bw[i >> 5] >> (i & 31)) & 1u;
        return g_op<T>(a, b, bit);
    }
};

template <typename T>
struct Frame {
    const Params &P;
    unsigned char *fs;  // this frame's shared memory block
    unsigned char *gs;  // this frame's global scratch block
    int cur;            // which half of the double-buffered path state is live

    __device__ Frame(const Params &p, unsigned char *f, unsigned char *g) : P(p), fs(f), gs(g), cur(0) {}

    __device__ __forceinline__ T *alpha_row(int s, int row) const {
        unsigned char *base = s >= P.lay.a_gfrom ? gs : fs;
        return reinterpret_cast<T *>(base + P.lay.a_off[s]) + row * P.lay.a_stride[s];
    }
    __device__ __forceinline__ uint32_t *beta_row(int s, int row) const {
        return reinterpret_cast<uint32_t *>(fs + P.lay.b_off[s]) + row * P.lay.b_stride[s];
    }
    __device__ __forceinline__ T *channel() const { return reinterpret_cast<T *>(fs + P.lay.ch_off); }
    __device__ __forceinline__ double *pm(int buf) const {
        return reinterpret_cast<double *>(fs + P.lay.pm_off) + buf * P.L;
    }
    __device__ __forceinline__ uint32_t *syn(int buf) const {
        return reinterpret_cast<uint32_t *>(fs + P.lay.syn_off) + buf * P.L;
    }
    __device__ __forceinline__ uint8_t *ia(int buf, int q) const {
        return fs + P.lay.ia_off + (buf * P.L + q) * P.lay.idx_stride;
    }
    __device__ __forceinline__ uint8_t *ib(int buf, int q) const {
        return fs + P.lay.ib_off + (buf * P.L + q) * P.lay.idx_stride;
    }
    __device__ __forceinline__ double *cd(int q) const {
        return reinterpret_cast<double *>(fs + P.lay.cd_off) + q * kMaxCand;
    }
    __device__ __forceinline__ uint16_t *clrb(int q) const {
        return reinterpret_cast<uint16_t *>(fs + P.lay.clrb_off) + q * 4;
    }
    __device__ __forceinline__ uint32_t *chs() const { return reinterpret_cast<uint32_t *>(fs + P.lay.chs_off); }
    __device__ __forceinline__ uint8_t *cflag() const { return fs + P.lay.cflag_off; }
    __device__ __forceinline__ uint8_t *asg() const { return fs + P.lay.asg_off; }
    __device__ __forceinline__ uint32_t *hard(int q) const {
        return reinterpret_cast<uint32_t *>(fs + P.lay.hard_off) + q * P.lay.hard_words;
    }
    __device__ __forceinline__ uint32_t *root() const { return reinterpret_cast<uint32_t *>(fs + P.lay.root_off); }

    // LLRs of path q at stage s
    __device__ __forceinline__ Src<T> src(int s, int q, int vmode) const {
        Src<T> r;
        r.ch = channel();
        r.half = P.N >> 1;
        r.bw = nullptr;
        if (s == P.n) {
            r.mode = VM_NONE;
            r.p = channel();
        } else if (s == P.n - 1) {
            r.mode = vmode;
            r.p = nullptr;
            if (vmode == VM_G) r.bw = beta_row(P.n - 1, ib(cur, q)[P.n - 1]);
        } else {
            r.mode = VM_NONE;
            r.p = alpha_row(s, ia(cur, q)[s]);
        }
        return r;
    }
};

// ---------------------------------------------------------------- F / G

template <typename T, bool IS_G>
__device__ void fg_op(Frame<T> &F, const DOp &o, int lane) {
    const int s = o.stage, h = 1 << (s - 1), np = o.pin;
    const int G = 32 / pow2ceil(np);
    const int q = lane / G, sub = lane & (G - 1);
    if (q < np) {
        Src<T> src = F.src(s, q, o.vmode);
        T *dst = F.alpha_row(s - 1, q);
        if (IS_G) {
            const uint32_t *bw = F.beta_row(s - 1, F.ib(F.cur, q)[s - 1]);
            for (int i = sub; i < h; i += G) {
                unsigned bit = (bw[i >> 5] >> (i & 31)) & 1u;
                Elem<T>::st(dst + i, g_op<T>(src.get(i), src.get(i + h), bit));
            }
        } else {
            for (int i = sub; i < h; i += G) Elem<T>::st(dst + i, f_op(src.get(i), src.get(i + h)));
        }
        if (sub == 0) F.ia(F.cur, q)[s - 1] = (uint8_t)q;
    }
}

// ------------------------------------------------- pairwise-exact sums
// numpy float32 pairwise summation (what the reference's sum(axis=1) runs):
// n < 8 sequential from 0; 8 <= n <= 128 eight strided accumulators combined
// ((0+1)+(2+3))+((4+5)+(6+7)); larger n halves recursively.  For the power-
// of-two node sizes that is a perfect binary tree over 8*nb accumulators
// (nb = max(1, n/128)), each a sequential sum of 16 (or n/8) elements.
// Lane j of an 8-lane group owns accumulator column j of every 128-block.

template <typename T, int NS>
struct SumOut {
    float v[NS];
};

// NS sums of functions of a: NS=1 -> sum(min(a,0)); NS=3 -> (sum min(a,0),
// sum max(a,0), sum a)
template <typename T, int NS>
__device__ __forceinline__ void acc_add(float (&acc)[NS], float a) {
    acc[0] = __fadd_rn(acc[0], fminf(a, 0.f));
    if (NS == 3) {
        acc[1] = __fadd_rn(acc[1], fmaxf(a, 0.f));
        acc[2] = __fadd_rn(acc[2], a);
    }
}
template <int NS>
__device__ __forceinline__ void acc_init(float (&acc)[NS], float a) {
    acc[0] = fminf(a, 0.f);
    if (NS == 3) {
        acc[1] = fmaxf(a, 0.f);
        acc[2] = a;
    }
}

// returns the sums in every lane of the 8-lane group (valid when the group's
// path is active)
template <typename T, int NS>
__device__ void group8_pairwise(const Src<T> &src, int m, bool active, int j, float (&out)[NS]) {
    if (m < 8) {
        float r[NS];
#pragma unroll
        for (int t = 0; t < NS; ++t) r[t] = 0.f;
        if (active && j == 0)
            for (int i = 0; i < m; ++i) acc_add<T, NS>(r, src.get(i));
        // broadcast from lane j==0 of the group
#pragma unroll
        for (int t = 0; t < NS; ++t) out[t] = __shfl_sync(FULL_MASK, r[t], (threadIdx.x & 31) & ~7);
        return;
    }
    const int blk = m < 128 ? m : 128;
    const int nb = m / blk;
    const int per = blk / 8;
    float stk[NS][8];  // binary-counter stack over blocks (nb <= 128 -> depth <= 7)
    float carry[NS];
    for (int b = 0; b < nb; ++b) {
        float acc[NS];
        const int base = b * blk + j;
        if (active) {
            acc_init<NS>(acc, src.get(base));
            for (int r = 1; r < per; ++r) acc_add<T, NS>(acc, src.get(base + 8 * r));
        } else {
#pragma unroll
            for (int t = 0; t < NS; ++t) acc[t] = 0.f;
        }
        // ((0+1)+(2+3))+((4+5)+(6+7)) within the block: xor 1, 2, 4
#pragma unroll
        for (int d = 1; d < 8; d <<= 1)
#pragma unroll
            for (int t = 0; t < NS; ++t) acc[t] = __fadd_rn(acc[t], __shfl_xor_sync(FULL_MASK, acc[t], d));
        // combine block sums as a binary tree in block order
#pragma unroll
        for (int t = 0; t < NS; ++t) carry[t] = acc[t];
        int lvl = 0;
        while ((b >> lvl) & 1) {
#pragma unroll
            for (int t = 0; t < NS; ++t) carry[t] = __fadd_rn(stk[t][lvl], carry[t]);
            ++lvl;
        }
#pragma unroll
        for (int t = 0; t < NS; ++t) stk[t][lvl] = carry[t];
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) out[t] = carry[t];
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
    // insert keeping ascending (magnitude, index): stable argsort order
    __device__ __forceinline__ void push(float v, int idx) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            bool lt = v < m[k] || (v == m[k] && idx < i[k]);
            float tm = m[k];
            int ti = i[k];
            if (lt) {
                m[k] = v;
                i[k] = idx;
                v = tm;
                idx = ti;
            }
        }
    }
};

// ------------------------------------------------------------ selection

__device__ __forceinline__ bool better(double am, int as, double bm, int bs) {
    return am > bm || (am == bm && as < bs);
}

// bitonic network over the first W lanes; desc = best first
__device__ __forceinline__ void bitonic_sort(double &m, int &s, int W, bool desc, int lane) {
    for (int k = 2; k <= W; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            double om = __shfl_xor_sync(FULL_MASK, m, j);
            int os = __shfl_xor_sync(FULL_MASK, s, j);
            bool seg_desc = ((lane & k) == 0) == desc;
            bool want_better = ((lane & j) == 0) == seg_desc;
            if (want_better == better(om, os, m, s)) {
                m = om;
                s = os;
            }
        }
}
__device__ __forceinline__ void bitonic_merge_desc(double &m, int &s, int W, int lane) {
    for (int j = W >> 1; j > 0; j >>= 1) {
        double om = __shfl_xor_sync(FULL_MASK, m, j);
        int os = __shfl_xor_sync(FULL_MASK, s, j);
        bool want_better = (lane & j) == 0;
        if (want_better == better(om, os, m, s)) {
            m = om;
            s = os;
        }
    }
}

// SPC flip sets relative to the ML word over the four LRB slots, emission
// order of listdec.py:157 (_SPC_PAIRS)
__device__ __constant__ uint8_t kSpcPairs[7] = {0x3, 0x5, 0x9, 0x6, 0xA, 0xC, 0xF};

__device__ __forceinline__ int flip_mask(int kind, int c, int odd) {
    if (kind == DK_R1) return c;  // (), (b1), (b2), (b1, b2)
    int ml = odd ? 1 : 0;
    return c == 0 ? ml : (kSpcPairs[c - 1] ^ ml);
}

// Phase B: choose survivors; writes asg[k] = (source, cand) for k < pout.
template <typename T>
__device__ void select_survivors(Frame<T> &F, const DOp &o, int lane) {
    const int np = o.pin, C = o.ncand, L = F.P.L;
    const bool valid_lane = lane < np;
    double met[kMaxCand];
    int seq[kMaxCand];
    const double pm = valid_lane ? F.pm(F.cur)[lane] : 0.0;
    const double *cd = F.cd(valid_lane ? lane : 0);
#pragma unroll
    for (int c = 0; c < kMaxCand; ++c) {
        bool v = valid_lane && c < C;
        met[c] = v ? pm + cd[c] : -INFINITY;
        seq[c] = v ? lane * kMaxCand + c : 0x7fff0000 + lane * kMaxCand + c;
    }
    unsigned mask;
    if (!o.select) {
        mask = valid_lane ? (1u << C) - 1 : 0u;
    } else {
        // sort this lane's column best-first (stable by cand index)
        if (C == 2 || C == 8) {
            // odd-even transposition sort, C passes (C <= 8)
#pragma unroll
            for (int pass = 0; pass < kMaxCand; ++pass) {
                if (pass >= C) break;
#pragma unroll
                for (int c = pass & 1; c + 1 < kMaxCand; c += 2) {
                    if (c + 1 < C && better(met[c + 1], seq[c + 1], met[c], seq[c])) {
                        double tm = met[c];
                        met[c] = met[c + 1];
                        met[c + 1] = tm;
                        int ts = seq[c];
                        seq[c] = seq[c + 1];
                        seq[c + 1] = ts;
                    }
                }
            }
        }
        // Rate-1 columns are already best-first: 0 >= -m1 >= -m2 >= -(m1+m2)
        const int W = pow2ceil(L);
        double Rm = met[0];
        int Rs = seq[0];
        bitonic_sort(Rm, Rs, W, true, lane);
        double Tm = __shfl_sync(FULL_MASK, Rm, L - 1);
        int Ts = __shfl_sync(FULL_MASK, Rs, L - 1);
#pragma unroll
        for (int j = 1; j < kMaxCand; ++j) {
            if (j >= C) break;
            double xm = met[j];
            int xs = seq[j];
            if (!__any_sync(FULL_MASK, better(xm, xs, Tm, Ts))) break;
            bitonic_sort(xm, xs, W, false, lane);
            if (better(xm, xs, Rm, Rs)) {
                Rm = xm;
                Rs = xs;
            }
            bitonic_merge_desc(Rm, Rs, W, lane);
            Tm = __shfl_sync(FULL_MASK, Rm, L - 1);
            Ts = __shfl_sync(FULL_MASK, Rs, L - 1);
        }
        mask = 0u;
#pragma unroll
        for (int c = 0; c < kMaxCand; ++c) {
            bool keep = valid_lane && c < C && (better(met[c], seq[c], Tm, Ts) || seq[c] == Ts);
            if (keep) mask |= 1u << (seq[c] & (kMaxCand - 1));
        }
    }
    // survivors in (source, cand) order
    int cnt = __popc(mask);
    int incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int v = __shfl_up_sync(FULL_MASK, incl, d);
        if (lane >= d) incl += v;
    }
    int k = incl - cnt;
    uint8_t *asg = F.asg();
    while (mask) {
        int c = __ffs(mask) - 1;
        mask &= mask - 1;
        asg[2 * k] = (uint8_t)lane;
        asg[2 * k + 1] = (uint8_t)c;
        ++k;
    }
}

// ----------------------------------------------------- leaf word + chain

// Word bits of the leaf decision for (source p, cand c): value of the 32-bit
// word w of an m-bit leaf word (m < 32: the m-bit value).
template <typename T>
__device__ __forceinline__ uint32_t leaf_word(const Frame<T> &F, int kind, int m, int p, int c, int w) {
    const uint32_t fullw = m >= 32 ? 0xffffffffu : ((1u << m) - 1u);
    if (kind == DK_R0) return 0u;
    if (kind == DK_REP) {
        bool ones = F.cflag()[p] ? (c == 0) : (c == 1);
        return ones ? fullw : 0u;
    }
    uint32_t v = F.hard(p)[w];
    int fm = flip_mask(kind, c, F.cflag()[p]);
    const uint16_t *lrb = F.clrb(p);
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if ((fm >> j) & 1) {
            int pos = lrb[j];
            if ((pos >> 5) == w) v ^= 1u << (pos & 31);
        }
    return v;
}

__device__ __forceinline__ uint32_t bits_get(const uint32_t *row, int off, int len) {
    uint32_t msk = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    return (row[off >> 5] >> (off & 31)) & msk;
}
__device__ __forceinline__ void bits_put(uint32_t *row, int off, int len, uint32_t v) {
    uint32_t msk = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    uint32_t &w = row[off >> 5];
    w = (w & ~(msk << (off & 31))) | ((v & msk) << (off & 31));
}

// Writes the leaf word of path k (decision (p, c) of leaf o) into dst at
// [E - m, E), then runs the leaf's combine chain t .. E's stage - 1:
//   dst[E - 2^(s+1), E - 2^s) = slot_s[row] ^ dst[E - 2^s, E)
// (listdec.py:327-332 with the right child's bits kept in place).
// All 32 lanes must call it (it synchronises the warp between steps).
template <typename T>
__device__ void word_and_chain(const Frame<T> &F, const DOp &o, int kind, bool active, int G, int sub,
                               int p, int c, const uint8_t *ibsrc, uint32_t *dst, int sE) {
    const int t = o.stage, m = 1 << t, E = 1 << sE;
    if (active) {
        if (m >= 32) {
            for (int w = sub; w < (m >> 5); w += G) dst[((E - m) >> 5) + w] = leaf_word(F, kind, m, p, c, w);
        } else if (sub == 0) {
            bits_put(dst, E - m, m, leaf_word(F, kind, m, p, c, 0));
        }
    }
    __syncwarp();
    for (int s = t; s < sE; ++s) {
        const int seg = 1 << s;
        if (active) {
            const uint32_t *sl = F.beta_row(s, ibsrc[s]);
            if (seg >= 32) {
                const int a = (E - 2 * seg) >> 5, b = (E - seg) >> 5;
                for (int w = sub; w < (seg >> 5); w += G) dst[a + w] = sl[w] ^ dst[b + w];
            } else if (sub == 0) {
                uint32_t v = (sl[0] & ((1u << seg) - 1u)) ^ bits_get(dst, E - seg, seg);
                bits_put(dst, E - 2 * seg, seg, v);
            }
        }
        __syncwarp();
    }
}

// ------------------------------------------------------------- leaves

template <typename T>
__device__ void leaf_op(Frame<T> &F, const DOp &o, int lane) {
    const Params &P = F.P;
    const int t = o.stage, m = 1 << t, np = o.pin;
    int kind = o.kind;
    if (kind == DK_R1 && m == 1) kind = DK_REP;  // listdec.py:347

    if (kind == DK_R0 || kind == DK_REP) {
        // 8 lanes per path, 4 paths per pass
        const int g8 = lane >> 3, j = lane & 7;
        for (int base = 0; base < np; base += 4) {
            const int q = base + g8;
            const bool active = q < np;
            Src<T> src = F.src(t, active ? q : 0, o.vmode);
            if (kind == DK_R0) {
                float r[1];
                group8_pairwise<T, 1>(src, m, active, j, r);
                if (active && j == 0) F.pm(F.cur)[q] += (double)r[0];  // listdec.py:341-343
            } else {
                float r[3];
                group8_pairwise<T, 3>(src, m, active, j, r);
                if (active && j == 0) {  // listdec.py:348-358
                    const bool ones_first = r[2] < 0.f;
                    double *cd = F.cd(q);
                    const double neg = (double)r[0], pos = (double)r[1];
                    cd[0] = ones_first ? -pos : neg;
                    cd[1] = ones_first ? neg : -pos;
                    F.cflag()[q] = ones_first;
                }
            }
        }
    } else {
        // Rate-1 / SPC scan: G lanes per path
        const int G = 32 / pow2ceil(np);
        const int q = lane / G, sub = lane & (G - 1);
        const bool active = q < np;
        Src<T> src = F.src(t, active ? q : 0, o.vmode);
        TopK<4> tk;
        tk.init();
        uint32_t hs = 0u, hword = 0u;
        int par = 0;
        const int iters = (m + G - 1) / G;
        uint32_t *hard = F.hard(active ? q : 0);
        for (int it = 0; it < iters; ++it) {
            const int i = it * G + sub;
            const bool valid = active && i < m;
            const float a = valid ? src.get(i) : 0.f;
            const bool neg = valid && a < 0.f;
            if (valid) {
                tk.push(fabsf(a), i);
                if (neg) hs ^= __ldg(P.msyn + o.off + i);
            }
            const uint32_t bal = __ballot_sync(FULL_MASK, neg);
            const uint32_t gb = G == 32 ? bal : (bal >> (q * G)) & ((1u << G) - 1u);
            const int base = it * G;
            hword |= gb << (base & 31);
            if (((base + G) & 31) == 0 || it == iters - 1) {
                if (active && sub == 0) hard[base >> 5] = hword;
                par ^= __popc(hword);
                hword = 0u;
            }
        }
        // merge across the group's lanes
        for (int d = 1; d < G; d <<= 1) {
            hs ^= __shfl_xor_sync(FULL_MASK, hs, d);
            float om[4];
            int oi[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                om[k] = __shfl_xor_sync(FULL_MASK, tk.m[k], d);
                oi[k] = __shfl_xor_sync(FULL_MASK, tk.i[k], d);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) tk.push(om[k], oi[k]);
        }
        if (active && sub == 0) {
            double *cd = F.cd(q);
            uint16_t *lrb = F.clrb(q);
#pragma unroll
            for (int k = 0; k < 4; ++k) lrb[k] = (uint16_t)(tk.i[k] < m ? tk.i[k] : 0);
            F.chs()[q] = hs;
            if (kind == DK_R1) {  // listdec.py:360-372
                const double w1 = (double)tk.m[0], w2 = (double)tk.m[1];
                cd[0] = 0.0;
                cd[1] = -w1;
                cd[2] = -w2;
                cd[3] = -(w1 + w2);
                F.cflag()[q] = 0;
            } else {  // SPC, listdec.py:373-394
                const int odd = par & 1;
                F.cflag()[q] = (uint8_t)odd;
                // slots in ascending position order (the order the reference sums in)
                int ord[4] = {0, 1, 2, 3};
#pragma unroll
                for (int x = 1; x < 4; ++x)
#pragma unroll
                    for (int y = x; y > 0; --y)
                        if (tk.i[ord[y]] < tk.i[ord[y - 1]]) {
                            int tt = ord[y];
                            ord[y] = ord[y - 1];
                            ord[y - 1] = tt;
                        }
                double w[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = (double)tk.m[k];
                for (int c = 0; c < o.ncand; ++c) {
                    const int fm = flip_mask(DK_SPC, c, odd);
                    double accd = 0.0;
                    bool any = false;
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                        if ((fm >> ord[x]) & 1) {
                            accd = any ? accd + w[ord[x]] : w[ord[x]];
                            any = true;
                        }
                    cd[c] = any ? -accd : 0.0;
                }
            }
        }
    }
    __syncwarp();

    const bool fork = kind != DK_R0;
    if (fork) {
        select_survivors(F, o, lane);
        __syncwarp();
    }

    // Phase C: materialise survivors k < pout
    const int npo = o.pout;
    const int G = 32 / pow2ceil(npo);
    const int k = lane / G, sub = lane & (G - 1);
    const bool active = k < npo;
    const int nxt = fork ? F.cur ^ 1 : F.cur;
    int p = k, c = 0;
    if (fork && active) {
        p = F.asg()[2 * k];
        c = F.asg()[2 * k + 1];
    }
    const uint8_t *ibsrc = F.ib(F.cur, active ? p : 0);
    if (active && sub == 0 && fork) {
        uint32_t sy = F.syn(F.cur)[p];
        if (kind == DK_REP) {
            bool ones = F.cflag()[p] ? (c == 0) : (c == 1);
            if (ones) sy ^= o.rep_syn;
        } else {
            sy ^= F.chs()[p];
            const int fm = flip_mask(kind, c, F.cflag()[p]);
            const uint16_t *lrb = F.clrb(p);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((fm >> j) & 1) sy ^= __ldg(P.msyn + o.off + lrb[j]);
        }
        F.syn(nxt)[k] = sy;
        F.pm(nxt)[k] = F.pm(F.cur)[p] + F.cd(p)[c];  // listdec.py:415
        const uint4 *sa = reinterpret_cast<const uint4 *>(F.ia(F.cur, p));
        const uint4 *sb = reinterpret_cast<const uint4 *>(F.ib(F.cur, p));
        uint4 *da = reinterpret_cast<uint4 *>(F.ia(nxt, k));
        uint4 *db = reinterpret_cast<uint4 *>(F.ib(nxt, k));
        for (int x = 0; x < (P.lay.idx_stride >> 4); ++x) {
            da[x] = sa[x];
            db[x] = sb[x];
        }
    }
    const int sE = o.target;
    if (sE < P.n) {
        word_and_chain(F, o, kind, active, G, sub, p, c, ibsrc, F.beta_row(sE, k), sE);
        if (active && sub == 0) F.ib(nxt, k)[sE] = (uint8_t)k;
    }
    __syncwarp();
    F.cur = nxt;
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

template <typename T>
__device__ void build_root(const Frame<T> &F, const DOp &fo, int k, uint32_t *dst, int lane) {
    int kind = fo.kind;
    if (kind == DK_R1 && fo.stage == 0) kind = DK_REP;
    int p = k, c = 0;
    if (kind != DK_R0) {
        p = F.asg()[2 * k];
        c = F.asg()[2 * k + 1];
    }
    // zero the word if it is partial (N < 32)
    if (F.P.N < 32 && lane == 0) dst[0] = 0u;
    __syncwarp();
    word_and_chain(F, fo, kind, true, 32, lane, p, c, F.ib(F.cur, k), dst, F.P.n);
}

template <typename T>
__device__ void finalize(Frame<T> &F, long long f, int np, int lane) {
    const Params &P = F.P;
    const DOp fo = P.prog[P.final_op];
    const bool live = lane < np;
    const double pmk = live ? F.pm(F.cur)[lane] : -INFINITY;
    const bool ok = live && P.has_crc && F.syn(F.cur)[lane] == P.crc_const;
    const bool anyok = __any_sync(FULL_MASK, ok);
    const bool elig = live && (!anyok || ok);
    // listdec.py:297-301: strictly greater metric wins, earliest on ties
    double bm = elig ? pmk : -INFINITY;
    int bk = elig ? lane : 64;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        double om = __shfl_xor_sync(FULL_MASK, bm, d);
        int ok2 = __shfl_xor_sync(FULL_MASK, bk, d);
        if (om > bm || (om == bm && ok2 < bk)) {
            bm = om;
            bk = ok2;
        }
    }
    const int wnr = bk;
    const bool wok = __shfl_sync(FULL_MASK, ok, wnr & 31);
    const int rw = P.lay.root_words;
    if (P.path_cw) {
        for (int kk = 0; kk < np; ++kk) {
            uint32_t *dst = P.path_cw + ((size_t)f * P.L + kk) * rw;
            build_root(F, fo, kk, dst, lane);
        }
        if (live) {
            P.path_pm[(size_t)f * P.L + lane] = pmk;
            P.path_crc[(size_t)f * P.L + lane] = ok;
        }
    }
    if (P.info_out) {
        uint32_t *u = F.root();
        build_root(F, fo, wnr, u, lane);
        polar_transform_words(u, P.N, lane);
        uint8_t *out = P.info_out + (size_t)f * P.k;
        for (int i = lane; i < P.k; i += 32) {
            const uint32_t pos = __ldg(P.info_pos + i);
            out[i] = (uint8_t)((u[pos >> 5] >> (pos & 31)) & 1u);
        }
    }
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[f] = wok;
        if (P.pm_out) P.pm_out[f] = bm;
        if (P.paths_used) P.paths_used[f] = np;
    }
    __syncwarp();
}

// ------------------------------------------------------------- kernel

template <typename T>
__device__ void load_channel(const Frame<T> &F, long long f, int lane) {
    const Params &P = F.P;
    T *ch = F.channel();
    const int N = P.N;
    if (P.in_type == PB_IN_I8) {
        const int8_t *src = reinterpret_cast<const int8_t *>(P.llr) + (size_t)f * N;
        for (int i = lane; i < N; i += 32) ch[i] = (T)src[i];
        return;
    }
    const float *src = reinterpret_cast<const float *>(P.llr) + (size_t)f * N;
    if ((N & 3) == 0) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        for (int i = lane; i < (N >> 2); i += 32) {
            float4 v = __ldcs(s4 + i);  // streamed once: evict-first
            float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                float a = e[x];
                if (Elem<T>::kInt)  // clip(rint(4x), -127, 127), half to even
                    a = fminf(fmaxf(rintf(a * 4.f), -127.f), 127.f);
                else  // clamp_llr: +-2^20 (kernels.py:34-36)
                    a = fminf(fmaxf(a, -1048576.f), 1048576.f);
                Elem<T>::st(ch + 4 * i + x, a);
            }
        }
    } else {
        for (int i = lane; i < N; i += 32) {
            float a = src[i];
            if (Elem<T>::kInt)
                a = fminf(fmaxf(rintf(a * 4.f), -127.f), 127.f);
            else
                a = fminf(fmaxf(a, -1048576.f), 1048576.f);
            Elem<T>::st(ch + i, a);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(32) k_decode(const Params P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    unsigned char *gs = P.gscratch ? P.gscratch + (size_t)blockIdx.x * P.lay.gbytes : nullptr;
    for (long long f = blockIdx.x; f < P.batch; f += gridDim.x) {
        Frame<T> F(P, smem, gs);
        load_channel(F, f, lane);
        if (lane == 0) {
            F.pm(0)[0] = 0.0;
            F.syn(0)[0] = 0u;
        }
        __syncwarp();
        int np = 1;
        for (int oi = 0; oi < P.n_ops; ++oi) {
            const DOp o = P.prog[oi];
            switch (o.kind) {
                case DK_F:
                    fg_op<T, false>(F, o, lane);
                    break;
                case DK_G:
                    fg_op<T, true>(F, o, lane);
                    break;
                case DK_NOP:
                    break;
                default:
                    leaf_op(F, o, lane);
                    np = o.pout;
                    break;
            }
            __syncwarp();
        }
        finalize(F, f, np, lane);
    }
}

}  // namespace pb

// launch wrappers (host)
extern "C" cudaError_t pb_launch_decode(const pb::Params *p, int mode, int grid, size_t smem,
                                        cudaStream_t stream) {
    if (mode == 0) {
        cudaFuncSetAttribute(pb::k_decode<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        pb::k_decode<float><<<grid, 32, smem, stream>>>(*p);
    } else {
        cudaFuncSetAttribute(pb::k_decode<int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        pb::k_decode<int8_t><<<grid, 32, smem, stream>>>(*p);
    }
    return cudaGetLastError();
}

extern "C" cudaError_t pb_occupancy(int mode, size_t smem, int *blocks_per_sm) {
    if (mode == 0) {
        cudaFuncSetAttribute(pb::k_decode<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, pb::k_decode<float>, 32, smem);
    }
    cudaFuncSetAttribute(pb::k_decode<int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, pb::k_decode<int8_t>, 32, smem);
}

// ssc_kernel.cu -- single-path (L = 1) Fast-SSC pass for sm_100a.
//
// polaris.fastssc.execute_schedule (fastssc.py:20-83) batched over frames,
// and the first stage of AdaptiveDecoder (listdec.py:437-459): decode every
// frame with one path, check its CRC, and hand the failing frames to the list
// kernel through a device-side index list (no host round trip).
//
// One warp per frame, lanes over the elements of each op (the list kernel
// spreads paths over lanes instead; with one path the elements are the only
// parallelism).  Per frame in shared memory: the channel, one alpha row per
// stage 0..n-2 (stage n-1 is recomputed from the channel halves, as in the
// list kernel), one beta word row per slot, the codeword.  Many independent
// frame warps per SM hide the latency of each op's short dependent chain.
//
// Leaf decisions (both semantics agree except for one rounding corner):
//   Rate-0  zeros, pm += pairwise sum of min(a, 0)               fastssc.py:70-72
//   Rate-1  hard decisions                                         73-74
//   Rep     SSC_FAST: ones iff the pairwise sum of a is < 0,
//           pm += ones ? -sum max(a,0) : sum min(a,0)              75-80
//           SSC_LIST_L1: the better of the two list candidates by
//           float64 metric, ties to the first (listdec.py:347-359, 63-100),
//           which is what ListDecoder(schedule, 1) returns
//   SPC     hard decisions, Wagner flip of the first least reliable
//           position if the parity is odd, pm -= its magnitude     81-88
//           (the ML candidate of listdec.py:373-394 at L = 1)
#include "decode_kernel.cuh"

namespace pb {
namespace ssc {

template <typename T>
struct Lin {  // a stored alpha row
    const T *p;
    __device__ __forceinline__ float get(int i) const { return Elem<T>::ld(p + i); }
};

// numpy float32 pairwise summation of one node (n < 8
// sequential; n <= 128 eight strided accumulators, ((0+1)+(2+3))+((4+5)+(6+7));
// above, halving -- a perfect binary tree over 128-element blocks for the
// power-of-two node sizes).  Lanes = (block group g, column c): lane 8g + c
// owns column c of the blocks of group g.  Result broadcast to all lanes.
// NS = 1: sum min(a,0); NS = 3: (sum min(a,0), sum max(a,0), sum a).
template <int NS, class S>
__device__ __forceinline__ void pw_sums32(const S &src, int m, int lane, float (&out)[NS]) {
    float r[NS];
#pragma unroll
    for (int t = 0; t < NS; ++t) r[t] = 0.f;
    if (m < 8) {
        if (lane == 0)
            for (int i = 0; i < m; ++i) acc_add<NS>(r, src.get(i));
    } else {
        const int blk = m < 128 ? m : 128, per = blk >> 3, nb = m / blk;
        const int groups = nb < 4 ? nb : 4, nbg = nb / groups;
        const int g = lane >> 3, c = lane & 7;
        const bool act = g < groups;
        float stk[8][NS];
        for (int j = 0; j < nbg; ++j) {
            float acc[NS];
            const int base = (g * nbg + j) * blk + c;
            if (act) {
                acc_init<NS>(acc, src.get(base));
                for (int q = 1; q < per; ++q) acc_add<NS>(acc, src.get(base + 8 * q));
            } else {
#pragma unroll
                for (int t = 0; t < NS; ++t) acc[t] = 0.f;
            }
#pragma unroll
            for (int d = 1; d < 8; d <<= 1)
#pragma unroll
                for (int t = 0; t < NS; ++t) acc[t] = __fadd_rn(acc[t], __shfl_xor_sync(FULL_MASK, acc[t], d));
            // blocks of this group in tree order (binary counter)
            int lvl = 0;
            while ((j >> lvl) & 1) {
#pragma unroll
                for (int t = 0; t < NS; ++t) acc[t] = __fadd_rn(stk[lvl][t], acc[t]);
                ++lvl;
            }
#pragma unroll
            for (int t = 0; t < NS; ++t) stk[lvl][t] = acc[t];
        }
        int top = 0;
        while ((1 << top) < nbg) ++top;
#pragma unroll
        for (int t = 0; t < NS; ++t) r[t] = stk[top][t];
        for (int d = 8; d < 8 * groups; d <<= 1)
#pragma unroll
            for (int t = 0; t < NS; ++t) r[t] = __fadd_rn(r[t], __shfl_xor_sync(FULL_MASK, r[t], d));
    }
#pragma unroll
    for (int t = 0; t < NS; ++t) out[t] = __shfl_sync(FULL_MASK, r[t], 0);
}

template <typename T>
struct Frame {
    const SscParams &P;
    unsigned char *sm;
    int lane;
    double pm;
    unsigned char *gch;  // this frame slot's global channel, or null
    __device__ __forceinline__ T *ch() const {
        return reinterpret_cast<T *>(gch ? gch : sm + P.lay.ch_off);
    }
    __device__ __forceinline__ T *a(int s) const { return reinterpret_cast<T *>(sm + P.lay.a_off[s]); }
    __device__ __forceinline__ uint32_t *b(int s) const { return reinterpret_cast<uint32_t *>(sm + P.lay.b_off[s]); }
    __device__ __forceinline__ uint32_t *root() const { return reinterpret_cast<uint32_t *>(sm + P.lay.root_off); }
};

// out[i] = F/G(src[i], src[i + h]) for i < h, lanes over i
template <typename T, bool IS_G, class S>
__device__ __forceinline__ void fg(const S &src, T *dst, const uint32_t *bw, int h, int lane) {
    if (h >= 32) {
        for (int c0 = 0; c0 < h; c0 += 128) {
            float a[4], b[4];
            uint32_t bits[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = c0 + 32 * u + lane;
                a[u] = i < h ? src.get(i) : 0.f;
                b[u] = i < h ? src.get(i + h) : 0.f;
                bits[u] = IS_G && i < h ? (bw[i >> 5] >> lane) & 1u : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = c0 + 32 * u + lane;
                if (i < h) Elem<T>::st(dst + i, IS_G ? g_op<T>(a[u], b[u], bits[u]) : f_op(a[u], b[u]));
            }
        }
    } else if (lane < h) {
        const float x = src.get(lane), y = src.get(lane + h);
        Elem<T>::st(dst + lane, IS_G ? g_op<T>(x, y, (bw[0] >> lane) & 1u) : f_op(x, y));
    }
}

// the leaf's chain of Combines t .. sE-1 in place, its word already in
// dst[E - m, E) (listdec.py:327-332 / fastssc.py:66-69 with the right
// child's bits kept where they are)
template <typename T>
__device__ __forceinline__ void chain(const Frame<T> &F, int t, int sE, uint32_t *dst) {
    const int E = 1 << sE, lane = F.lane;
    __syncwarp();
    for (int s = t; s < sE; ++s) {
        const int seg = 1 << s;
        const uint32_t *sl = F.b(s);
        if (seg >= 32) {
            const int a = (E - 2 * seg) >> 5, bb = (E - seg) >> 5;
            for (int w = lane; w < (seg >> 5); w += 32) dst[a + w] = sl[w] ^ dst[bb + w];
        } else if (lane == 0) {
            const uint32_t v = (sl[0] & ((1u << seg) - 1u)) ^ bits_get(dst, E - seg, seg);
            bits_put(dst, E - 2 * seg, seg, v);
        }
        __syncwarp();
    }
}

// a constant leaf word (all zeros / all ones) into dst[E - m, E), then the chain
template <typename T>
__device__ __forceinline__ void store_const_and_chain(const Frame<T> &F, int t, int sE, uint32_t *dst, bool ones) {
    const int m = 1 << t, E = 1 << sE, lane = F.lane;
    if (m >= 32) {
        for (int w = lane; w < (m >> 5); w += 32) dst[((E - m) >> 5) + w] = ones ? 0xffffffffu : 0u;
    } else if (lane == 0) {
        bits_put(dst, E - m, m, ones ? (1u << m) - 1u : 0u);
    }
    chain(F, t, sE, dst);
}

template <typename T, class S>
__device__ __forceinline__ void leaf(Frame<T> &F, const DOp &o, const S &src) {
    const SscParams &P = F.P;
    const int lane = F.lane, t = o.stage, m = 1 << t, sE = o.target;
    int kind = o.kind;
    uint32_t *dst = sE < P.n ? F.b(sE) : F.root();
    if (kind == DK_R0) {
        float r[1];
        pw_sums32<1>(src, m, lane, r);
        F.pm += (double)r[0];
        store_const_and_chain(F, t, sE, dst, false);
        return;
    }
    if (kind == DK_R1 && m == 1 && P.semantics == SSC_LIST_L1) kind = DK_REP;  // listdec.py:347
    if (kind == DK_REP) {
        float r[3];
        pw_sums32<3>(src, m, lane, r);
        const bool ones_first = r[2] < 0.f;
        bool ones = ones_first;
        const double neg = (double)r[0], pos = -(double)r[1];
        if (P.semantics == SSC_LIST_L1) {
            // listdec.py:348-358 candidates in order, the better metric wins,
            // the first on ties (listdec.py:63-100)
            const double m0 = F.pm + (ones_first ? pos : neg), m1 = F.pm + (ones_first ? neg : pos);
            ones = (m1 > m0) ? !ones_first : ones_first;
        }
        F.pm += ones ? pos : neg;
        store_const_and_chain(F, t, sE, dst, ones);
        return;
    }
    // Rate-1 / SPC: hard decisions by ballot; SPC also the parity and the
    // first least reliable position (argmin |a|, lowest index on ties)
    const int E = 1 << sE;
    int par = 0;
    float wm = INFINITY;
    int wi = 0x7fffffff;
    const int nw = m >= 32 ? m >> 5 : 1;
    for (int w = 0; w < nw; ++w) {
        const int i = 32 * w + lane;
        const bool valid = i < m;
        const float a = valid ? src.get(i) : 0.f;
        const uint32_t bits = __ballot_sync(FULL_MASK, valid && a < 0.f);
        par ^= __popc(bits);
        if (valid && fabsf(a) < wm) {
            wm = fabsf(a);
            wi = i;
        }
        if (lane == 0) {
            if (m >= 32)
                dst[((E - m) >> 5) + w] = bits;
            else
                bits_put(dst, E - m, m, bits);
        }
    }
    if (kind == DK_SPC && (par & 1)) {
        const unsigned mb = __reduce_min_sync(FULL_MASK, __float_as_uint(wm));  // |a| >= 0: bit order
        const int widx = (int)__reduce_min_sync(FULL_MASK, __float_as_uint(wm) == mb ? (unsigned)wi : 0x7fffffffu);
        if (lane == 0) dst[(E - m + widx) >> 5] ^= 1u << ((E - m + widx) & 31);
        F.pm -= (double)__uint_as_float(mb);
    }
    chain(F, t, sE, dst);
}

template <typename T>
__device__ __forceinline__ void run_frame(Frame<T> &F, long long f) {
    const SscParams &P = F.P;
    const int lane = F.lane, N = P.N, n = P.n;
    // channel: clamp_llr (kernels.py:34-36) or the int8 quantiser, 128-bit loads
    T *ch = F.ch();
    if (P.in_type == PB_IN_I8) {
        const int8_t *src = reinterpret_cast<const int8_t *>(P.llr) + (size_t)f * N;
        for (int i = lane; i < N; i += 32) ch[i] = (T)src[i];
    } else {
        const float *src = reinterpret_cast<const float *>(P.llr) + (size_t)f * N;
        if ((N & 3) == 0) {
            const float4 *s4 = reinterpret_cast<const float4 *>(src);
            for (int i = lane; i < (N >> 2); i += 32) {
                const float4 v = __ldcs(s4 + i);
                Elem<T>::st(ch + 4 * i + 0, ingest<T>(v.x));
                Elem<T>::st(ch + 4 * i + 1, ingest<T>(v.y));
                Elem<T>::st(ch + 4 * i + 2, ingest<T>(v.z));
                Elem<T>::st(ch + 4 * i + 3, ingest<T>(v.w));
            }
        } else {
            for (int i = lane; i < N; i += 32) Elem<T>::st(ch + i, ingest<T>(src[i]));
        }
    }
    __syncwarp();
    F.pm = 0.0;
    DOp onext = P.prog[0];
    for (int oi = 0; oi < P.n_ops; ++oi) {
        const DOp o = onext;
        if (oi + 1 < P.n_ops) onext = P.prog[oi + 1];
        const int s = o.stage;
        if (o.kind == DK_NOP) continue;
        if (o.kind == DK_F || o.kind == DK_G) {
            const int h = 1 << (s - 1);
            const bool g = o.kind == DK_G;
            const uint32_t *bw = F.b(s - 1);
            T *dst = F.a(s - 1);
            if (s == n - 1) {
                if (o.vmode == VM_F) {
                    const VirtF<T> src{ch, N >> 1};
                    g ? fg<T, true>(src, dst, bw, h, lane) : fg<T, false>(src, dst, bw, h, lane);
                } else {
                    const VirtG<T> src{ch, F.b(n - 1), N >> 1};
                    g ? fg<T, true>(src, dst, bw, h, lane) : fg<T, false>(src, dst, bw, h, lane);
                }
            } else {
                const Lin<T> src{F.a(s)};
                g ? fg<T, true>(src, dst, bw, h, lane) : fg<T, false>(src, dst, bw, h, lane);
            }
        } else if (s == n) {
            leaf(F, o, ChanSrc<T>{ch});
        } else if (s == n - 1) {
            if (o.vmode == VM_F)
                leaf(F, o, VirtF<T>{ch, N >> 1});
            else
                leaf(F, o, VirtG<T>{ch, F.b(n - 1), N >> 1});
        } else {
            leaf(F, o, Lin<T>{F.a(s)});
        }
        __syncwarp();
    }
    // CRC of the codeword (syndrome rows in the codeword domain, as the list
    // kernel's finalize), then the outputs
    uint32_t *x = F.root();
    const int nwd = N >= 32 ? N >> 5 : 1;
    uint32_t syn = 0u;
    for (int w = lane; w < nwd; w += 32) {
        uint32_t v = x[w];
        if (N < 32) v &= (1u << N) - 1u;
        if (P.cw_out) P.cw_out[(size_t)f * nwd + w] = v;
        const uint32_t *tb = P.xsyn4 + (size_t)w * 128;
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) syn ^= __ldg(tb + nb * 16 + ((v >> (4 * nb)) & 15u));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) syn ^= __shfl_xor_sync(FULL_MASK, syn, d);
    const bool ok = P.has_crc && syn == P.crc_const;
    if (P.semantics == SSC_ADAPTIVE && !ok) {  // the list decoder takes this frame
        if (lane == 0) {
            P.fail_idx[atomicAdd(P.fail_count, 1)] = (int32_t)f;
            if (P.invoked) P.invoked[f] = 1;
        }
        __syncwarp();
        return;
    }
    if (P.info_out) {
        __syncwarp();
        polar_transform_words(x, N, lane);
        uint8_t *out = P.info_out + (size_t)f * P.k;
        for (int i = lane; i < P.k; i += 32) {
            const uint32_t pos = __ldg(P.info_pos + i);
            out[i] = (uint8_t)((x[pos >> 5] >> (pos & 31)) & 1u);
        }
    }
    if (lane == 0) {
        if (P.crc_ok) P.crc_ok[f] = ok;
        if (P.pm_out) P.pm_out[f] = F.pm;
        if (P.paths_used) P.paths_used[f] = 1;
        if (P.invoked) P.invoked[f] = 0;
    }
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(PB_SSC_MAXT, 1) k_ssc(const __grid_constant__ SscParams P) {
    const int warp = threadIdx.x >> 5;
    unsigned char *gch = P.gch ? P.gch + ((size_t)blockIdx.x * P.fpc + warp) * P.N * sizeof(T) : nullptr;
    Frame<T> F{P, g_smem + (size_t)warp * P.lay.smem_bytes, (int)(threadIdx.x & 31), 0.0, gch};
    const long long stride = (long long)gridDim.x * P.fpc;
    for (long long f = (long long)blockIdx.x * P.fpc + warp; f < P.batch; f += stride) run_frame(F, f);
}

template <typename T>
cudaError_t launch(const SscParams *p, int grid, cudaStream_t st) {
    const size_t smem = (size_t)p->lay.smem_bytes * p->fpc;
    cudaError_t e = cudaFuncSetAttribute(k_ssc<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_ssc<T><<<grid, 32 * p->fpc, smem, st>>>(*p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t occupancy(int fpc, size_t smem_frame, int *bps) {
    const size_t smem = smem_frame * fpc;
    cudaError_t e = cudaFuncSetAttribute(k_ssc<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k_ssc<T>, 32 * fpc, smem);
}

}  // namespace ssc
}  // namespace pb

extern "C" cudaError_t pb_launch_ssc(const pb::SscParams *p, int mode, int grid, cudaStream_t st) {
    return mode == 0 ? pb::ssc::launch<float>(p, grid, st) : pb::ssc::launch<int8_t>(p, grid, st);
}
extern "C" cudaError_t pb_occupancy_ssc(int mode, int fpc, size_t smem_frame, int *bps) {
    return mode == 0 ? pb::ssc::occupancy<float>(fpc, smem_frame, bps) : pb::ssc::occupancy<int8_t>(fpc, smem_frame, bps);
}

// frame_gen.cu -- on-device frame generation and error counting (SURVEY 8f
// #3 / #2): the input and output sides of the decode path for throughput
// sweeps, so a Monte-Carlo point runs without host traffic.
//
// Per frame (one warp):
//   payload   k uniform bits                         sim.py:173 (rng.integers)
//   CRC       appended in the u domain: c = const ^ XOR of the syndrome
//             rows of the set payload bits -- the affine GF(2) map of
//             codes.py:127-156, the same table the decoders check with
//   encode    u at the info positions (payload, then CRC;  encode.py:56-73),
//             x = u G_N by word butterflies (encode.py:29-53)
//   channel   BPSK 0 -> +1, AWGN sigma = sqrt(1 / (2 R 10^(EbN0/10))),
//             LLR = 2y / sigma^2 clamped to +-2^20          sim.py:79-91
//             (int8 output: clip(rint(4 llr), +-127))
// Randomness: Philox4x32-10 keyed by (seed, frame); every frame owns its
// counter space, so shards / batch splits never change a frame.  It is NOT
// numpy's Philox + Generator.normal stream (that one cannot be reproduced on
// the device bit for bit), so device frames are statistically equivalent to
// the reference harness's frames, not identical: parity runs use host frames
// (channel.generate_frames), throughput sweeps use these.
#include <cuda_runtime.h>
#include <stdint.h>

#include "decoder.cuh"

namespace pb {
namespace gen {


__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
        c[0] = hi1 ^ c[1] ^ k0;
        c[1] = lo1;
        c[2] = hi0 ^ c[3] ^ k1;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// 128 random bits: block `blk` of frame f's stream (stream 0 = payload, 1 = noise)
__device__ __forceinline__ void block(const GenParams &P, long long f, uint32_t stream, uint32_t blk, uint32_t (&o)[4]) {
    o[0] = blk;
    o[1] = stream;
    o[2] = (uint32_t)f;
    o[3] = (uint32_t)((unsigned long long)f >> 32);
    philox(o, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
}

__global__ void __launch_bounds__(256) k_gen(const __grid_constant__ GenParams P) {
    extern __shared__ uint32_t sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = P.N >= 32 ? P.N >> 5 : 1;
    uint32_t *u = sh + warp * nw;
    const long long stride = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + warp; t < P.count; t += stride) {
        const long long f = P.first + t;
        for (int w = lane; w < nw; w += 32) u[w] = 0u;
        __syncwarp();
        // payload words: one Philox block gives four
        uint32_t crc = 0u;
        for (int w = lane; w < P.kw; w += 32) {
            uint32_t o[4];
            block(P, f, 0u, (uint32_t)(w >> 2), o);
            uint32_t v = o[w & 3];
            if (32 * w + 32 > P.k) v &= (1u << (P.k - 32 * w)) - 1u;
            if (P.payload) P.payload[t * P.kw + w] = v;
            for (uint32_t b = v; b; b &= b - 1) {
                const int j = 32 * w + __ffs(b) - 1;
                crc ^= __ldg(P.hu + j);
                const uint32_t pos = __ldg(P.info_pos + j);
                atomicOr(u + (pos >> 5), 1u << (pos & 31));
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) crc ^= __shfl_xor_sync(0xffffffffu, crc, d);
        crc ^= P.crc_const;
        if (lane < P.crc_w && ((crc >> lane) & 1u)) {
            const uint32_t pos = __ldg(P.info_pos + P.k + lane);
            atomicOr(u + (pos >> 5), 1u << (pos & 31));
        }
        __syncwarp();
        // x = u G_N (in place)
        {
            const int hin = P.N < 32 ? P.N : 32;
            const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
            for (int w = lane; w < nw; w += 32) {
                uint32_t v = u[w];
#pragma unroll
                for (int b = 0; b < 5; ++b)
                    if ((1 << b) < hin) v ^= (v >> (1 << b)) & masks[b];
                u[w] = v;
            }
            __syncwarp();
            for (int H = 1; H < nw; H <<= 1) {
                for (int w = lane; w < nw; w += 32)
                    if ((w & H) == 0) u[w] ^= u[w + H];
                __syncwarp();
            }
        }
        // BPSK + AWGN -> LLR, four elements per Philox block (Box-Muller pairs)
        for (int q = lane; q < (P.N + 3) / 4; q += 32) {
            uint32_t o[4];
            block(P, f, 1u, (uint32_t)q, o);
            float z[4];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const float u1 = ((float)o[2 * p] + 0.5f) * 2.3283064365386963e-10f;  // (0, 1)
                const float u2 = (float)o[2 * p + 1] * 2.3283064365386963e-10f;
                const float r = sqrtf(-2.0f * __logf(u1));
                float s, c;
                __sincosf(6.283185307179586f * u2, &s, &c);
                z[2 * p] = r * c;
                z[2 * p + 1] = r * s;
            }
            float l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 4 * q + e;
                const float x = (i < P.N && ((u[i >> 5] >> (i & 31)) & 1u)) ? -1.f : 1.f;
                const float v = (x + P.sigma * z[e]) * P.scale;
                l[e] = fminf(fmaxf(v, -1048576.f), 1048576.f);
            }
            if (P.out_type == 0) {
                float *dst = reinterpret_cast<float *>(P.llr) + t * P.N + 4 * q;
                if ((P.N & 3) == 0) {
                    *reinterpret_cast<float4 *>(dst) = make_float4(l[0], l[1], l[2], l[3]);
                } else {
                    for (int e = 0; e < 4 && 4 * q + e < P.N; ++e) dst[e] = l[e];
                }
            } else {
                int8_t *dst = reinterpret_cast<int8_t *>(P.llr) + t * P.N + 4 * q;
                for (int e = 0; e < 4 && 4 * q + e < P.N; ++e)
                    dst[e] = (int8_t)fminf(fmaxf(rintf(l[e] * 4.f), -127.f), 127.f);
            }
        }
        __syncwarp();
    }
}

// Frame / bit errors of decoded payload bytes [B][k] vs packed payload
// words [B][kw], accumulated per chunk of `chunk` frames into
// counts[chunk][3] = (frames, frame errors, bit errors) -- the counters of
// sim.py:_chunk_counts, so the host applies the reference's stop rule chunk
// by chunk.
__global__ void __launch_bounds__(256) k_count(const uint8_t *info, const uint32_t *payload, long long batch, int k,
                                               int kw, int chunk, unsigned long long *counts) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long f = (long long)blockIdx.x * (blockDim.x >> 5) + warp; f < batch; f += stride) {
        unsigned e = 0;
        for (int i = lane; i < k; i += 32) {
            const uint32_t pb = (payload[f * kw + (i >> 5)] >> (i & 31)) & 1u;
            e += (info[f * k + i] & 1u) != pb;
        }
        e = __reduce_add_sync(0xffffffffu, e);
        if (lane == 0) {
            unsigned long long *c = counts + 3 * (f / chunk);
            atomicAdd(c + 0, 1ull);
            if (e) atomicAdd(c + 1, 1ull);
            atomicAdd(c + 2, (unsigned long long)e);
        }
    }
}

}  // namespace gen
}  // namespace pb

extern "C" cudaError_t pb_launch_gen(const pb::gen::GenParams *p, int sms, cudaStream_t st) {
    const int nw = p->N >= 32 ? p->N >> 5 : 1;
    const size_t smem = (size_t)8 * nw * 4;
    cudaError_t e = cudaFuncSetAttribute(pb::gen::k_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    long long blocks = (p->count + 7) / 8;
    const long long cap = (long long)sms * 8;
    pb::gen::k_gen<<<(int)(blocks < cap ? blocks : cap), 256, smem, st>>>(*p);
    return cudaGetLastError();
}

extern "C" cudaError_t pb_launch_errcount(const uint8_t *info, const uint32_t *payload, long long batch, int k, int kw,
                                       int chunk, unsigned long long *counts, int sms, cudaStream_t st) {
    long long blocks = (batch + 7) / 8;
    const long long cap = (long long)sms * 8;
    pb::gen::k_count<<<(int)(blocks < cap ? blocks : cap), 256, 0, st>>>(info, payload, batch, k, kw, chunk, counts);
    return cudaGetLastError();
}

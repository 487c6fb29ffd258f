// net_layers.cu -- the non-block layers of a LAS-ResNet:
// stem weight packing for the tcgen05 stem (conv_tc.cu, mode STEM), the 3x3
// stride-2 max pool after the stem, and the head (global average pool + fully
// connected classifier).  None of these is on the dynamic block's hot path;
// they are plain CUDA-core kernels sized for the whole batch.
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"

namespace lasnet {

// [64][7][7][8] (OHWI, channels padded to 8) -> [64][7][8][8]: kernel row dy,
// window position p = 0..7 holds tap dx = p - 1 (position 0 is the unused
// input pixel 2*ox - 4 of the 8-pixel window, weight 0).
__global__ void pack_stem_kernel(const __nv_bfloat16 *__restrict__ w, __nv_bfloat16 *__restrict__ wp) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // over 64 * 7 * 8 * 8
    if (i >= 64 * 448) return;
    const int c = i & 7, p = (i >> 3) & 7, dy = (i >> 6) % 7, o = i / 448;
    wp[i] = p == 0 ? __float2bfloat16(0.f) : w[((o * 7 + dy) * 7 + (p - 1)) * 8 + c];
}

cudaError_t launch_pack_stem(const void *w, void *wp, cudaStream_t st) {
    return launch_k(pack_stem_kernel, dim3((64 * 448 + 255) / 256), dim3(256), 0, st,
                    static_cast<const __nv_bfloat16 *>(w), static_cast<__nv_bfloat16 *>(wp));
}

// 3x3 stride-2 max pool, padding 1 (padded positions never win: -inf), NHWC bf16;
// one thread per 8-channel vector of an output pixel.
__global__ void __launch_bounds__(256) maxpool_kernel(const uint4 *__restrict__ x, uint4 *__restrict__ y, int n_img,
                                                      int Ho, int Wo, int vpp) {
    pdl_wait();
    pdl_trigger();
    const int Hi = 2 * Ho, Wi = 2 * Wo;
    const long total = (long)n_img * Ho * Wo * vpp;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % vpp);
        const long p = i / vpp;
        const int ox = (int)(p % Wo);
        const long pr = p / Wo;
        const int oy = (int)(pr % Ho), n = (int)(pr / Ho);
        // all nine loads issued before the maxima (out-of-image taps load nothing and never win)
        uint4 q[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int yy = 2 * oy + t / 3 - 1, xx = 2 * ox + t % 3 - 1;
            const bool ok = yy >= 0 && yy < Hi && xx >= 0 && xx < Wi;
            q[t] = ok ? __ldg(x + (((long)n * Hi + yy) * Wi + xx) * vpp + v) : make_uint4(0xFF80FF80u, 0xFF80FF80u,
                                                                                          0xFF80FF80u, 0xFF80FF80u);
        }
        float m[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) m[e] = -INFINITY;
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const uint32_t u[4] = {q[t].x, q[t].y, q[t].z, q[t].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                m[2 * e] = fmaxf(m[2 * e], __uint_as_float(u[e] << 16));
                m[2 * e + 1] = fmaxf(m[2 * e + 1], __uint_as_float(u[e] & 0xFFFF0000u));
            }
        }
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)  // maxima of bf16 values are bf16 values: the conversion is exact
            o[e] = (__float_as_uint(m[2 * e]) >> 16) | (__float_as_uint(m[2 * e + 1]) & 0xFFFF0000u);
        y[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

cudaError_t launch_maxpool(const void *x, void *y, int n_img, int Ho, int Wo, int c, int num_sms, cudaStream_t st) {
    const long total = (long)n_img * Ho * Wo * (c / 8);
    if (total == 0) return cudaSuccess;
    long grid = (total + 255) / 256;
    if (grid > 32L * num_sms) grid = 32L * num_sms;
    return launch_k(maxpool_kernel, dim3((unsigned)grid), dim3(256), 0, st, static_cast<const uint4 *>(x),
                    static_cast<uint4 *>(y), n_img, Ho, Wo, c / 8);
}

// Head, pass 1: global average pool [n][hw][c] bf16 -> pooled [n][c] fp32
// (fixed-order fp32 sum over the hw pixels, then / hw); a thread owns 8
// consecutive channels (16-B loads, coalesced along the channels).
__global__ void __launch_bounds__(256) avgpool_kernel(const __nv_bfloat16 *__restrict__ x, float *__restrict__ pooled,
                                                      int n_img, int hw, int c) {
    pdl_wait();
    pdl_trigger();
    const int cv = c / 8;
    const long total = (long)n_img * cv;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % cv);
        const long n = i / cv;
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const uint4 *src = reinterpret_cast<const uint4 *>(x + n * hw * c) + v;
#pragma unroll 8
        for (int p = 0; p < hw; ++p) {  // loads hoisted by the unroll; the adds stay in pixel order
            const uint4 q = __ldg(src + (long)p * cv);
            const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                s[2 * e] += __uint_as_float(u[e] << 16);
                s[2 * e + 1] += __uint_as_float(u[e] & 0xffff0000u);
            }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) pooled[n * c + 8 * v + e] = s[e] / (float)hw;
    }
}

// Head, pass 2: logits[n][k] = b[k] + sum_c pooled[n][c] w[k][c] -- a SIMT GEMM tile
// of 32 images x 32 classes per 256-thread CTA: four K slices of 64 threads, each
// thread a 4 x 4 register block over its slice's 64-channel chunks (transposed in
// shared memory so every thread's four images / classes are one 16-B load); the four
// slice partials are then added in slice order (deterministic).  8 warps per CTA keep
// the FMA pipes fed (a 2-warp CTA was latency-bound at ~120 us).
constexpr int kFcT = 32, kFcK = 64, kFcP = 36, kFcS = 4;  // tile, K chunk, padded row, K slices
__global__ void __launch_bounds__(256) fc_kernel(const float *__restrict__ pooled, const __nv_bfloat16 *__restrict__ w,
                                                 const float *__restrict__ b, float *__restrict__ logits, int n_img,
                                                 int c, int classes) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) float fsm[];
    const int slice = threadIdx.x >> 6, lt = threadIdx.x & 63;
    float(*sa)[kFcP] = reinterpret_cast<float(*)[kFcP]>(fsm + slice * 2 * kFcK * kFcP);
    float(*sb)[kFcP] = reinterpret_cast<float(*)[kFcP]>(fsm + slice * 2 * kFcK * kFcP + kFcK * kFcP);
    const int tx = lt & 7, ty = lt >> 3;
    const int k0 = blockIdx.x * kFcT, n0 = blockIdx.y * kFcT;
    float acc[4][4] = {};
    // the next chunk's 8 (pooled, weight) vectors per thread are loaded into registers while the
    // current chunk is multiplied out of shared memory (the loads were a round trip per chunk)
    constexpr int kPer = kFcT * kFcK / 8 / 64;  // 16-B vector pairs per thread per chunk (4)
    float4 pa[kPer][2];
    uint4 pw[kPer];
    auto load = [&](int c0) {
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int e = lt + 64 * t;
            const int r = e / (kFcK / 8), cc = (e % (kFcK / 8)) * 8, ch = c0 + cc;
            const int n = n0 + r, k = k0 + r;
            pa[t][0] = pa[t][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            pw[t] = make_uint4(0u, 0u, 0u, 0u);
            if (c0 < c && n < n_img && ch < c) {
                pa[t][0] = *reinterpret_cast<const float4 *>(pooled + (long)n * c + ch);
                pa[t][1] = *reinterpret_cast<const float4 *>(pooled + (long)n * c + ch + 4);
            }
            if (c0 < c && k < classes && ch < c) pw[t] = __ldg(reinterpret_cast<const uint4 *>(w + (long)k * c + ch));
        }
    };
    load(slice * kFcK);
    for (int c0 = slice * kFcK; c0 < c; c0 += kFcS * kFcK) {
#pragma unroll
        for (int t = 0; t < kPer; ++t) {
            const int e = lt + 64 * t;
            const int r = e / (kFcK / 8), cc = (e % (kFcK / 8)) * 8;
            const float av[8] = {pa[t][0].x, pa[t][0].y, pa[t][0].z, pa[t][0].w,
                                 pa[t][1].x, pa[t][1].y, pa[t][1].z, pa[t][1].w};
            const uint32_t u[4] = {pw[t].x, pw[t].y, pw[t].z, pw[t].w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                sa[cc + q][r] = av[q];
                sb[cc + q][r] = (q & 1) ? __uint_as_float(u[q >> 1] & 0xffff0000u) : __uint_as_float(u[q >> 1] << 16);
            }
        }
        __syncwarp();
        asm volatile("bar.sync %0, 64;" ::"r"(1 + slice));  // this slice's 2 warps
        load(c0 + kFcS * kFcK);  // in flight during this chunk's products
        const int kk_end = min(kFcK, c - c0);
#pragma unroll 4
        for (int kk = 0; kk < kk_end; ++kk) {
            const float4 a4 = *reinterpret_cast<const float4 *>(&sa[kk][ty * 4]);
            const float4 b4 = *reinterpret_cast<const float4 *>(&sb[kk][tx * 4]);
            const float av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + slice));
    }
    // slice partials -> logits, added in slice order
    __syncthreads();
    float *red = fsm;  // [kFcS][32][33]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) red[(slice * 32 + ty * 4 + i) * 33 + tx * 4 + j] = acc[i][j];
    __syncthreads();
    for (int e = threadIdx.x; e < kFcT * kFcT; e += 256) {
        const int r = e / kFcT, col = e % kFcT, n = n0 + r, k = k0 + col;
        if (n < n_img && k < classes) {
            float v = red[r * 33 + col];
            for (int sl = 1; sl < kFcS; ++sl) v += red[(sl * 32 + r) * 33 + col];
            logits[(long)n * classes + k] = v + b[k];
        }
    }
}

cudaError_t launch_head(const void *x, const void *w, const float *b, float *pooled, float *logits, int n_img, int hw,
                        int c, int classes, int num_sms, cudaStream_t st) {
    if (n_img == 0) return cudaSuccess;
    if (c % 8) return cudaErrorInvalidValue;
    long g1 = ((long)n_img * (c / 8) + 255) / 256;
    if (g1 > 8L * num_sms) g1 = 8L * num_sms;
    cudaError_t e = launch_k(avgpool_kernel, dim3((unsigned)g1), dim3(256), 0, st,
                             static_cast<const __nv_bfloat16 *>(x), pooled, n_img, hw, c);
    if (e != cudaSuccess) return e;
    const dim3 g2((unsigned)((classes + kFcT - 1) / kFcT), (unsigned)((n_img + kFcT - 1) / kFcT));
    const int smem = kFcS * 2 * kFcK * kFcP * 4;  // >= the [4][32][33] partials
    static bool configured = false;
    if (!configured) {
        e = cudaFuncSetAttribute(fc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    return launch_k(fc_kernel, g2, dim3(256), smem, st, static_cast<const float *>(pooled),
                    static_cast<const __nv_bfloat16 *>(w), b, logits, n_img, c, classes);
}

}  // namespace lasnet

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

// 3x3 stride-2 max pool, padding 1 (padded positions never win: -inf), NHWC bf16.
// A thread owns one 8-channel vector of a 2 x 2 block of output pixels: the 5 x 5
// input window they share is loaded once (25 loads for 4 outputs instead of 36),
// row by row: each input row's horizontal maxima feed the output rows it belongs to.
__device__ __forceinline__ uint4 max8(uint4 a, uint4 b) {
    uint4 r;
    uint32_t *pa = &a.x, *pb = &b.x, *pr = &r.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const __nv_bfloat162 m = __hmax2(*reinterpret_cast<__nv_bfloat162 *>(pa + e), *reinterpret_cast<__nv_bfloat162 *>(pb + e));
        pr[e] = *reinterpret_cast<const uint32_t *>(&m);
    }
    return r;
}

__global__ void __launch_bounds__(256) maxpool_kernel(const uint4 *x, uint4 *__restrict__ y, int n_img,
                                                      int Ho, int Wo, int vpp) {
    pdl_wait();
    pdl_trigger();
    const int Hi = 2 * Ho, Wi = 2 * Wo;
    const int Hb = (Ho + 1) / 2, Wb = (Wo + 1) / 2;  // 2 x 2 output blocks
    const long total = (long)n_img * Hb * Wb * vpp;
    const uint4 ninf = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % vpp);
        const long p = i / vpp;
        const int bx = (int)(p % Wb);
        const long pr = p / Wb;
        const int by = (int)(pr % Hb), n = (int)(pr / Hb);
        const int oy = 2 * by, ox = 2 * bx;
        uint4 o[2][2] = {{ninf, ninf}, {ninf, ninf}};
#pragma unroll
        for (int dy = 0; dy < 5; ++dy) {  // input row 2 oy - 1 + dy
            const int yy = 2 * oy - 1 + dy;
            uint4 q[5];
#pragma unroll
            for (int dx = 0; dx < 5; ++dx) {
                const int xx = 2 * ox - 1 + dx;
                const bool ok = yy >= 0 && yy < Hi && xx >= 0 && xx < Wi;
                q[dx] = ok ? __ldca(x + (((long)n * Hi + yy) * Wi + xx) * vpp + v) : ninf;  // coherent (PDL)
            }
            const uint4 h0 = max8(max8(q[0], q[1]), q[2]), h1 = max8(max8(q[2], q[3]), q[4]);
            if (dy <= 2) {
                o[0][0] = max8(o[0][0], h0);
                o[0][1] = max8(o[0][1], h1);
            }
            if (dy >= 2) {
                o[1][0] = max8(o[1][0], h0);
                o[1][1] = max8(o[1][1], h1);
            }
        }
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                if (oy + a < Ho && ox + b < Wo) y[(((long)n * Ho + oy + a) * Wo + ox + b) * vpp + v] = o[a][b];
    }
}

cudaError_t launch_maxpool(const void *x, void *y, int n_img, int Ho, int Wo, int c, int num_sms, cudaStream_t st) {
    const long total = (long)n_img * ((Ho + 1) / 2) * ((Wo + 1) / 2) * (c / 8);
    if (total == 0) return cudaSuccess;
    long grid = (total + 255) / 256;
    if (grid > 32L * num_sms) grid = 32L * num_sms;
    return launch_k(maxpool_kernel, dim3((unsigned)grid), dim3(256), 0, st, static_cast<const uint4 *>(x),
                    static_cast<uint4 *>(y), n_img, Ho, Wo, c / 8);
}

// Head, pass 1: global average pool [n][hw][c] bf16 -> pooled [n][c] fp32.  CTA =
// (image, 32 channel vectors of 8 channels); its 8 warps take the pixels p = warp,
// warp + 8, ... (fp32 sums in pixel order), and the 8 partials are added in warp order
// (fixed order), then / hw.  16-B loads coalesced along the channels.
constexpr int kPoolGroups = 8;
__global__ void __launch_bounds__(32 * kPoolGroups) avgpool_kernel(const __nv_bfloat16 *x,
                                                                   float *__restrict__ pooled, int n_img, int hw,
                                                                   int c) {
    pdl_wait();
    pdl_trigger();
    __shared__ float part[kPoolGroups][32][9];
    const int cv = c / 8, lane = threadIdx.x & 31, pg = threadIdx.x >> 5;
    const int vblocks = (cv + 31) / 32;
    const long n = blockIdx.x / vblocks;
    const int v = (blockIdx.x - (int)(n * vblocks)) * 32 + lane;
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (v < cv) {
        const uint4 *src = reinterpret_cast<const uint4 *>(x + n * hw * c) + v;
#pragma unroll 4
        for (int p = pg; p < hw; p += kPoolGroups) {
            const uint4 q = __ldca(src + (long)p * cv);  // coherent: the previous kernel wrote x
            const uint32_t u[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                s[2 * e] += __uint_as_float(u[e] << 16);
                s[2 * e + 1] += __uint_as_float(u[e] & 0xffff0000u);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) part[pg][lane][e] = s[e];
    __syncthreads();
    // thread (lane, e = pg): channel 8 v + e, partials added in group order
    if (v < cv) {
        float t = part[0][lane][pg];
#pragma unroll
        for (int k = 1; k < kPoolGroups; ++k) t += part[k][lane][pg];
        pooled[n * c + 8 * v + pg] = t / (float)hw;
    }
}

// Head, pass 2: logits[n][k] = b[k] + sum_c pooled[n][c] w[k][c] on the tensor cores
// (mma.sync m16n8k16, bf16 x bf16 -> fp32).  The fp32 pooled operand is split into three
// bf16 terms, p = p0 + p1 + p2 (p0 = RNE_bf16(p), p1 = RNE_bf16(p - p0), p2 = RNE_bf16(p - p0 - p1):
// 3 x 8 significand bits cover fp32's 24: exact for |p| >= 2^-110, absolute error < 2^-133 below;
// tests/test_head_split.py), and the bf16 x bf16 products are exact in fp32,
// so the three MMAs over the same bf16 weights see the fp32 operand; only the fp32
// accumulation order differs from a scalar loop.  CTA = 16 images x 32 classes, its four
// warps take four K slices (each warp: 16 x 32 as four n8 blocks), and the slice partials
// are added in slice order (deterministic).  (The SIMT GEMM this replaces took 74 us.)
constexpr int kFcImg = 16, kFcCls = 32, kFcSlices = 4;

__device__ __forceinline__ void split3_bf16x2(float2 v, uint32_t (&o)[3]) {
    float x = v.x, y = v.y;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const __nv_bfloat16 bx = __float2bfloat16_rn(x), by = __float2bfloat16_rn(y);
        o[p] = (uint32_t)__bfloat16_as_ushort(bx) | ((uint32_t)__bfloat16_as_ushort(by) << 16);
        x -= __bfloat162float(bx);
        y -= __bfloat162float(by);
    }
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(32 * kFcSlices) fc_kernel(const float *pooled,
                                                            const __nv_bfloat16 *__restrict__ w,
                                                            const float *__restrict__ b, float *__restrict__ logits,
                                                            int n_img, int c, int classes) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[kFcSlices][kFcImg][kFcCls + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int n0 = blockIdx.y * kFcImg, k0 = blockIdx.x * kFcCls;
    // fragment rows (images) g, g + 8 and columns (classes) g of the four n8 blocks; rows / classes
    // past the end read a valid row (clamped) and are never stored
    const float *pa0 = pooled + (long)min(n0 + g, n_img - 1) * c;
    const float *pa1 = pooled + (long)min(n0 + g + 8, n_img - 1) * c;
    const __nv_bfloat16 *wb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) wb[j] = w + (long)min(k0 + 8 * j + g, classes - 1) * c;
    const int ksl = (c + 16 * kFcSlices - 1) / (16 * kFcSlices) * 16;  // K slice (multiple of 16)
    const int kbeg = warp * ksl, kend = min(c, kbeg + ksl);
    float acc[4][4] = {};
#pragma unroll 4
    for (int kk = kbeg; kk < kend; kk += 16) {
        const int ka = kk + 2 * t, kb = ka + 8;  // (c % 8 == 0: kb < c unless c % 16 == 8 at the tail)
        const float2 z = make_float2(0.f, 0.f);
        // (the pooled features come from the previous kernel: coherent loads, PDL)
        const float2 x00 = __ldcg(reinterpret_cast<const float2 *>(pa0 + ka));
        const float2 x10 = __ldcg(reinterpret_cast<const float2 *>(pa1 + ka));
        const float2 x01 = kb < c ? __ldcg(reinterpret_cast<const float2 *>(pa0 + kb)) : z;
        const float2 x11 = kb < c ? __ldcg(reinterpret_cast<const float2 *>(pa1 + kb)) : z;
        uint32_t bw[4][2];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            bw[j][0] = __ldg(reinterpret_cast<const unsigned *>(wb[j] + ka));
            bw[j][1] = kb < c ? __ldg(reinterpret_cast<const unsigned *>(wb[j] + kb)) : 0u;
        }
        uint32_t s00[3], s10[3], s01[3], s11[3];
        split3_bf16x2(x00, s00);
        split3_bf16x2(x10, s10);
        split3_bf16x2(x01, s01);
        split3_bf16x2(x11, s11);
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const uint32_t a[4] = {s00[p], s10[p], s01[p], s11[p]};
#pragma unroll
            for (int j = 0; j < 4; ++j) mma_bf16_16816(acc[j], a, bw[j][0], bw[j][1]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        red[warp][g][8 * j + 2 * t] = acc[j][0];
        red[warp][g][8 * j + 2 * t + 1] = acc[j][1];
        red[warp][g + 8][8 * j + 2 * t] = acc[j][2];
        red[warp][g + 8][8 * j + 2 * t + 1] = acc[j][3];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kFcImg * kFcCls; e += 32 * kFcSlices) {
        const int r = e / kFcCls, col = e % kFcCls, n = n0 + r, k = k0 + col;
        if (n < n_img && k < classes) {
            float v = red[0][r][col];
#pragma unroll
            for (int sl = 1; sl < kFcSlices; ++sl) v += red[sl][r][col];
            logits[(long)n * classes + k] = v + b[k];
        }
    }
}

cudaError_t launch_head(const void *x, const void *w, const float *b, float *pooled, float *logits, int n_img, int hw,
                        int c, int classes, int num_sms, cudaStream_t st) {
    if (n_img == 0) return cudaSuccess;
    if (c % 8) return cudaErrorInvalidValue;
    (void)num_sms;
    const long g1 = (long)n_img * ((c / 8 + 31) / 32);
    cudaError_t e = launch_k(avgpool_kernel, dim3((unsigned)g1), dim3(32 * kPoolGroups), 0, st,
                             static_cast<const __nv_bfloat16 *>(x), pooled, n_img, hw, c);
    if (e != cudaSuccess) return e;
    const dim3 g2((unsigned)((classes + kFcCls - 1) / kFcCls), (unsigned)((n_img + kFcImg - 1) / kFcImg));
    return launch_k(fc_kernel, g2, dim3(32 * kFcSlices), 0, st, static_cast<const float *>(pooled),
                    static_cast<const __nv_bfloat16 *>(w), b, logits, n_img, c, classes);
}

}  // namespace lasnet

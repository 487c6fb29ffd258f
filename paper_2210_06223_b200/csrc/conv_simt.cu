// conv_simt.cu -- fp32 CUDA-core path of the three convolutions (config 1,
// tolerance 1e-5; TF32 tensor cores would be too coarse).  Same row mapping
// (rowmap.cuh) and the same gather / im2col / scatter-add semantics as the
// tcgen05 path; fp32 FMA accumulation in natural K order.
#include <cstdint>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "rowmap.cuh"

namespace lasnet {

// Latency-oriented tiling for the small batches this path serves (config 1 is
// N = 1): 16 rows x 32 columns per 128-thread CTA (each thread 2 x 2 outputs) so
// even a few hundred GEMM rows spread over ~100 CTAs, and the next 32-wide K chunk
// is loaded into registers while the current one is multiplied out of shared
// memory.  A chunk never straddles a 3x3 tap (a_ld is a multiple of 64), so the
// tap decode happens once per chunk.
constexpr int kSBM = 16, kSBN = 32, kSBK = 32, kSThreads = 128;

template <int MODE>
__device__ __forceinline__ const float *simt_row_ptr(const ConvArgs &a, int src, int aux, int tap, int c0) {
    // pointer to A[row][tap * a_ld + c0] or nullptr for a zero row segment
    const float *A = static_cast<const float *>(a.a_src);
    if (src < 0) return nullptr;
    if (MODE == CONV2_DYN || MODE == CONV2_DENSE) {
        const int dy = tap / 3, dx = tap - dy * 3;
        if (MODE == CONV2_DENSE) {
            const int sy = (aux >> 16) + dy - 1, sx = (aux & 0xFFFF) + dx - 1;
            if (sy < 0 || sy >= a.H || sx < 0 || sx >= a.W) return nullptr;
            return A + (size_t)(src + (dy - 1) * a.W + (dx - 1)) * a.a_ld + c0;
        }
        return A + (size_t)(src + (dy - 1) * a.hs + (dx - 1)) * a.a_ld + c0;
    }
    return A + (size_t)src * a.a_ld + c0;
}

template <int MODE>
__global__ void __launch_bounds__(kSThreads) conv_simt_kernel(const __grid_constant__ ConvArgs a) {
    __shared__ float As[2][kSBK][kSBM + 1];
    __shared__ float Bs[2][kSBK][kSBN + 1];
    __shared__ int src_s[kSBM], aux_s[kSBM], orow_s[kSBM], zero_s[kSBM];
    pdl_wait();  // the previous kernel's outputs (x / h1 / h2, idx, count) are complete from here on
    pdl_trigger();
    const int M = gemm_rows(MODE, a);
    const int m0 = blockIdx.x * kSBM, n0 = blockIdx.y * kSBN;
    if (m0 >= M) return;
    const int tid = threadIdx.x;
    if (tid < kSBM) {
        const int r = m0 + tid;
        int src, aux = 0, orow, zero = 0;
        if (MODE == CONV1_DYN) {
            src = halo_pixel(a, r, M);
            orow = r < M ? r : -1;
            zero = src < 0;
        } else if (MODE == CONV2_DYN) {
            src = conv2_center_row(a, r, M);
            orow = r < M ? r : -1;
        } else if (MODE == CONV3_DYN) {
            src = r < M ? r : -1;
            orow = out_pixel(a, r, M);
        } else {
            src = r < M ? r : -1;
            orow = src;
            if (MODE == CONV2_DENSE) aux = (((r / a.W) % a.H) << 16) | (r % a.W);
        }
        src_s[tid] = src;
        aux_s[tid] = aux;
        orow_s[tid] = orow;
        zero_s[tid] = zero;
    }
    __syncthreads();
    // loader mapping: A chunk 16 x 32 (4 per thread: row ar, k ak..ak+3), B chunk 32 x 32 (8 per thread)
    const int ar = tid >> 3, ak = (tid & 7) * 4;
    const int bn = tid >> 2, bk = (tid & 3) * 8;
    const float *Wt = static_cast<const float *>(a.w);
    const int nk = a.K / kSBK;
    float ra[4], rb[8];
    auto load = [&](int kc) {
        const int k0 = kc * kSBK;
        const int tap = (MODE == CONV2_DYN || MODE == CONV2_DENSE) ? k0 / a.a_ld : 0;
        const int c0 = k0 - tap * a.a_ld;
        const float *p = simt_row_ptr<MODE>(a, src_s[ar], aux_s[ar], tap, c0 + ak);
        if (p) {
            const float4 v = *reinterpret_cast<const float4 *>(p);
            ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
        } else {
            ra[0] = ra[1] = ra[2] = ra[3] = 0.f;
        }
        const float4 *wp = reinterpret_cast<const float4 *>(Wt + (size_t)(n0 + bn) * a.K + k0 + bk);
        const float4 w0 = wp[0], w1 = wp[1];
        rb[0] = w0.x; rb[1] = w0.y; rb[2] = w0.z; rb[3] = w0.w;
        rb[4] = w1.x; rb[5] = w1.y; rb[6] = w1.z; rb[7] = w1.w;
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int e = 0; e < 4; ++e) As[buf][ak + e][ar] = ra[e];
#pragma unroll
        for (int e = 0; e < 8; ++e) Bs[buf][bk + e][bn] = rb[e];
    };
    const int tx = tid & 15, ty = tid >> 4;  // outputs: rows 2ty, 2ty+1; cols 2tx, 2tx+1
    float acc[2][2] = {};
    load(0);
    store(0);
    __syncthreads();
    for (int kc = 0; kc < nk; ++kc) {
        const int buf = kc & 1;
        if (kc + 1 < nk) load(kc + 1);  // in flight while this chunk is multiplied
#pragma unroll 8
        for (int kk = 0; kk < kSBK; ++kk) {
            const float a0 = As[buf][kk][2 * ty], a1 = As[buf][kk][2 * ty + 1];
            const float b0 = Bs[buf][kk][2 * tx], b1 = Bs[buf][kk][2 * tx + 1];
            acc[0][0] = fmaf(a0, b0, acc[0][0]);
            acc[0][1] = fmaf(a0, b1, acc[0][1]);
            acc[1][0] = fmaf(a1, b0, acc[1][0]);
            acc[1][1] = fmaf(a1, b1, acc[1][1]);
        }
        if (kc + 1 < nk) store(buf ^ 1);
        __syncthreads();
    }
    float *O = static_cast<float *>(a.out);
    const float *R = static_cast<const float *>(a.resid);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int rr = 2 * ty + i;
        const int orow = orow_s[rr];
        if (orow < 0) continue;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int col = n0 + 2 * tx + j;
            float v = acc[i][j] + a.bias[col];
            if (MODE == CONV3_DYN || MODE == CONV3_DENSE) v += R[(size_t)orow * a.out_ld + col];
            v = fmaxf(v, 0.f);
            if (zero_s[rr]) v = 0.f;
            O[(size_t)orow * a.out_ld + col] = v;
        }
    }
}

cudaError_t launch_conv_simt(int mode, const ConvArgs &a, int max_rows, cudaStream_t st) {
    if (a.N % kSBN != 0 || a.K % kSBK != 0 || a.a_ld % kSBK != 0) return cudaErrorInvalidValue;
    dim3 grid((max_rows + kSBM - 1) / kSBM, a.N / kSBN);
    if (grid.x == 0) return cudaSuccess;
    switch (mode) {
        case CONV1_DYN: conv_simt_kernel<CONV1_DYN><<<grid, kSThreads, 0, st>>>(a); break;
        case CONV2_DYN: conv_simt_kernel<CONV2_DYN><<<grid, kSThreads, 0, st>>>(a); break;
        case CONV3_DYN: conv_simt_kernel<CONV3_DYN><<<grid, kSThreads, 0, st>>>(a); break;
        case CONV1_DENSE: conv_simt_kernel<CONV1_DENSE><<<grid, kSThreads, 0, st>>>(a); break;
        case CONV2_DENSE: conv_simt_kernel<CONV2_DENSE><<<grid, kSThreads, 0, st>>>(a); break;
        case CONV3_DENSE: conv_simt_kernel<CONV3_DENSE><<<grid, kSThreads, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace lasnet

// conv_simt.cu -- fp32 CUDA-core path of the three convolutions (config 1,
// tolerance 1e-5; TF32 tensor cores would be too coarse).  Same row mapping
// (rowmap.cuh) and the same gather / im2col / scatter-add semantics as the
// tcgen05 path; fp32 FMA accumulation in natural K order.
// Tile: 32 rows x 64 columns per 256-thread CTA, K staged through shared
// memory 32 at a time; each thread owns 2 rows x 4 columns.
#include <cstdint>
#include <cuda_runtime.h>

#include "rowmap.cuh"

namespace lasnet {

constexpr int kSBM = 32, kSBN = 64, kSBK = 32;

template <int MODE>
__device__ __forceinline__ const float *simt_a_ptr(const ConvArgs &a, int src, int aux, int k) {
    // returns pointer to A[row][k] or nullptr for a zero element
    const float *A = static_cast<const float *>(a.a_src);
    if (src < 0) return nullptr;
    if (MODE == CONV2_DYN || MODE == CONV2_DENSE) {
        const int tap = k / a.a_ld, c = k - tap * a.a_ld;
        const int dy = tap / 3, dx = tap - dy * 3;
        if (MODE == CONV2_DENSE) {
            const int sy = (aux >> 16) + dy - 1, sx = (aux & 0xFFFF) + dx - 1;
            if (sy < 0 || sy >= a.H || sx < 0 || sx >= a.W) return nullptr;
            return A + (size_t)(src + (dy - 1) * a.W + (dx - 1)) * a.a_ld + c;
        }
        return A + (size_t)(src + (dy - 1) * (a.S + 2) + (dx - 1)) * a.a_ld + c;
    }
    return A + (size_t)src * a.a_ld + k;
}

template <int MODE>
__global__ void __launch_bounds__(256) conv_simt_kernel(const __grid_constant__ ConvArgs a) {
    __shared__ float As[kSBK][kSBM + 1];
    __shared__ float Bs[kSBK][kSBN + 1];
    __shared__ int src_s[kSBM], aux_s[kSBM], orow_s[kSBM], zero_s[kSBM];
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
    const int tx = tid & 15, ty = tid >> 4;
    float acc[2][4] = {};
    const float *Wt = static_cast<const float *>(a.w);
    for (int k0 = 0; k0 < a.K; k0 += kSBK) {
        for (int i = tid; i < kSBM * kSBK; i += 256) {
            const int rr = i / kSBK, kk = i - rr * kSBK;
            const float *p = simt_a_ptr<MODE>(a, src_s[rr], aux_s[rr], k0 + kk);
            As[kk][rr] = p ? *p : 0.f;
        }
        for (int i = tid; i < kSBN * kSBK; i += 256) {
            const int nn = i / kSBK, kk = i - nn * kSBK;
            Bs[kk][nn] = Wt[(size_t)(n0 + nn) * a.K + k0 + kk];
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < kSBK; ++kk) {
            const float a0 = As[kk][2 * ty], a1 = As[kk][2 * ty + 1];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float b = Bs[kk][4 * tx + j];
                acc[0][j] = fmaf(a0, b, acc[0][j]);
                acc[1][j] = fmaf(a1, b, acc[1][j]);
            }
        }
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
        for (int j = 0; j < 4; ++j) {
            const int col = n0 + 4 * tx + j;
            float v = acc[i][j] + a.bias[col];
            if (MODE == CONV3_DYN || MODE == CONV3_DENSE) v += R[(size_t)orow * a.out_ld + col];
            v = fmaxf(v, 0.f);
            if (zero_s[rr]) v = 0.f;
            O[(size_t)orow * a.out_ld + col] = v;
        }
    }
}

cudaError_t launch_conv_simt(int mode, const ConvArgs &a, int max_rows, cudaStream_t st) {
    if (a.N % kSBN != 0 || a.K % kSBK != 0) return cudaErrorInvalidValue;
    dim3 grid((max_rows + kSBM - 1) / kSBM, a.N / kSBN);
    if (grid.x == 0) return cudaSuccess;
    switch (mode) {
        case CONV1_DYN: conv_simt_kernel<CONV1_DYN><<<grid, 256, 0, st>>>(a); break;
        case CONV2_DYN: conv_simt_kernel<CONV2_DYN><<<grid, 256, 0, st>>>(a); break;
        case CONV3_DYN: conv_simt_kernel<CONV3_DYN><<<grid, 256, 0, st>>>(a); break;
        case CONV1_DENSE: conv_simt_kernel<CONV1_DENSE><<<grid, 256, 0, st>>>(a); break;
        case CONV2_DENSE: conv_simt_kernel<CONV2_DENSE><<<grid, 256, 0, st>>>(a); break;
        case CONV3_DENSE: conv_simt_kernel<CONV3_DENSE><<<grid, 256, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace lasnet

// proj_block.cu -- helpers of the static projection (first) block of a ResNet
// stage (the stride-2 / downsampling first blocks run
// static until their dynamic form is built).  The block reuses the tcgen05
// convolutions; this file holds the stride-s subsampling of an NHWC tensor
// (x for the 1x1 stride-s shortcut, the stride-1 3x3 output for the stride-s
// 3x3): out[n][y][x][:] = in[n][s*y][s*x][:], 16-B vector copies, coalesced
// along channels.
#include <cstdint>
#include <cuda_runtime.h>

#include "launch.cuh"

namespace lasnet {

__global__ void __launch_bounds__(256) subsample_kernel(const uint4 *in, uint4 *__restrict__ out, int n_img,
                                                        int Ho, int Wo, int vpp, int stride) {
    pdl_wait();
    pdl_trigger();
    const long total = (long)n_img * Ho * Wo * vpp;
    const int Wi = Wo * stride, Hi = Ho * stride;
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % vpp);
        const long p = i / vpp;
        const int xo = (int)(p % Wo);
        const long q = p / Wo;
        const int yo = (int)(q % Ho), n = (int)(q / Ho);
        out[i] = in[(((long)n * Hi + (long)yo * stride) * Wi + (long)xo * stride) * vpp + v];
    }
}

// in [n][Ho*stride][Wo*stride][c], out [n][Ho][Wo][c]; c * elt a multiple of 16 bytes.
cudaError_t launch_subsample(const void *in, void *out, int n_img, int Ho, int Wo, int c_bytes, int stride, int num_sms,
                             cudaStream_t st) {
    const long total = (long)n_img * Ho * Wo * (c_bytes / 16);
    if (total == 0) return cudaSuccess;
    long grid = (total + 255) / 256;
    if (grid > 8L * num_sms) grid = 8L * num_sms;
    return launch_k(subsample_kernel, dim3((unsigned)grid), dim3(256), 0, st, static_cast<const uint4 *>(in),
                    static_cast<uint4 *>(out), n_img, Ho, Wo, c_bytes / 16, stride);
}

// out[i] = a[i] + b[i] (fp32): the conv3 and shortcut biases of a projection block,
// applied once by the K-concatenated GEMM.
__global__ void add_bias_kernel(const float *__restrict__ a, const float *__restrict__ b, float *__restrict__ out,
                                int n) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] + b[i];
}

cudaError_t launch_add_bias(const float *a, const float *b, float *out, int n, cudaStream_t st) {
    return launch_k(add_bias_kernel, dim3((n + 255) / 256), dim3(256), 0, st, a, b, out, n);
}

}  // namespace lasnet

// masker_probe.cu -- bandwidth of masker-style cell reductions over a
// [128,28,28,512] bf16 NHWC tensor, L2 flushed by a 256 MB read beforehand.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/masker_probe tools/masker_probe.cu
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

__global__ void rd(const uint4 *p, long n, unsigned *o) {
    unsigned a = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) a ^= p[i].x;
    if (a == 7) o[0] = a;
}

// VARIANT 0: vector-major (v loop outer), 8-deep; 1: pixel-major items, DEPTH-deep
template <int VARIANT, int DEPTH>
__global__ void __launch_bounds__(256) cellsum(const __nv_bfloat16 *x, const float *wm, int N, int H, int W, int C,
                                               int S, float *out) {
    const int lane = threadIdx.x & 31;
    const long cell = (long)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int Gh = (H + S - 1) / S, Gw = (W + S - 1) / S;
    if (cell >= (long)N * Gh * Gw) return;
    const int G = Gh * Gw, n = (int)(cell / G), g = (int)(cell % G), gy = g / Gw, gx = g % Gw;
    const int y0 = gy * S, x0 = gx * S, cw = min(x0 + S, W) - x0, npix = (min(y0 + S, H) - y0) * cw;
    const uint4 *xv = reinterpret_cast<const uint4 *>(x);
    const int nvec = C / 8, nvl = nvec / 32;  // vectors per lane (C >= 256)
    float acc = 0.f;
    if (VARIANT == 0) {
        for (int v = lane; v < nvec; v += 32)
            for (int p0 = 0; p0 < npix; p0 += DEPTH) {
                uint4 q[DEPTH];
#pragma unroll
                for (int u = 0; u < DEPTH; ++u)
                    if (p0 + u < npix) {
                        int p = p0 + u;
                        q[u] = __ldg(xv + (((long)n * H + y0 + p / cw) * W + x0 + p % cw) * nvec + v);
                    }
#pragma unroll
                for (int u = 0; u < DEPTH; ++u)
                    if (p0 + u < npix) acc += __uint_as_float(q[u].x << 16) * wm[v * 8];
            }
    } else {
        const int items = npix * nvl;
        for (int i0 = 0; i0 < items; i0 += DEPTH) {
            uint4 q[DEPTH];
#pragma unroll
            for (int u = 0; u < DEPTH; ++u) {
                const int i = i0 + u;
                if (i < items) {
                    const int p = i / nvl, v = (i - p * nvl) * 32 + lane;
                    const int py = p / cw;
                    q[u] = __ldg(xv + (((long)n * H + y0 + py) * W + x0 + (p - py * cw)) * nvec + v);
                }
            }
#pragma unroll
            for (int u = 0; u < DEPTH; ++u)
                if (i0 + u < items) acc += __uint_as_float(q[u].x << 16) * wm[lane * 8];
        }
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[cell] = acc;
}

int main() {
    const int N = 128, H = 28, W = 28, C = 512;
    size_t bytes = (size_t)N * H * W * C * 2;
    __nv_bfloat16 *x;
    float *wm, *out;
    uint4 *fl;
    unsigned *o;
    cudaMalloc(&x, bytes);
    cudaMemset(x, 0x3c, bytes);
    cudaMalloc(&wm, C * 4);
    cudaMemset(wm, 0, C * 4);
    cudaMalloc(&out, 200000 * 4);
    cudaMalloc(&fl, 256 << 20);
    cudaMemset(fl, 1, 256 << 20);
    cudaMalloc(&o, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto flush = [&]() { rd<<<148 * 4, 512>>>(fl, (256 << 20) / 16, o); };
    auto run = [&](const char *name, auto kern, int S) {
        int Gh = (H + S - 1) / S, Gw = (W + S - 1) / S;
        long cells = (long)N * Gh * Gw;
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            flush();
            cudaEventRecord(a);
            kern<<<(unsigned)((cells + 7) / 8), 256>>>(x, wm, N, H, W, C, S, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-28s S=%d : %7.2f us  %7.1f GB/s\n", name, S, best * 1e3, bytes / best / 1e6);
    };
    {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            flush();
            cudaEventRecord(a);
            rd<<<148 * 4, 512>>>((const uint4 *)x, bytes / 16, o);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("plain stream read            : %7.2f us  %7.1f GB/s\n", best * 1e3, bytes / best / 1e6);
    }
    for (int S : {1, 2, 4, 7}) {
        run("v-major depth8", cellsum<0, 8>, S);
        run("pixel-major depth8", cellsum<1, 8>, S);
        run("pixel-major depth16", cellsum<1, 16>, S);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

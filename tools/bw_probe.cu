// bw_probe.cu -- read-bandwidth calibration on the B200: LDG.128 streaming and
// TMA tiled loads with the box shapes the LASNet kernels use, as a function of
// bytes in flight per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void ldg_sum(const uint4 *__restrict__ p, long n16, int unroll_dummy, unsigned *out) {
    unsigned acc = 0;
    const long stride = (long)gridDim.x * blockDim.x;
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n16; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += stride) {
        uint4 v = __ldg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Each CTA streams `iters` boxes through an ST-stage ring; a box is `nbox`
// TMA ops of `box_bytes` each at coordinates derived from the iteration.
// mode 0: 2-D box {64, rows} over a [rows_total][C] matrix
// mode 1: 4-D box {64, bw, bh, 1} over [N][H][W][C] (per-patch halo boxes)
__global__ void tma_stream(const __grid_constant__ CUtensorMap tm, int mode, int stages, int nbox, int box_bytes,
                           int iters, int rows_total, int C, int H, int W, int N, int oob, unsigned *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[16];
    uint32_t base = (su32(smem) + 1023) & ~1023u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int stage_bytes = nbox * box_bytes;
    unsigned long long seed = blockIdx.x * 7919ull + 1;
    auto issue = [&](int it, int s) {
        uint32_t bar = su32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(stage_bytes));
        for (int b = 0; b < nbox; ++b) {
            // oob bit 1: keep the same boxes for C/64 consecutive iterations (k-block sweep)
            if (!(oob & 2) || (it % (C / 64)) == 0) seed = seed * 6364136223846793005ull + 1442695040888963407ull;
            unsigned long long sd = seed + (unsigned long long)b * 0x9E3779B97F4A7C15ull;
            uint32_t dst = base + s * stage_bytes + b * box_bytes;
            int kc = (it % (C / 64)) * 64;
            if (mode == 0) {
                int row = (int)((sd >> 33) % (unsigned)(rows_total / 128)) * 128;
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                             ::"r"(dst), "l"((uint64_t)&tm), "r"(bar), "r"(kc), "r"(row) : "memory");
            } else {
                int n = (int)((sd >> 33) % (unsigned)N);
                int gy = (int)((sd >> 20) % (unsigned)(H / 4 - 1)), gx = (int)((sd >> 40) % (unsigned)(W / 4 - 1));
                int d = (oob & 1) ? 1 : 0;
                if (mode == 1) {
                    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                                 ::"r"(dst), "l"((uint64_t)&tm), "r"(bar), "r"(kc), "r"(gx * 4 + 1 - d - d), "r"(gy * 4 + 1 - d - d), "r"(n) : "memory");
                } else if (mode == 3) {  // h1-like [P][6][6][128]: box {64,4,4,8}
                    const int p0 = (int)((sd >> 33) % 3000u);
                    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                                 ::"r"(dst), "l"((uint64_t)&tm), "r"(bar), "r"((it & 1) * 64), "r"(it % 3), "r"((it / 3) % 3), "r"(p0) : "memory");
                } else {  // mode 2: 3-D box {64, 6, 6} over [N*H][W][C]
                    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                                 ::"r"(dst), "l"((uint64_t)&tm), "r"(bar), "r"(kc), "r"(gx * 4 + 1 - d - d), "r"(n * H + gy * 4 + 1 - d - d) : "memory");
                }
            }
        }
    };
    for (int s = 0; s < stages && s < iters; ++s) issue(s, s);
    for (int it = 0; it < iters; ++it) {
        int s = it % stages;
        uint32_t par = (it / stages) & 1;
        uint32_t bar = su32(&full[s]);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(bar), "r"(par));
        if (it + stages < iters) issue(it + stages, s);
    }
    out[blockIdx.x] = 1;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) { float ms; cudaEventElapsedTime(&ms, a, b); return ms; }

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int N = 128, H = 28, W = 28, C = 512;
    const size_t bytes = (size_t)N * H * W * C * 2;  // 102.8 MB like config 2
    const size_t big = 1ull << 30;
    uint8_t *d, *flush;
    unsigned *out;
    cudaMalloc(&d, big);
    cudaMalloc(&flush, 512 << 20);
    cudaMalloc(&out, 4096 * 4);
    cudaMemset(d, 1, big);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto flushl2 = [&]() { cudaMemsetAsync(flush, 0, 512 << 20); };
    // LDG streaming read of 1 GiB and of 102.8 MB
    for (size_t nb : {big, bytes}) {
        for (int threads : {512}) {
            for (int blocks_per_sm : {4}) {
                int grid = sms * blocks_per_sm;
                flushl2();
                ldg_sum<<<grid, threads>>>((const uint4 *)d, (long)(nb / 16), 0, out);
                flushl2();
                cudaEventRecord(e0);
                ldg_sum<<<grid, threads>>>((const uint4 *)d, (long)(nb / 16), 0, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = time_ms(e0, e1);
                printf("LDG   bytes=%6.1fMB threads=%d ctas/SM=%d : %7.1f GB/s\n", nb / 1e6, threads, blocks_per_sm,
                       nb / ms / 1e6);
            }
        }
    }
    // TMA streams
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    auto enc = [&](CUtensorMap *m, int rank, const cuuint64_t *gd, const cuuint64_t *gs, const cuuint32_t *bx,
                   CUtensorMapL2promotion promo) {
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, d, gd, gs, bx, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode failed %d\n", (int)r);
    };
    const cuuint64_t gd2[2] = {(cuuint64_t)C, (cuuint64_t)N * H * W}, gs2[1] = {(cuuint64_t)C * 2};
    const cuuint64_t gd4[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
    const cuuint64_t gs4[3] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * W, (cuuint64_t)C * 2 * W * H};
    const cuuint64_t gd3[3] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H * N};
    const cuuint64_t gs3[2] = {(cuuint64_t)C * 2, (cuuint64_t)C * 2 * W};
    CUtensorMap t2_128, t2_36, t4_66, t4_66_np, t4_66_128, t3_66, t4_28x4, th1;
    const cuuint64_t gdh[4] = {128, 6, 6, 3200}, gsh[3] = {256, 256 * 6, 256 * 36};
    const cuuint32_t bh[4] = {64, 4, 4, 8};
    enc(&th1, 4, gdh, gsh, bh, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    const cuuint32_t b2_128[2] = {64, 128}, b2_36[2] = {64, 36}, b4_66[4] = {64, 6, 6, 1}, b3_66[3] = {64, 6, 6},
                     b4_28[4] = {64, 28, 4, 1};
    enc(&t2_128, 2, gd2, gs2, b2_128, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    enc(&t2_36, 2, gd2, gs2, b2_36, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    enc(&t4_66, 4, gd4, gs4, b4_66, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    enc(&t4_66_np, 4, gd4, gs4, b4_66, CU_TENSOR_MAP_L2_PROMOTION_NONE);
    enc(&t4_66_128, 4, gd4, gs4, b4_66, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
    enc(&t3_66, 3, gd3, gs3, b3_66, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    enc(&t4_28x4, 4, gd4, gs4, b4_28, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    struct Cfg { const CUtensorMap *tm; int mode, stages, nbox, box_bytes, flags; const char *name; };
    std::vector<Cfg> cfgs = {
        {&t2_128, 0, 8, 1, 16384, 0, "2D {64,128} rand rows, 8 stg"},
        {&t2_128, 0, 8, 1, 16384, 2, "2D {64,128} rand rows, k-sweep, 8 stg"},
        {&t2_36, 0, 8, 3, 4608, 0, "2D {64,36} x3 rand rows, 8 stg"},
        {&t4_66, 1, 8, 3, 4608, 0, "4D {64,6,6,1} x3 in-bounds, 8 stg"},
        {&t4_66, 1, 8, 3, 4608, 1, "4D {64,6,6,1} x3 OOB corner, 8 stg"},
        {&t4_66, 1, 8, 3, 4608, 2, "4D {64,6,6,1} x3 in-bounds k-sweep, 8 stg"},
        {&t4_66, 1, 16, 3, 4608, 2, "4D {64,6,6,1} x3 in-bounds k-sweep, 16 stg"},
        {&t4_66_np, 1, 8, 3, 4608, 2, "4D {64,6,6,1} no-promo k-sweep, 8 stg"},
        {&t4_66_128, 1, 8, 3, 4608, 2, "4D {64,6,6,1} promo128 k-sweep, 8 stg"},
        {&t3_66, 2, 8, 3, 4608, 2, "3D {64,6,6} k-sweep, 8 stg"},
        {&t4_28x4, 1, 8, 1, 14336, 2, "4D {64,28,4,1} k-sweep, 8 stg"},
        {&th1, 3, 4, 1, 16384, 0, "h1 im2col 4D {64,4,4,8} (L2-resident), 4 stg"},
        {&th1, 3, 8, 1, 16384, 0, "h1 im2col 4D {64,4,4,8} (L2-resident), 8 stg"},
    };
    for (auto &c : cfgs) {
        const int iters = 256;
        int smem = c.stages * c.nbox * c.box_bytes + 1024;
        for (int rep = 0; rep < 2; ++rep) {
            flushl2();
            cudaEventRecord(e0);
            tma_stream<<<sms, 32, smem>>>(*c.tm, c.mode, c.stages, c.nbox, c.box_bytes, iters, N * H * W, C, H, W, N,
                                          c.flags, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaError_t err = cudaGetLastError();
            float ms = time_ms(e0, e1);
            double tot = (double)sms * iters * c.nbox * c.box_bytes;
            if (rep == 1) printf("TMA %-48s : %7.1f GB/s (%s)\n", c.name, tot / ms / 1e6, cudaGetErrorString(err));
        }
    }
    return 0;
}

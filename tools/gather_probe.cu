// gather_probe.cu -- throughput of the conv1 halo gather pattern (no MMA):
// rows = (patch, halo pixel) of 6x6 windows of random 4x4 cells of a
// [128,28,28,512] bf16 NHWC tensor; per K-block 128 rows x 128 B into a ring of
// smem stages.  Variants: cp.async (k-major: one 128-B chunk of each row per
// stage, like the GEMM), cp.async with more threads, and plain LDG + st.shared.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void rd(const uint4 *p, long n, unsigned *o) {
    unsigned a = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) a ^= p[i].x;
    if (a == 7) o[0] = a;
}

// tiles of 128 rows; each CTA handles tiles blockIdx.x, +grid, ...; per tile 8 K-blocks.
// THREADS producer threads; row r of a tile -> random halo pixel (deterministic hash).
template <int THREADS, int STAGES, int MODE>  // MODE 0 cp.async, 1 LDG+STS
__global__ void __launch_bounds__(THREADS + 32) gather(const uint8_t *x, int tiles, unsigned *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const uint32_t base = (su32(smem) + 1023) & ~1023u;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(THREADS));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int H = 28, W = 28, C = 512;
    if (tid < THREADS) {
        constexpr int RPT = 128 * 8 / THREADS;  // 16-B chunks per thread per stage
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            // row -> pixel: patch p = t*3 + row/36 (3 patches of 6x6 per tile)
            long pix[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int q = tid + i * THREADS, row = q >> 3;
                const int patch = t * 3 + min(row / 36, 2), j = row % 36;
                unsigned h = (unsigned)patch * 2654435761u;
                const int n = h % 128, gy = (h >> 8) % 7, gx = (h >> 16) % 7;
                const int yy = min(max(gy * 4 - 1 + j / 6, 0), H - 1), xx = min(max(gx * 4 - 1 + j % 6, 0), W - 1);
                pix[i] = ((long)(n * H + yy) * W + xx) * C * 2;
            }
            for (int kb = 0; kb < 8; ++kb, ++it) {
                const int s = it % STAGES;
                const uint32_t par = ((it / STAGES) & 1) ^ 1;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(su32(&empty[s])), "r"(par));
                const uint32_t sa = base + s * 16384;
                if (MODE == 0) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const int q = tid + i * THREADS, row = q >> 3, ch = q & 7;
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + row * 128 + ((ch ^ (row & 7)) << 4)),
                                     "l"(x + pix[i] + kb * 128 + ch * 16) : "memory");
                    }
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
                } else {
                    uint4 v[RPT];
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const int q = tid + i * THREADS, ch = q & 7;
                        v[i] = *reinterpret_cast<const uint4 *>(x + pix[i] + kb * 128 + ch * 16);
                    }
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const int q = tid + i * THREADS, row = q >> 3, ch = q & 7;
                        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sa + row * 128 + ((ch ^ (row & 7)) << 4)),
                                     "r"(v[i].x), "r"(v[i].y), "r"(v[i].z), "r"(v[i].w) : "memory");
                    }
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
                }
            }
        }
    } else if (tid == THREADS) {
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x)
            for (int kb = 0; kb < 8; ++kb, ++it) {
                const int s = it % STAGES;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(su32(&full[s])), "r"((it / STAGES) & 1));
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
        out[blockIdx.x] = it;
    }
}

// TMA tile::gather4 variant: ISSUERS threads each issue 32/ISSUERS gather4 ops per K-block
// (4 rows x 128 B each) into an mbarrier-tracked ring.
template <int STAGES, int ISSUERS>
__global__ void __launch_bounds__(64) gather_tma(const __grid_constant__ CUtensorMap tm, int tiles, unsigned *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const uint32_t base = (su32(smem) + 1023) & ~1023u;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(ISSUERS));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int H = 28, W = 28;
    if (tid < ISSUERS) {
        constexpr int OPS = 32 / ISSUERS;
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int rows[OPS * 4];
#pragma unroll
            for (int i = 0; i < OPS * 4; ++i) {
                const int row = (tid * OPS * 4 + i);
                const int patch = t * 3 + min(row / 36, 2), j = row % 36;
                unsigned h = (unsigned)patch * 2654435761u;
                const int n = h % 128, gy = (h >> 8) % 7, gx = (h >> 16) % 7;
                const int yy = min(max(gy * 4 - 1 + j / 6, 0), H - 1), xx = min(max(gx * 4 - 1 + j % 6, 0), W - 1);
                rows[i] = (n * H + yy) * W + xx;
            }
            for (int kb = 0; kb < 8; ++kb, ++it) {
                const int s = it % STAGES;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(su32(&empty[s])), "r"(((it / STAGES) & 1) ^ 1));
                const uint32_t bar = su32(&full[s]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(OPS * 512));
#pragma unroll
                for (int o = 0; o < OPS; ++o) {
                    const uint32_t dst = base + s * 16384 + (tid * OPS + o) * 512;
                    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                                 " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                                 ::"r"(dst), "l"((uint64_t)&tm), "r"(bar), "r"(kb * 64), "r"(rows[4 * o]),
                                 "r"(rows[4 * o + 1]), "r"(rows[4 * o + 2]), "r"(rows[4 * o + 3]) : "memory");
                }
            }
        }
    } else if (tid == 32) {
        int it = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x)
            for (int kb = 0; kb < 8; ++kb, ++it) {
                const int s = it % STAGES;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(done) : "r"(su32(&full[s])), "r"((it / STAGES) & 1));
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
        out[blockIdx.x] = it;
    }
}

int main() {
    const size_t bytes = (size_t)128 * 28 * 28 * 512 * 2;
    uint8_t *x;
    uint4 *fl;
    unsigned *o;
    cudaMalloc(&x, bytes);
    cudaMemset(x, 1, bytes);
    cudaMalloc(&fl, 256 << 20);
    cudaMemset(fl, 1, 256 << 20);
    cudaMalloc(&o, 4096 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int tiles = 1046;  // conv1 dyn tiles of the bench workload
    auto run = [&](const char *name, auto kern, int stages, int threads) {
        const int smem = stages * 16384 + 1024;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            rd<<<148 * 4, 512>>>(fl, (256 << 20) / 16, o);
            cudaEventRecord(a);
            kern<<<148, threads + 32, smem>>>(x, tiles, o);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        const double moved = (double)tiles * 8 * 16384;
        printf("%-34s stages=%2d : %7.2f us  %7.1f GB/s gathered  (%s)\n", name, stages, best * 1e3, moved / best / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("cp.async 128 thr", gather<128, 4, 0>, 4, 128);
    run("cp.async 128 thr", gather<128, 6, 0>, 6, 128);
    run("cp.async 128 thr", gather<128, 8, 0>, 8, 128);
    run("cp.async 128 thr", gather<128, 12, 0>, 12, 128);
    run("cp.async 256 thr", gather<256, 4, 0>, 4, 256);
    run("cp.async 256 thr", gather<256, 6, 0>, 6, 256);
    run("cp.async 256 thr", gather<256, 8, 0>, 8, 256);
    run("cp.async 512 thr", gather<512, 6, 0>, 6, 512);
    {
        CUtensorMap tm;
        cuuint64_t gd[2] = {512, 128ull * 28 * 28}, gs[1] = {1024};
        cuuint32_t bx[2] = {64, 1}, es[2] = {1, 1};
        CUresult e = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, gd, gs, bx, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("gather4 tensor map: %d\n", (int)e);
        auto run4 = [&](const char *name, auto kern, int stages) {
            const int smem = stages * 16384 + 1024;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                rd<<<148 * 4, 512>>>(fl, (256 << 20) / 16, o);
                cudaEventRecord(a);
                kern<<<148, 64, smem>>>(tm, tiles, o);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            const double moved = (double)tiles * 8 * 16384;
            printf("%-34s stages=%2d : %7.2f us  %7.1f GB/s gathered  (%s)\n", name, stages, best * 1e3, moved / best / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        };
        run4("TMA gather4, 1 issuer", gather_tma<6, 1>, 6);
        run4("TMA gather4, 4 issuers", gather_tma<6, 4>, 6);
        run4("TMA gather4, 4 issuers", gather_tma<10, 4>, 10);
        run4("TMA gather4, 32 issuers", gather_tma<10, 32>, 10);
    }
    return 0;
}

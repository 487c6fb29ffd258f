// gather4_probe.cu -- hardware probe: throughput of TMA tile::gather4 row gathers (4 arbitrary
// 128-B rows per instruction, 128-B swizzle) from an L2-resident [rows][64] bf16 tensor into a
// ring of 16 KB stages (128 rows each), vs the same gather by cp.async (8 warps x 16 B), at
// several ring depths.  Also checks the landed bytes of one gather4 against the source rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/gather4_probe tools/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hrow(uint32_t a, uint32_t b, uint32_t R) {
    uint32_t x = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u;
    x ^= x >> 15; x *= 0x2C1B3C6Du; x ^= x >> 12;
    return x % R;
}
__device__ __forceinline__ void wait_par(uint32_t b, uint32_t par) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(b), "r"(par) : "memory");
}

// mode 0: gather4 by the 32 lanes of warp 0 (one instruction per 4 rows); mode 1: cp.async by 8 warps
template <int MODE>
__global__ void __launch_bounds__(256) gk(const __grid_constant__ CUtensorMap tm, const uint16_t *src, uint32_t R,
                                          int nkb, int ST, uint16_t *check) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[16], empty[16];
    const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(MODE == 0 ? 1 : 256));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    // consumer: thread 255 waits full, releases empty (models the MMA)
    if (tid == 255 && MODE == 0) {
        for (int it = 0; it < nkb; ++it) {
            const int s = it % ST;
            wait_par(smem_u32(&full[s]), (it / ST) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
        return;
    }
    if (MODE == 0) {
        if (warp != 0) return;
        for (int it = 0; it < nkb; ++it) {
            const int s = it % ST;
            wait_par(smem_u32(&empty[s]), ((it / ST) & 1) ^ 1);
            const uint32_t fb = smem_u32(&full[s]);
            if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(16384) : "memory");
            __syncwarp();
            const uint32_t dst = base + s * 16384 + lane * 512;
            int r[4];
            for (int k = 0; k < 4; ++k) r[k] = (int)hrow(blockIdx.x * 131071u + it, lane * 4 + k, R);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                ::"r"(dst), "l"((uint64_t)&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(fb) : "memory");
            if (check && blockIdx.x == 0 && it == 0) {  // verify the first stage after it lands
                wait_par(fb, 0);
                for (int k = 0; k < 4; ++k)
                    for (int c = 0; c < 8; ++c) {
                        const int row = lane * 4 + k;
                        const uint16_t *sp = reinterpret_cast<const uint16_t *>(
                            smem + (base - smem_u32(smem)) + s * 16384 + row * 128 + ((c ^ (row & 7)) << 4));
                        for (int e = 0; e < 8; ++e) check[(row * 8 + c) * 8 + e] = sp[e] ^ src[(size_t)r[k] * 64 + c * 8 + e];
                    }
            }
        }
    } else {
        // cp.async: thread -> (row group tid >> 3, chunk tid & 7), 4 rows per thread per stage
        for (int it = 0; it < nkb; ++it) {
            const int s = it % ST;
            wait_par(smem_u32(&empty[s]), ((it / ST) & 1) ^ 1);
            for (int i = 0; i < 4; ++i) {
                const int row = (tid >> 3) + 32 * i, c = tid & 7;
                const uint32_t rr = hrow(blockIdx.x * 131071u + it, row, R);
                const uint32_t dst = base + s * 16384 + row * 128 + ((c ^ (row & 7)) << 4);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + (size_t)rr * 64 + c * 8) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
            if (tid == 0) {  // consumer role folded into thread 0: wait this stage, release it
                wait_par(smem_u32(&full[s]), (it / ST) & 1);
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            }
        }
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const uint32_t R = 200704;  // 4 x 50176 rows of 64 bf16 = 25.7 MB
    uint16_t *src;
    cudaMalloc(&src, (size_t)R * 128);
    std::vector<uint16_t> h((size_t)R * 64);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
    cudaMemcpy(src, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    uint16_t *chk;
    cudaMalloc(&chk, 128 * 64 * 2);
    cudaMemset(chk, 0xFF, 128 * 64 * 2);
    int sms = 148;
    for (int boxh : {1, 4}) {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {64, R}, str[1] = {128};
        const cuuint32_t box[2] = {64, (cuuint32_t)boxh}, es[2] = {1, 1};
        CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("boxh %d encode %d\n", boxh, (int)cr);
        if (cr) continue;
        for (int ST : {3, 6, 10}) {
            const int smem = ST * 16384 + 1024;
            cudaFuncSetAttribute(gk<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(gk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (int mode = 0; mode < 2; ++mode) {
                if (mode == 1 && boxh == 4) continue;
                const int nkb = 2000;
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEventRecord(a);
                    if (mode == 0) gk<0><<<sms, 256, smem>>>(tm, src, R, nkb, ST, rep == 0 ? chk : nullptr);
                    else gk<1><<<sms, 256, smem>>>(tm, src, R, nkb, ST, nullptr);
                    cudaEventRecord(b);
                    cudaError_t e = cudaEventSynchronize(b);
                    if (e) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                }
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double bytes = (double)sms * nkb * 16384;
                printf("  %s ST=%2d: %.1f us  %.2f TB/s total  %.1f GB/s/SM\n", mode ? "cp.async" : "gather4 ", ST,
                       ms * 1e3, bytes / ms / 1e9, bytes / ms / 1e6 / sms);
            }
        }
        std::vector<uint16_t> hc(128 * 64);
        cudaMemcpy(hc.data(), chk, hc.size() * 2, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (auto v : hc) bad += v != 0;
        printf("  gather4 landed-bytes check: %d mismatching elements of %zu\n", bad, hc.size());
        cudaMemset(chk, 0xFF, 128 * 64 * 2);
    }
    return 0;
}

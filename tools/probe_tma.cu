// probe_tma.cu -- hardware probe: where does a 128B-swizzled TMA box land in
// shared memory when its destination is 128-B but not 1024-B aligned?
// Also checks 4-D boxes with negative (out-of-bounds) coordinates zero-fill.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma tools/probe_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm4,
                      int off_bytes, int rows, uint16_t *out2, uint16_t *out4) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    uint8_t *gbase = smem + (base - smem_u32(smem));
    for (int i = threadIdx.x; i < 32768 / 2; i += blockDim.x) reinterpret_cast<uint16_t *>(gbase)[i] = 0xFFFF;
    __syncthreads();
    uint32_t b = smem_u32(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(rows * 128));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(base + off_bytes), "l"((uint64_t)&tm2), "r"(b), "r"(0), "r"(0) : "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b));
        }
        // 4-D box {64, 6, 6, 1} at (0, -1, -1, 0): first row/col must be zero-filled
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(36 * 128));
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
                     ::"r"(base + 16384), "l"((uint64_t)&tm4), "r"(b), "r"(0), "r"(-1), "r"(-1), "r"(0) : "memory");
        done = 0;
        while (!done) {
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(b));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 16384 / 2; i += blockDim.x) {
        out2[i] = reinterpret_cast<uint16_t *>(gbase)[i];
        out4[i] = reinterpret_cast<uint16_t *>(gbase + 16384)[i];
    }
}

int main() {
    // global 2-D tensor [64 rows][64 cols] bf16-sized values: v = row*64 + col
    const int R = 64, C = 64;
    std::vector<uint16_t> h(R * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 64 + c);
    uint16_t *d, *o2, *o4;
    cudaMalloc(&d, h.size() * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    cudaMalloc(&o2, 16384);
    cudaMalloc(&o4, 16384);
    // 4-D tensor [N=1][H=8][W=8][C=64] with the same values (pixel p = y*8+x -> row p)
    CUtensorMap tm2, tm4;
    cuuint64_t gd2[2] = {64, 64}, gs2[1] = {128};
    cuuint32_t bx2[2] = {64, 0}, es2[2] = {1, 1};
    cuuint64_t gd4[4] = {64, 8, 8, 1}, gs4[3] = {128, 128 * 8, 128 * 64};
    cuuint32_t bx4[4] = {64, 6, 6, 1}, es4[4] = {1, 1, 1, 1};
    int rows_list[3] = {6, 9, 36};
    int offs[6] = {0, 128, 256, 640, 768, 4608};
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    int bad_total = 0;
    for (int ri = 0; ri < 3; ++ri) {
        int rows = rows_list[ri];
        bx2[1] = rows;
        CUresult e1 = cuTensorMapEncodeTiled(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, gd2, gs2, bx2, es2,
                                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult e2 = cuTensorMapEncodeTiled(&tm4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, d, gd4, gs4, bx4, es4,
                                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (e1 || e2) { printf("encode failed %d %d\n", e1, e2); return 1; }
        for (int oi = 0; oi < 6; ++oi) {
            int off = offs[oi];
            probe<<<1, 128, 40000>>>(tm2, tm4, off, rows, o2, o4);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("launch failed %s\n", cudaGetErrorString(e)); return 1; }
            std::vector<uint16_t> s2(8192), s4(8192);
            cudaMemcpy(s2.data(), o2, 16384, cudaMemcpyDeviceToHost);
            cudaMemcpy(s4.data(), o4, 16384, cudaMemcpyDeviceToHost);
            // hypothesis A: swizzle keyed on absolute smem row ((off/128 + r) & 7)
            // hypothesis B: swizzle keyed on box-relative row (r & 7)
            int badA = 0, badB = 0;
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < 64; ++c) {
                    int j = c / 8, e8 = c % 8;
                    int rowabs = off / 128 + r;
                    int ia = (rowabs * 128 + ((j ^ (rowabs & 7)) * 16)) / 2 + e8;
                    int ib = (off + r * 128 + ((j ^ (r & 7)) * 16)) / 2 + e8;
                    uint16_t want = (uint16_t)(r * 64 + c);
                    badA += s2[ia] != want;
                    badB += s2[ib] != want;
                }
            printf("2D rows=%2d off=%5d : absolute-address swizzle mismatches=%d, box-relative mismatches=%d\n",
                   rows, off, badA, badB);
            if (ri == 0 && oi == 0) {
                // 4-D: box row q = wy*6+wx holds pixel (y=wy-1, x=wx-1) or zeros when OOB; swizzle at offset 16384 (aligned)
                int bad4 = 0;
                for (int wy = 0; wy < 6; ++wy)
                    for (int wx = 0; wx < 6; ++wx)
                        for (int c = 0; c < 64; ++c) {
                            int q = wy * 6 + wx, j = c / 8;
                            int ia = (q * 128 + ((j ^ (q & 7)) * 16)) / 2 + c % 8;
                            int y = wy - 1, x = wx - 1;
                            uint16_t want = (y < 0 || x < 0) ? 0 : (uint16_t)((y * 8 + x) * 64 + c);
                            bad4 += s4[ia] != want;
                        }
                printf("4D box {64,6,6,1} at (0,-1,-1,0): mismatches=%d (zero-fill of OOB rows)\n", bad4);
                bad_total += bad4;
            }
        }
    }
    printf("done\n");
    return 0;
}

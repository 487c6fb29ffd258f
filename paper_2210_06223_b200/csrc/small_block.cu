// small_block.cu -- the whole fp32 block in ONE launch for small batches
// (BASELINE configs[0]: N = 1, 14x14x256, c_mid 64, S = 2).
//
// At N = 1 the block is a chain of tiny dependent steps (masker, compaction,
// conv1, conv2, conv3 + scatter-add: ~10 MFLOP), so five or six launches cost
// far more than their arithmetic.  Here one cooperative grid runs the steps as
// phases separated by a software grid barrier (every CTA is co-resident:
// cooperative launch):
//   phase 0  masker (dynamic only; P:109 avg-pool + 1x1 conv, App. B P:562 sign
//            form): one warp per cell, fp64 sum of the exact products
//            w_c x[p,c] (fp32 x fp32 fits a double), logit = sum / |Omega| + b,
//            active iff logit > 0 (R3); mask out
//   phase 1  every CTA rebuilds the ascending active-cell list and
//            the set U of pixels some active cell's (S+2)^2 window needs, in
//            shared memory (CTA 0 writes idx / count); conv1 runs ONCE per
//            pixel of U (the dilated union of the active cells: each h1 pixel
//            computed once however many windows share it, instead of once per
//            window as the halo gather does) -> h1 [pixel][c_mid]
//   phase 2  conv2 on the active output pixels: im2col rows read h1 at the nine
//            neighbours (0 outside the image, R6) -> h2 [row][c_mid]
//   phase 3  conv3 + residual + ReLU, written in place to the active pixels
//            (inactive pixels keep x)
// The dense comparator (wm == NULL) runs phases 1-3 on every pixel.
// GEMM work items are 16 rows x 32 output channels; a CTA stages the item's A
// rows and weight rows for a K piece with cp.async (all loads of the piece in
// flight at once: one memory round trip); the eight warps split the piece's K and
// keep 16 row sums per lane, added in a fixed order at the end (fp32 FMA).
#include <cstdint>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "small_block.cuh"

namespace lasnet {

#ifdef LASNET_TRACE
// globaltimer of CTA 0 / last CTA at: [0] start, [1] masker done, [2] phase-1 lists, [3] conv1 done,
// [4] barrier 2 passed, [5] conv2 done, [6] barrier 3 passed, [7] end  (CTA 0: [0..7], last CTA: [8..15])
__device__ unsigned long long g_small_trace[16];
__device__ __forceinline__ void small_mark(int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (threadIdx.x == 0 && blockIdx.x == 0) g_small_trace[k] = t;
    if (threadIdx.x == 0 && blockIdx.x == gridDim.x - 1) g_small_trace[8 + k] = t;
}
extern "C" int lasnet_small_trace_read(unsigned long long *h) {
    return (int)cudaMemcpyFromSymbol(h, g_small_trace, sizeof(g_small_trace));
}
#define SMARK(k) small_mark(k)
#else
#define SMARK(k) do { } while (0)
#endif

constexpr int kSmThreads = 256;
constexpr int kSmRows = 16, kSmCols = 32, kSmKPiece = 288;  // 9 x 32: conv2's taps split evenly
constexpr int kSmMaxCells = 4096, kSmMaxPx = 16384;

__device__ __forceinline__ void cp_async_f4(float *dst, const float *src, bool ok) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16u : 0u) : "memory");
}

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Software grid barrier (all CTAs co-resident), sense by generation count.
__device__ void grid_barrier(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acq(bar + 1);
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            bar[0] = 0u;
            asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar + 1) : "memory");
        } else {
            while (ld_acq(bar + 1) == gen) __nanosleep(32);
        }
    }
    __syncthreads();
}

// One 16 x 32 GEMM item: out[r][c0 + j] = act(sum_k A[r][k] B[c0 + j][k] + bias (+ resid)).
// rowptr(r, k0) returns the address of A[r][k0 .. k0 + 3] or nullptr (zero), k0 % 4 == 0
// and a float4 never straddles a 3x3 tap (cm % 32 == 0); B rows are K contiguous floats.
// Shared memory: A [16][piece] and B [32][piece + 4] (both cp.async, all loads of a piece in
// flight at once).  The eight warps split the piece's k-quads (warp w takes quads w, w + 8,
// ...); lane l owns column l and keeps all 16 row sums, so each 16-B B load (lane-distinct,
// conflict-free at the padded pitch) and each broadcast A load feed 16 or 4 FMAs.  The
// warps' partial sums are added in warp order at the end (fixed order).
constexpr int kSmBPitch = kSmKPiece + 4;
template <typename RowPtr, typename Store>
__device__ void gemm_item(int K, const float *B, int c0, RowPtr rowptr, Store store, float *sA, float *sB) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float acc[kSmRows];
#pragma unroll
    for (int r = 0; r < kSmRows; ++r) acc[r] = 0.f;
    for (int k0 = 0; k0 < K; k0 += kSmKPiece) {
        const int kp = min(kSmKPiece, K - k0), kv = kp / 4;
        __syncthreads();  // the previous piece's reads are done
        for (int i = tid; i < kSmRows * kv; i += kSmThreads) {
            const int r = i / kv, v = i - r * kv;
            const float *p = rowptr(r, k0 + 4 * v);
            cp_async_f4(sA + r * kSmKPiece + 4 * v, p ? p : B, p != nullptr);
        }
        for (int i = tid; i < kSmCols * kv; i += kSmThreads) {
            const int c = i / kv, v = i - c * kv;
            cp_async_f4(sB + c * kSmBPitch + 4 * v, B + (size_t)(c0 + c) * K + k0 + 4 * v, true);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        const float *bl = sB + lane * kSmBPitch;
        for (int v = warp; v < kv; v += kSmThreads / 32) {
            const float4 bq = *reinterpret_cast<const float4 *>(bl + 4 * v);
#pragma unroll
            for (int r = 0; r < kSmRows; ++r) {
                const float4 aq = *reinterpret_cast<const float4 *>(sA + r * kSmKPiece + 4 * v);
                acc[r] = fmaf(aq.x, bq.x, acc[r]);
                acc[r] = fmaf(aq.y, bq.y, acc[r]);
                acc[r] = fmaf(aq.z, bq.z, acc[r]);
                acc[r] = fmaf(aq.w, bq.w, acc[r]);
            }
        }
    }
    // cross-warp reduction through shared memory (reuses sB), fixed warp order
    __syncthreads();
    float *red = sB;  // [8 warps][16 rows][32 cols]
#pragma unroll
    for (int r = 0; r < kSmRows; ++r) red[(warp * kSmRows + r) * kSmCols + lane] = acc[r];
    __syncthreads();
    for (int o = tid; o < kSmRows * kSmCols / 2; o += kSmThreads) {  // thread: rows 2 rr, 2 rr + 1 of column c
        const int c = o % kSmCols, rr = 2 * (o / kSmCols);
        float v0 = 0.f, v1 = 0.f;
        for (int w = 0; w < kSmThreads / 32; ++w) {
            v0 += red[(w * kSmRows + rr) * kSmCols + c];
            v1 += red[(w * kSmRows + rr + 1) * kSmCols + c];
        }
        store(rr, c, v0, v1);
    }
}

__global__ void __launch_bounds__(kSmThreads) small_block_kernel(const SmallArgs a) {
    extern __shared__ float4 smem4[];
    float *sA = reinterpret_cast<float *>(smem4);
    float *sB = sA + kSmRows * kSmKPiece;
    int *s_idx = reinterpret_cast<int *>(sB + kSmCols * kSmBPitch);  // [ncells] active cell ids
    int *s_u = s_idx + kSmMaxCells;                                   // [px] pixels of U, ascending
    uint8_t *s_mask = reinterpret_cast<uint8_t *>(s_u + kSmMaxPx);     // [ncells] decisions
    __shared__ int s_cnt, s_nu;
    __shared__ int s_wsum[kSmThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool dense = a.wm == nullptr;
    const int S = a.S, ss = S * S;
    pdl_wait();
    pdl_trigger();
    SMARK(0);

    // ---- phase 0: masker, one warp per cell (fp64, exact products) ----
    if (!dense) {
        const int nwarps = gridDim.x * (kSmThreads / 32);
        const int nv = a.ci / 4;
        for (int c = blockIdx.x * (kSmThreads / 32) + warp; c < a.ncells; c += nwarps) {
            const int G = a.Gh * a.Gw, n = c / G, g = c - n * G, gy = g / a.Gw, gx = g - gy * a.Gw;
            const int y0 = gy * S, x0 = gx * S, y1 = min(y0 + S, a.H), x1 = min(x0 + S, a.W);
            // item j = (pixel, channel vector) of the cell; a lane's items in batches of 8 loads
            // in flight (fixed order: pixel-major, vector-minor)
            const int cw = x1 - x0, nitems = (y1 - y0) * cw * nv;
            double s = 0.0;
            for (int b0 = lane; b0 < nitems; b0 += 8 * 32) {
                float4 q[8], w[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int it = b0 + 32 * j;
                    q[j] = w[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (it < nitems) {
                        const int p = it / nv, v = it - p * nv, yy = y0 + p / cw, xx = x0 + p % cw;
                        q[j] = reinterpret_cast<const float4 *>(a.x + ((size_t)(n * a.H + yy) * a.W + xx) * a.ci)[v];
                        w[j] = reinterpret_cast<const float4 *>(a.wm)[v];
                    }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    s = fma((double)w[j].x, (double)q[j].x, s);
                    s = fma((double)w[j].y, (double)q[j].y, s);
                    s = fma((double)w[j].z, (double)q[j].z, s);
                    s = fma((double)w[j].w, (double)q[j].w, s);
                }
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) {
                const double logit = s / (double)((y1 - y0) * (x1 - x0)) + (double)a.bm;
                a.mask[c] = logit > 0.0 ? 1 : 0;
            }
        }
        SMARK(1);
        grid_barrier(a.bar);
    }

    // ---- phase 1: active list, the needed-pixel set U, conv1 on U ----
    // ascending compaction of a 0/1 predicate over [0, m) into out (every CTA, block scan)
    auto compact = [&](int m, auto pred, int *out) -> int {
        int base = 0;
        for (int b0 = 0; b0 < m; b0 += kSmThreads) {
            const int i = b0 + tid;
            const int f = i < m && pred(i);
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (lane == 0) s_wsum[warp] = __popc(bal);
            __syncthreads();
            int off = base;
            for (int w = 0; w < warp; ++w) off += s_wsum[w];
            if (f) out[off + __popc(bal & ((1u << lane) - 1u))] = i;
            int tot = 0;
            for (int w = 0; w < kSmThreads / 32; ++w) tot += s_wsum[w];
            base += tot;
            __syncthreads();
        }
        return base;
    };
    if (!dense) {  // the decisions into shared memory (one coalesced pass; written by other CTAs)
        const volatile uint8_t *vmask = a.mask;
        for (int i = tid; i < a.ncells; i += kSmThreads) s_mask[i] = vmask[i];
        __syncthreads();
    }
    const int cnt = dense ? a.ncells : compact(a.ncells, [&](int c) { return s_mask[c] != 0; }, s_idx);
    // pixel p is needed iff a cell whose (S+2)^2 window covers p is active: p = (n, yy, xx) lies in the
    // window of cell (gy, gx) iff gy*S - 1 <= yy <= gy*S + S, i.e. gy in [ceil((yy-S)/S), floor((yy+1)/S)]
    const int nu = dense ? a.px : compact(a.px, [&](int p) {
        const int n = p / (a.H * a.W), rem = p - n * a.H * a.W, yy = rem / a.W, xx = rem - yy * a.W;
        // window rows of cell row gy: [gy*S - 1, gy*S + S]  =>  ceil(yy/S) - 1 <= gy <= (yy + 1) / S
        const int gy0 = max(0, (yy + S - 1) / S - 1), gy1 = min(a.Gh - 1, (yy + 1) / S);
        const int gx0 = max(0, (xx + S - 1) / S - 1), gx1 = min(a.Gw - 1, (xx + 1) / S);
        for (int gy = gy0; gy <= gy1; ++gy)
            for (int gx = gx0; gx <= gx1; ++gx)
                if (s_mask[(n * a.Gh + gy) * a.Gw + gx]) return true;
        return false;
    }, s_u);
    if (tid == 0) {
        s_cnt = cnt;
        s_nu = nu;
    }
    if (!dense && blockIdx.x == 0) {  // the ids and count outputs
        for (int i = tid; i < cnt; i += kSmThreads) a.idx[i] = s_idx[i];
        if (tid == 0) *a.count = cnt;
    }
    __syncthreads();
    SMARK(2);
    {
        const int rtiles = (nu + kSmRows - 1) / kSmRows, ctiles = a.cm / kSmCols;
        for (int item = blockIdx.x; item < rtiles * ctiles; item += gridDim.x) {
            const int rt = item / ctiles, c0 = (item - rt * ctiles) * kSmCols;
            gemm_item(
                a.ci, a.w1, c0,
                [&](int r, int k) -> const float * {
                    const int u = rt * kSmRows + r;
                    return u < nu ? a.x + (size_t)(dense ? u : s_u[u]) * a.ci + k : nullptr;
                },
                [&](int r, int c, float v0, float v1) {  // rows r, r + 1 of column c
                    const float bias = a.b1[c0 + c];
                    for (int i = 0; i < 2; ++i) {
                        const int u = rt * kSmRows + r + i;
                        if (u < nu) a.h1[(size_t)(dense ? u : s_u[u]) * a.cm + c0 + c] = fmaxf((i ? v1 : v0) + bias, 0.f);
                    }
                },
                sA, sB);
        }
    }
    SMARK(3);
    grid_barrier(a.bar);
    SMARK(4);

    // output pixel of GEMM row r of phases 2-3 (or -1: past the end / clipped at the border, R7)
    const int rows = dense ? a.px : cnt * ss;
    // per GEMM row of phases 2-3 (decoded once per CTA, reusing the U list's space): the output
    // pixel (or -1: clipped at the border, R7) and its (y, x) packed as y << 16 | x
    int *s_opix = s_u, *s_oyx = s_u + kSmMaxPx / 2;
    for (int r = tid; r < rows; r += kSmThreads) {
        int p, yy, xx;
        if (dense) {
            p = r;
            const int rem = r % (a.H * a.W);
            yy = rem / a.W;
            xx = rem - yy * a.W;
        } else {
            const int t = r / ss, j = r - t * ss;
            const int c = s_idx[t], G = a.Gh * a.Gw, n = c / G, g = c - n * G, gy = g / a.Gw, gx = g - gy * a.Gw;
            yy = gy * S + j / S;
            xx = gx * S + j % S;
            p = (yy < a.H && xx < a.W) ? (n * a.H + yy) * a.W + xx : -1;
        }
        s_opix[r] = p;
        s_oyx[r] = (yy << 16) | xx;
    }
    __syncthreads();
    auto out_px = [&](int r) -> int { return r < rows ? s_opix[r] : -1; };

    // ---- phase 2: conv2 (3x3, zero padding) on the active pixels ----
    {
        const int K = 9 * a.cm;
        const int rtiles = (rows + kSmRows - 1) / kSmRows, ctiles = a.cm / kSmCols;
        for (int item = blockIdx.x; item < rtiles * ctiles; item += gridDim.x) {
            const int rt = item / ctiles, c0 = (item - rt * ctiles) * kSmCols;
            gemm_item(
                K, a.w2, c0,
                [&](int r, int k) -> const float * {
                    const int rr = rt * kSmRows + r;
                    const int p = out_px(rr);
                    if (p < 0) return nullptr;
                    const int tap = k / a.cm, ch = k - tap * a.cm, dy = tap / 3 - 1, dx = tap - 3 * (tap / 3) - 1;
                    const int yx = s_oyx[rr], yy = (yx >> 16) + dy, xx = (yx & 0xFFFF) + dx;
                    if (yy < 0 || yy >= a.H || xx < 0 || xx >= a.W) return nullptr;
                    return a.h1 + (size_t)(p + dy * a.W + dx) * a.cm + ch;
                },
                [&](int r, int c, float v0, float v1) {
                    const float bias = a.b2[c0 + c];
                    for (int i = 0; i < 2; ++i) {
                        const int rr = rt * kSmRows + r + i;
                        if (out_px(rr) >= 0) a.h2[(size_t)rr * a.cm + c0 + c] = fmaxf((i ? v1 : v0) + bias, 0.f);
                    }
                },
                sA, sB);
        }
    }
    SMARK(5);
    grid_barrier(a.bar);
    SMARK(6);

    // ---- phase 3: conv3 + residual + ReLU -> y (in place on the active pixels) ----
    {
        const int rtiles = (rows + kSmRows - 1) / kSmRows, ctiles = a.co / kSmCols;
        for (int item = blockIdx.x; item < rtiles * ctiles; item += gridDim.x) {
            const int rt = item / ctiles, c0 = (item - rt * ctiles) * kSmCols;
            gemm_item(
                a.cm, a.w3, c0,
                [&](int r, int k) -> const float * {
                    const int rr = rt * kSmRows + r;
                    return out_px(rr) >= 0 ? a.h2 + (size_t)rr * a.cm + k : nullptr;
                },
                [&](int r, int c, float v0, float v1) {
                    const float bias = a.b3[c0 + c];
                    for (int i = 0; i < 2; ++i) {
                        const int p = out_px(rt * kSmRows + r + i);
                        if (p < 0) continue;
                        const size_t o = (size_t)p * a.co + c0 + c;
                        const float res = a.x[o];  // read before the (in-place) write, same thread
                        a.y[o] = fmaxf((i ? v1 : v0) + bias + res, 0.f);
                    }
                },
                sA, sB);
        }
    }
    SMARK(7);
}

size_t small_block_smem_bytes() {
    static_assert(kSmCols * kSmBPitch >= (kSmThreads / 32) * kSmRows * kSmCols, "reduction buffer");
    return (size_t)(kSmRows * kSmKPiece + kSmCols * kSmBPitch) * 4 + (size_t)(kSmMaxCells + kSmMaxPx) * 4 +
           kSmMaxCells;
}

// Eligible shapes: fp32, stride 1, identity widths, c_in % 4, c_mid / c_out % 32, and the
// per-CTA lists fit shared memory.  Returns cudaErrorNotSupported otherwise (nothing launched).
cudaError_t launch_small_block(const SmallArgs &a, int num_sms, cudaStream_t st) {
    if (a.ncells > kSmMaxCells || a.px > kSmMaxPx / 2 || a.ncells * a.S * a.S > kSmMaxPx / 2 || a.ci % 4 ||
        a.cm % kSmCols || a.co % kSmCols)
        return cudaErrorNotSupported;
    const size_t smem = small_block_smem_bytes();
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(small_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    // enough CTAs for the largest phase, at most one per SM (all co-resident: cooperative launch)
    const int rows = a.wm ? a.ncells * a.S * a.S : a.px;
    const int items = ((rows > a.px ? rows : a.px) + kSmRows - 1) / kSmRows * (a.co / kSmCols);
    const int grid = items < num_sms ? (items > 0 ? items : 1) : num_sms;
    return launch_k_coop(small_block_kernel, dim3(grid), dim3(kSmThreads), smem, st, a);
}

}  // namespace lasnet

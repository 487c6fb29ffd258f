// decide_gather.cu -- steps 1 (decision) and 2 of the masker-fused schedule,
// plus the h1 halo gather that feeds the fused conv2+conv3 kernel.
//
// The paper's best schedule (Table 1; sec. 3.4; App. B
// P:556-565) fuses the masker into a STATIC conv1: conv1 runs on every pixel and
// the masker's pooled 1x1 conv rides along.  Here the dense conv1 kernel
// (conv_tc.cu, CONV1_DENSE_MASK) leaves per pixel p, for the lower (h = 0) and the
// upper (h = 1) 32 channels of every 64-channel K-block, the fp32 partials
//   a_ph = sum_c wm_c x[p,c]   and   m_ph = sum_c |wm_c x[p,c]|,
// and one cooperative launch finishes steps 1-2 (a second one the gathered copy, when used):
//   (a) decides each cell (P:109 avg-pool + 1x1 conv, P:562 sign form):
//       z = sum_{p in Omega} (a_p0 + a_p1) + bm*|Omega| in fp64.  With gamma_n =
//       n u/(1-n u) (Higham, recursive summation): every channel term of a_ph
//       passes through at most 8 (FFMA chain of its 16-B chunk) + c_in/32 (chunk
//       sums into two chains) + 2 fp32 roundings (the bound uses c_in/16 + 10), and through at most 2|Omega| + 4 fp64 additions
//       here, so |z - z_exact| <= (gamma_{c_in/16+10}(2^-24) + gamma_{2|Omega|+4}(2^-53))
//       * sum |terms|, and sum |terms| <= 1.01 sum m_ph (the m are fp32 sums of
//       non-negative terms, relative error < 1e-3 for c_in < 16k).
//       When |z| exceeds that bound the sign is the exact sign; otherwise (~1e-5
//       of the cells) the cell is re-summed from x in fp64 (exact products) --
//       the rule of the standalone masker (R20).
//       decide_kernel<true>, four lanes per cell, 64-cell chunks (a CTA takes several
//       when the map has more chunks than the grid can hold co-resident): writes the
//       mask and the active count of every 32-cell group, then after a software grid
//       barrier (cooperative launch) each chunk sums the counts before it and writes
//       its ids (ascending) and group prefixes; the last chunk writes the count.
//       (decide_kernel<false>, the fallback: one chunk per CTA, the last CTA to finish
//       turns the counts into prefixes; compact_idx_kernel writes the ids.)
//   (b) compact_gather_kernel, one warp per (group, 64-channel chunk, halo row):
//       the group's active cells get positions prefix + ballot rank (ascending
//       cell ids, App. B: idx/count), and the warp copies that halo row
//       of h1 of each of them from the dense h1 [c_mid/64][n][h][w][64] into the
//       patch-major gathered layout [c_mid/64][cap][S+2][S+2][64] that conv23's
//       im2col TMA box reads; pixels outside the image are 0 (R6: conv2's zero
//       padding).  Thousands of independent warps keep the copy bandwidth-bound.
// The done counter is zero on entry and reset by the last CTA (no memset).
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"

namespace lasnet {

struct DecideArgs {
    const float4 *mpart;        // [n*h*w] (a_p0, m_p0, a_p1, m_p1)
    const __nv_bfloat16 *x;     // [n][h][w][c_in] (exact fallback)
    const float *wm;            // [c_in]
    float bm;
    int n_img, H, W, c_in, S, Gh, Gw;
    int ncells, ngroups;        // cells, 32-cell groups
    uint8_t *dec;               // [ncells] decisions (caller's mask or workspace)
    int32_t *gpre;              // [ngroups] group counts -> exclusive prefixes
    int32_t *count;
    int32_t *idx;               // COOP: active cell ids
    int32_t *gpx;               // COOP: [ngroups] exclusive group prefixes
    unsigned *done;             // [0] CTAs finished (zero on entry, reset by the last); COOP: [1] arrivals, [2] generation
};

constexpr int kDecThreads = 256;

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// fp64 sum_{p in Omega} sum_c wm_c x[p,c] of one cell by the whole CTA (bf16 x
// fp32 products are exact in fp64): thread t takes the 16-B channel vectors
// t, t + 256, ... of the cell, four loads in flight, then a fixed-order warp and
// CTA reduction.  Every thread calls it; the result is returned to all.
__device__ double cell_exact(const DecideArgs &a, int n, int y0, int x0, int ch, int cw, double *s_red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nvec = a.c_in / 8, total = ch * cw * nvec;  // 16-B vectors of the cell
    double s = 0.0;
    for (int i0 = tid; i0 < total; i0 += 4 * kDecThreads) {
        uint4 q[4];
        int v8[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * kDecThreads;
            q[u] = make_uint4(0u, 0u, 0u, 0u);
            v8[u] = 0;
            if (i < total) {
                const int p = i / nvec, v = i - p * nvec, py = p / cw, px = p - py * cw;
                const uint4 *row = reinterpret_cast<const uint4 *>(
                    a.x + ((size_t)((n * a.H + y0 + py) * a.W) + x0 + px) * a.c_in);
                q[u] = __ldg(row + v);
                v8[u] = 8 * v;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t qq[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
            for (int e = 0; e < 8; ++e) {  // a zero vector (past the end) adds exact zeros
                const uint32_t b = (e & 1) ? (qq[e >> 1] >> 16) : (qq[e >> 1] & 0xFFFFu);
                s = fma((double)__ldg(a.wm + v8[u] + e), (double)__uint_as_float(b << 16), s);
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) s_red[warp] = s;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) t += s_red[w];
    __syncthreads();  // s_red is reused by the next call
    return t;
}

// Four lanes per cell (a quad): lane j of the quad sums the partials of the
// cell's pixel rows j, j+4, ... in fp64, the quad combines them (fixed order).
constexpr int kDecCells = kDecThreads / 4;  // cells per CTA (a multiple of 32)

// the partials were written by the previous kernel (conv1) while this grid may already be resident
// (programmatic dependent launch): read them at L2, never through the non-coherent path
__device__ __forceinline__ float4 ld_cg_f4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// COOP (all CTAs co-resident; the direct schedule): a CTA decides the 64-cell chunks
// blockIdx.x, blockIdx.x + gridDim.x, ... (the grid is capped at the co-residency
// capacity, so large maps take several chunks per CTA), then a grid barrier, then
// for each of its chunks it sums the group counts before the chunk and writes the ids
// of its active cells -- no last-CTA scan and no second launch.  !COOP: one chunk per
// CTA, the last CTA to finish turns the group counts into prefixes (ids by a second launch).
template <bool COOP>
__global__ void __launch_bounds__(kDecThreads) decide_kernel(const DecideArgs a) {
    __shared__ int s_unc[kDecCells], s_nunc;
    __shared__ uint8_t s_dec[kDecCells];
    __shared__ int s_last;
    __shared__ double s_red[kDecThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = a.Gh * a.Gw;
    const int lc = tid >> 2, q = tid & 3;  // local cell, lane in the quad
    const int nchunks = (a.ncells + kDecCells - 1) / kDecCells;
    pdl_wait();
    pdl_trigger();
    for (int chunk = blockIdx.x; chunk < (COOP ? nchunks : (int)blockIdx.x + 1); chunk += gridDim.x) {
        const int cell0 = chunk * kDecCells;
        if (tid == 0) s_nunc = 0;
        __syncthreads();

        // certified decision per cell from the fused conv1's partials
        const int cell = cell0 + lc;
        const bool valid = cell < a.ncells;
        int n = 0, y0 = 0, x0 = 0, ch = 0, cw = 0;
        double z = 0.0, m = 0.0;
        if (valid) {
            n = cell / G;
            const int g = cell - n * G, gy = g / a.Gw, gx = g - gy * a.Gw;
            y0 = gy * a.S;
            x0 = gx * a.S;
            ch = min(y0 + a.S, a.H) - y0;
            cw = min(x0 + a.S, a.W) - x0;
            for (int py = q; py < ch; py += 4) {  // rows q, q + 4, ...: a row's loads in flight first
                const float4 *row = a.mpart + (size_t)(n * a.H + y0 + py) * a.W + x0;
                for (int p0 = 0; p0 < cw; p0 += 8) {
                    float4 v[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        v[i] = p0 + i < cw ? ld_cg_f4(row + p0 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        z += (double)v[i].x + (double)v[i].z;
                        m += (double)v[i].y + (double)v[i].w;
                    }
                }
            }
        }
        z += __shfl_xor_sync(0xffffffffu, z, 1);
        m += __shfl_xor_sync(0xffffffffu, m, 1);
        z += __shfl_xor_sync(0xffffffffu, z, 2);
        m += __shfl_xor_sync(0xffffffffu, m, 2);
        if (valid && q == 0) {
            const double u32 = 5.9604644775390625e-8, u64 = 1.1102230246251565e-16;  // 2^-24, 2^-53
            const double n32 = (double)(a.c_in / 16 + 10), n64 = (double)(2 * ch * cw + 4);
            const double gam = n32 * u32 / (1.0 - n32 * u32) + n64 * u64 / (1.0 - n64 * u64);
            // m_p are fp32 sums (relative error <= c_in 2^-24 < 1e-3 for c_in < 16k): x1.01
            const double err = m * 1.01 * gam + 1e-300;
            z += (double)a.bm * (double)(ch * cw);
            int dec = 0;
            if (fabs(z) > err) dec = z > 0.0;
            else s_unc[atomicAdd(&s_nunc, 1)] = lc;
            s_dec[lc] = (uint8_t)dec;
        }
        __syncthreads();
        // fp64 re-sum of the undecided cells (rare), each by the whole CTA: one
        // load round trip per 1024 vectors instead of a warp's serial pixel loop
        for (int k = 0; k < s_nunc; ++k) {
            const int t = s_unc[k], c = cell0 + t;
            const int cn = c / G, g = c - cn * G, gy = g / a.Gw, gx = g - gy * a.Gw;
            const int cy0 = gy * a.S, cx0 = gx * a.S;
            const int cch = min(cy0 + a.S, a.H) - cy0, ccw = min(cx0 + a.S, a.W) - cx0;
            const double sum = cell_exact(a, cn, cy0, cx0, cch, ccw, s_red);
            if (tid == 0) s_dec[t] = (sum / (double)(cch * ccw) + (double)a.bm) > 0.0;
        }
        __syncthreads();
        // decisions out, one count per 32-cell group (warps 0 .. kDecCells/32 - 1)
        if (tid < kDecCells) {
            const int c = cell0 + tid;
            const int d = c < a.ncells ? s_dec[tid] : 0;
            if (c < a.ncells) a.dec[c] = (uint8_t)d;
            const unsigned bal = __ballot_sync(0xffffffffu, d);
            if (lane == 0 && cell0 / 32 + warp < a.ngroups) a.gpre[cell0 / 32 + warp] = __popc(bal);
        }
    }

    if constexpr (COOP) {
        // grid barrier, sense reversal: done[1] counts arrivals (reset by the last), done[2] is
        // the generation the last arrival advances (read before arriving; any start value)
        __syncthreads();
        if (tid == 0) {
            const unsigned gen = ld_acquire(a.done + 2);
            if (atom_add_acqrel(a.done + 1, 1u) == gridDim.x - 1) {
                a.done[1] = 0u;
                atom_add_acqrel(a.done + 2, 1u);
            } else {
                while (ld_acquire(a.done + 2) == gen) __nanosleep(64);
            }
        }
        __syncthreads();
        __shared__ int s_part[kDecThreads / 32], s_wcnt[kDecCells / 32];
        for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
            // the chunk's base: the active cells of all groups before its first one
            const int cell0 = chunk * kDecCells, g0 = cell0 / 32;
            int part = 0;
            for (int g = tid; g < g0; g += kDecThreads) {
                int v;
                asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(a.gpre + g));
                part += v;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if (lane == 0) s_part[warp] = part;
            int d = 0;
            unsigned bal = 0u;
            if (tid < kDecCells) {  // this CTA's own decisions of the chunk (written above)
                d = cell0 + tid < a.ncells ? a.dec[cell0 + tid] : 0;
                bal = __ballot_sync(0xffffffffu, d);
                if (lane == 0) s_wcnt[warp] = __popc(bal);
            }
            __syncthreads();
            int base = 0;
#pragma unroll
            for (int w = 0; w < kDecThreads / 32; ++w) base += s_part[w];
            if (tid < kDecCells) {
                int off = base;
                for (int w = 0; w < warp; ++w) off += s_wcnt[w];
                if (d) a.idx[off + __popc(bal & ((1u << lane) - 1u))] = cell0 + tid;
                // exclusive group prefixes for the gather (a separate array: other CTAs may
                // still be summing the counts)
                if (lane == 0 && g0 + warp < a.ngroups) a.gpx[g0 + warp] = off;
            }
            if (tid == 0 && chunk == nchunks - 1) {
                int tot = base;
                for (int w = 0; w < kDecCells / 32; ++w) tot += s_wcnt[w];
                *a.count = tot;
            }
            __syncthreads();  // s_part / s_wcnt are reused by the next chunk
        }
        return;
    }
    // the last CTA: exclusive prefix over the group counts, total count
    __syncthreads();
    if (tid == 0) s_last = atom_add_acqrel(a.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __shared__ int s_wsum[kDecThreads / 32];
    __shared__ int s_base;
    if (tid == 0) s_base = 0;
    __syncthreads();
    for (int g0 = 0; g0 < a.ngroups; g0 += kDecThreads) {
        const int g = g0 + tid;
        int v = 0;
        if (g < a.ngroups) asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(v) : "l"(a.gpre + g));
        int incl = v;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += t;
        }
        if (lane == 31) s_wsum[warp] = incl;
        __syncthreads();
        int woff = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kDecThreads / 32; ++w) {
            woff += w < warp ? s_wsum[w] : 0;
            tot += s_wsum[w];
        }
        if (g < a.ngroups) a.gpre[g] = s_base + woff + incl - v;
        __syncthreads();
        if (tid == 0) s_base += tot;
        __syncthreads();
    }
    if (tid == 0) {
        *a.count = s_base;
        *a.done = 0u;  // kernel completion orders this before the next launch
    }
}

struct GatherArgs {
    const uint8_t *dec;         // [ncells]
    const int32_t *gpre;        // [ngroups] exclusive prefixes
    int32_t *idx;
    const __nv_bfloat16 *h1d;   // dense h1 [c_mid/64][n][h][w][64]
    __nv_bfloat16 *h1g;         // gathered h1 [c_mid/64][cap][S+2][S+2][64]
    int n_img, H, W, S, Gh, Gw, ncells, ngroups, nch, cap;
};

// One warp per task (32-cell group g, 64-channel chunk cc, halo row hr).  Lane
// k first decodes the k-th active cell of the group into source/destination
// row bases (no division in the copy loop); then lane l copies 16-B vector
// w = l + 32 i (pixel w/8, part w%8) of that halo row for every active cell,
// 8 loads in flight before the stores.
__global__ void __launch_bounds__(256) compact_gather_kernel(const GatherArgs a) {
    __shared__ long s_src[8][32], s_dst[8][32];
    __shared__ int s_x0[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int hs = a.S + 2;
    pdl_wait();
    pdl_trigger();
    const long task = (long)blockIdx.x * 8 + wib;
    const long ntask = (long)a.ngroups * a.nch * hs;
    if (task >= ntask) return;
    const int g = (int)(task / (a.nch * hs));
    const int rem = (int)(task - (long)g * a.nch * hs);
    const int cc = rem / hs, hr = rem - cc * hs;
    const int cell = g * 32 + lane;
    const int d = cell < a.ncells ? a.dec[cell] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, d);
    if (bal == 0u) return;
    const int rank = __popc(bal & ((1u << lane) - 1u));
    if (d) {
        const int pos = a.gpre[g] + rank;
        if (cc == 0 && hr == 0) a.idx[pos] = cell;
        const int G = a.Gh * a.Gw;
        const int n = cell / G, gg = cell - n * G, gy = gg / a.Gw, gx = gg - gy * a.Gw;
        const int hy = gy * a.S - 1 + hr;
        const long pix_all = (long)a.n_img * a.H * a.W;
        // source: vector index of pixel (hy, gx*S) in chunk cc (halo pixel px is px - 1
        // from it); a row outside the image gets an x origin no pixel can pass
        const bool row_ok = hy >= 0 && hy < a.H;
        s_src[wib][rank] = (cc * pix_all + ((long)n * a.H + (row_ok ? hy : 0)) * a.W + gx * a.S) * 8;
        s_dst[wib][rank] = (((long)cc * a.cap + pos) * hs * hs + hr * hs) * 8;
        s_x0[wib][rank] = row_ok ? gx * a.S - 1 : -(1 << 30);
    }
    __syncwarp();
    const int nact = __popc(bal);
    const int per = hs * 8;  // vectors of one halo row of one cell
    const uint4 *src = reinterpret_cast<const uint4 *>(a.h1d);
    uint4 *dst = reinterpret_cast<uint4 *>(a.h1g);
    for (int w = lane; w < per; w += 32) {
        const int px = w >> 3;
        constexpr int kU = 8;
        for (int k0 = 0; k0 < nact; k0 += kU) {
            uint4 val[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                val[u] = make_uint4(0u, 0u, 0u, 0u);
                const int k = k0 + u;
                if (k < nact) {
                    const int hx = s_x0[wib][k] + px;
                    if (hx >= 0 && hx < a.W) val[u] = __ldg(src + s_src[wib][k] + w - 8);
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (k0 + u < nact) dst[s_dst[wib][k0 + u] + w] = val[u];
        }
    }
}

// Compaction only (the direct schedule, no gather): one warp per 32-cell group
// writes the ids of its active cells at the group's prefix.
__global__ void __launch_bounds__(256) compact_idx_kernel(const uint8_t *dec, const int32_t *gpre,
                                                          int32_t *__restrict__ idx, int ncells, int ngroups) {
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (g >= ngroups) return;
    const int cell = g * 32 + lane;
    const int d = cell < ncells ? dec[cell] : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, d);
    if (d) idx[gpre[g] + __popc(bal & ((1u << lane) - 1u))] = cell;
}

size_t decide_sync_bytes(int ncells, int) {
    // control words (16 B) + decisions (ncells) + group counts / prefixes + cooperative prefixes (ngroups ints each)
    const long ngroups = ((long)ncells + 31) / 32;
    return 16 + ((size_t)ncells + 15) / 16 * 16 + (size_t)ngroups * 8;
}

// sync: decide_sync_bytes() bytes whose first 16 are zero before the first call
// (words 0-1 are left zero; word 2 is a barrier generation of any value).
// h1d == nullptr: decisions, prefixes and count only; h1g == nullptr: + ids;
// else + ids and the halo gather of h1d into h1g.
cudaError_t launch_decide_gather(const float4 *mpart, const void *x, const float *wm, float bm, int n_img, int H,
                                 int W, int c_in, int S, uint8_t *mask, int32_t *idx, int32_t *count, void *sync,
                                 const void *h1d, void *h1g, int c_mid, int cap, int num_sms, cudaStream_t st,
                                 int *launched) {
    *launched = 1;
    (void)num_sms;
    DecideArgs a;
    a.mpart = mpart;
    a.x = static_cast<const __nv_bfloat16 *>(x);
    a.wm = wm;
    a.bm = bm;
    a.n_img = n_img;
    a.H = H;
    a.W = W;
    a.c_in = c_in;
    a.S = S;
    a.Gh = (H + S - 1) / S;
    a.Gw = (W + S - 1) / S;
    a.ncells = n_img * a.Gh * a.Gw;
    if (a.ncells == 0) return cudaMemsetAsync(count, 0, sizeof(int32_t), st);
    a.ngroups = (a.ncells + 31) / 32;
    uint8_t *base = static_cast<uint8_t *>(sync);
    a.done = reinterpret_cast<unsigned *>(base);
    uint8_t *decs = base + 16;
    a.dec = mask ? mask : decs;
    a.gpre = reinterpret_cast<int32_t *>(decs + ((size_t)a.ncells + 15) / 16 * 16);
    a.count = count;
    a.idx = idx;
    const int grid = (a.ncells + kDecCells - 1) / kDecCells;
    // ids-only with every CTA co-resident: one cooperative launch (LASNET_DECIDE_2K=1: two launches).
    // The co-residency capacity is measured per device; the launch itself carries the
    // cooperative attribute, so the runtime refuses it (nothing runs) rather than let a
    // grid barrier spin on CTAs that cannot be scheduled -- then the two-launch path runs.
    static const bool two_k = [] {
        const char *e = getenv("LASNET_DECIDE_2K");
        return e && e[0] == '1';
    }();
    constexpr int kMaxDev = 64;
    static int coop_cap_dev[kMaxDev] = {};  // 0 = not measured yet, -1 = unavailable
    int dev = 0;
    cudaGetDevice(&dev);
    int coop_cap = 0;
    if (!two_k && dev >= 0 && dev < kMaxDev) {
        if (coop_cap_dev[dev] == 0) {
            int per_sm = 0, sms = 0, coop_ok = 0;
            cudaDeviceGetAttribute(&coop_ok, cudaDevAttrCooperativeLaunch, dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            if (coop_ok &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decide_kernel<true>, kDecThreads, 0) == cudaSuccess &&
                per_sm * sms > 0)
                coop_cap_dev[dev] = per_sm * sms;
            else
                coop_cap_dev[dev] = -1;
        }
        coop_cap = coop_cap_dev[dev] > 0 ? coop_cap_dev[dev] : 0;
    }
    a.gpx = a.gpre + a.ngroups;
    // the cooperative grid is capped at the co-residency capacity (a CTA then takes several chunks)
    bool coop = h1d != nullptr && coop_cap > 0;
    cudaError_t e = cudaErrorUnknown;
    if (coop) {
        e = launch_k_coop(decide_kernel<true>, dim3(grid < coop_cap ? grid : coop_cap), dim3(kDecThreads), 0, st, a);
        if (e == cudaErrorCooperativeLaunchTooLarge) {  // not co-resident now: the two-launch form
            (void)cudaGetLastError();
            coop = false;
        }
    }
    if (!coop) e = launch_k(decide_kernel<false>, dim3(grid), dim3(kDecThreads), 0, st, a);
    if (e != cudaSuccess || h1d == nullptr || (coop && h1g == nullptr)) return e;
    *launched = 2;
    if (h1g == nullptr)  // ids only: steps 4-5 read the dense h1 directly
        return launch_k(compact_idx_kernel, dim3((unsigned)((a.ngroups + 7) / 8)), dim3(256), 0, st,
                        static_cast<const uint8_t *>(a.dec), static_cast<const int32_t *>(a.gpre), idx, a.ncells,
                        a.ngroups);
    GatherArgs g;
    g.dec = a.dec;
    g.gpre = coop ? a.gpx : a.gpre;  // exclusive prefixes
    g.idx = idx;
    g.h1d = static_cast<const __nv_bfloat16 *>(h1d);
    g.h1g = static_cast<__nv_bfloat16 *>(h1g);
    g.n_img = n_img;
    g.H = H;
    g.W = W;
    g.S = S;
    g.Gh = a.Gh;
    g.Gw = a.Gw;
    g.ncells = a.ncells;
    g.ngroups = a.ngroups;
    g.nch = c_mid / 64;
    g.cap = cap;
    const long ntask = (long)a.ngroups * g.nch * (S + 2);
    return launch_k(compact_gather_kernel, dim3((unsigned)((ntask + 7) / 8)), dim3(256), 0, st, g);
}

}  // namespace lasnet

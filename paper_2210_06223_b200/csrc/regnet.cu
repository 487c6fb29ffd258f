// regnet.cu -- the kernels the LAS-RegNetY Y-block needs beyond the ResNet
// bottleneck's ("bottleneck structure with different
// channel numbers and convolution groups ... equipped with Squeeze-and-Excitation"):
//
//   gconv_kernel      grouped 3x3 (group width 16), bias, ReLU, bf16: on the gathered
//                     (S+2)^2 windows of the active patches (dynamic block, valid conv,
//                     P:163-166) or on a dense map (static block, zero padding 1,
//                     stride 1 or 2).  Per group the contraction is only 144 deep and 16
//                     wide, so it runs on warp-level mma.sync m16n8k16 (bf16 x bf16 ->
//                     fp32) rather than 128-row tcgen05 tiles: a warp owns 16 output
//                     rows and walks all groups, nine taps x two 8-wide halves each.
//   se_kernel         squeeze-and-excitation per image: the mean of h2 over the image's
//                     computed pixels (its ACTIVE in-image pixels in a dynamic block,
//                     reading R23), then s = sigmoid(W2 ReLU(W1 p + b1) + b2); one CTA
//                     per image, fixed summation order (deterministic).
//   se_apply_kernel   h2 <- rnd(h2 * s[image]) in place, 16-B vectors.
//   regnet_stem_kernel the RegNet stem: 3x3 stride-2 conv 3 -> 32 channels + bias +
//                     ReLU (zero channels 32..63 for the 64-wide K-blocks downstream).
// Layouts: h1 channel-chunk-major [C/64][rows][64] (what conv_tc's conv1 stores);
// h2 row-major [rows][C]; weights wb [C][3][3][16] (OHWI within the group).
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "regnet.cuh"

namespace lasnet {

__device__ __forceinline__ uint32_t ldg_u32(const __nv_bfloat16 *p) {
    return __ldg(reinterpret_cast<const uint32_t *>(p));
}

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Grouped 3x3, one CTA (8 warps) per tile of up to 128 output rows.  Per 64-channel
// chunk (4 groups) the tile's input rows are staged in shared memory with cp.async
// (16-B pieces XOR-swizzled by row, zero-filled outside the image) together with the
// chunk's weights; each warp then runs 16 output rows x 4 groups x 9 taps x 2
// halves of mma.sync m16n8k16, its A fragments loaded by ldmatrix.x4 from the
// tap-shifted input rows.  Dynamic: a tile is upt whole patches, whose (S+2)^2
// windows are one contiguous range of gathered rows; dense: a tile is trows whole
// output rows of one image, staged with their halo (stride 1 or 2, padding 1).
constexpr int kGcThreads = 256;
constexpr int kGcMaxIn = 576;  // staged input rows per chunk (72 KB: two CTAs per SM)

template <bool DYN>
__global__ void __launch_bounds__(kGcThreads, 2) gconv_kernel(const GconvArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(128) uint8_t gsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    uint8_t *s_in = gsm;                                    // [in_rows][128 B] swizzled
    __nv_bfloat16 *s_w = reinterpret_cast<__nv_bfloat16 *>(gsm + kGcMaxIn * 128);  // [64][9][16]
    int *s_src = reinterpret_cast<int *>(gsm + kGcMaxIn * 128 + 64 * 9 * 16 * 2);  // [128][9] staged row per tap
    int *s_pn = s_src + 128 * 9, *s_py = s_pn + 128, *s_px = s_py + 128;         // direct: window origin per patch
    // ---- tile geometry ----
    int rows, in_rows;
    int64_t out_row0;
    int64_t in_row0 = 0;  // dynamic: first gathered row of the tile
    int n0 = 0, oy0 = 0, iy0 = 0, ih = 0, iw = 0;  // dense: image, first output row, staged input box
    if (DYN) {
        const int upt = a.upt;
        const int cnt = *a.count;
        const int t0 = blockIdx.x * upt;
        if (t0 >= cnt) return;
        const int np = min(upt, cnt - t0);
        rows = np * a.S * a.S;
        out_row0 = (int64_t)t0 * a.S * a.S;
        in_row0 = (int64_t)t0 * a.hs * a.hs;
        in_rows = np * a.hs * a.hs;
        if (a.direct)  // window origin (image, y, x) of each patch of the tile, from its cell id
            for (int p = threadIdx.x; p < np; p += kGcThreads) {
                const int c = __ldcg(a.idx + t0 + p), n = c / a.G, g = c - n * a.G, gy = g / a.Gw;
                s_pn[p] = n;
                s_py[p] = gy * a.S - 1;
                s_px[p] = (g - gy * a.Gw) * a.S - 1;
            }
    } else {
        const int bands = (a.Ho + a.trows - 1) / a.trows;
        n0 = blockIdx.x / bands;
        if (n0 >= a.n_img) return;
        oy0 = (blockIdx.x - n0 * bands) * a.trows;
        const int nr = min(a.trows, a.Ho - oy0);
        rows = nr * a.Wo;
        out_row0 = ((int64_t)n0 * a.Ho + oy0) * a.Wo;
        iy0 = a.stride * oy0 - 1;
        ih = a.stride * (nr - 1) + 3;
        iw = a.stride * (a.Wo - 1) + 3;
        in_rows = ih * iw;
    }
    // staged row of (output row r, tap t)
    for (int e = threadIdx.x; e < 128 * 9; e += kGcThreads) {
        const int r = e / 9, t = e - r * 9, dy = t / 3, dx = t - dy * 3;
        int sr = 0;
        if (r < rows) {
            if (DYN) {
                const int ss = a.S * a.S, p = r / ss, j = r - p * ss, py = j / a.S, px = j - py * a.S;
                sr = p * a.hs * a.hs + (py + dy) * a.hs + (px + dx);
            } else {
                const int oy = r / a.Wo, ox = r - oy * a.Wo;
                sr = (a.stride * oy + dy) * iw + (a.stride * ox + dx);
            }
        }
        s_src[e] = sr;
    }
    const int wr0 = warp * 16;  // this warp's first output row of the tile
    const int groups_total = a.C / 16;
    for (int ch = 0; ch < a.C / 64; ++ch) {
        __syncthreads();  // previous chunk's smem reads done (and s_src written)
        // stage the input rows of this chunk: 8 x 16-B pieces per row, piece k at k ^ (row & 7)
        const __nv_bfloat16 *src_chunk = a.h1 + (int64_t)ch * a.h1_rows * 64;
        for (int e = threadIdx.x; e < in_rows * 8; e += kGcThreads) {
            const int row = e >> 3, k = e & 7;
            const uint32_t dst = smem_addr(s_in + row * 128 + ((k ^ (row & 7)) << 4));
            const __nv_bfloat16 *g = src_chunk;
            uint32_t bytes = 16;
            if (DYN && a.direct) {  // window pixel (wy, wx) of patch p, read from the dense h1
                const int hs2 = a.hs * a.hs, p = row / hs2, j = row - p * hs2, wy = j / a.hs;
                const int yy = s_py[p] + wy, xx = s_px[p] + (j - wy * a.hs);
                if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
                    g = src_chunk + (((int64_t)s_pn[p] * a.H + yy) * a.W + xx) * 64 + k * 8;
                else
                    bytes = 0;  // conv2's zero padding outside the image (R6)
            } else if (DYN) {
                g = src_chunk + (in_row0 + row) * 64 + k * 8;
            } else {
                const int yy = iy0 + row / iw, xx = row - (row / iw) * iw - 1;
                if (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W)
                    g = src_chunk + (((int64_t)n0 * a.H + yy) * a.W + xx) * 64 + k * 8;
                else
                    bytes = 0;  // zero padding
            }
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(g), "r"(bytes) : "memory");
        }
        // the chunk's weights [64 out][9][16]
        const __nv_bfloat16 *wsrc = a.wb + (int64_t)ch * 64 * 9 * 16;
        for (int e = threadIdx.x; e < 64 * 9 * 16 / 8; e += kGcThreads)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(s_w + e * 8)), "l"(wsrc + e * 8)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();
        if (wr0 >= rows) continue;
        // ldmatrix.x4 lane roles: matrix m = lane / 8 (rows 0-7 / 8-15, k 0-7 / 8-15)
        const int lr = (lane & 7) + ((lane >> 3) & 1) * 8;  // A row of this lane's address
        const int khalf = lane >> 4;                        // 0: k 0-7, 1: k 8-15
        for (int gl = 0; gl < 4; ++gl) {
            const int g = ch * 4 + gl;
            if (g >= groups_total) break;
            float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int sr = s_src[(wr0 + lr) * 9 + t];
                const int piece = (gl * 2 + khalf) ^ (sr & 7);
                const uint32_t addr = smem_addr(s_in + sr * 128 + (piece << 4));
                uint32_t af[4];
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                             : "=r"(af[0]), "=r"(af[1]), "=r"(af[2]), "=r"(af[3])
                             : "r"(addr));
#pragma unroll
                for (int nh = 0; nh < 2; ++nh) {
                    const __nv_bfloat16 *wp = s_w + ((gl * 16 + nh * 8 + gq) * 9 + t) * 16 + 2 * tq;
                    const uint32_t b0 = *reinterpret_cast<const uint32_t *>(wp);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t *>(wp + 8);
                    asm volatile(
                        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                        "{%0,%1,%2,%3};"
                        : "+f"(acc[nh][0]), "+f"(acc[nh][1]), "+f"(acc[nh][2]), "+f"(acc[nh][3])
                        : "r"(af[0]), "r"(af[1]), "r"(af[2]), "r"(af[3]), "r"(b0), "r"(b1));
                }
            }
#pragma unroll
            for (int nh = 0; nh < 2; ++nh) {
                const int c = g * 16 + nh * 8 + 2 * tq;
                const float b0 = __ldg(a.bias + c), b1 = __ldg(a.bias + c + 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = wr0 + gq + 8 * h;
                    if (r < rows) {
                        const __nv_bfloat162 v = __floats2bfloat162_rn(fmaxf(acc[nh][2 * h] + b0, 0.f),
                                                                       fmaxf(acc[nh][2 * h + 1] + b1, 0.f));
                        *reinterpret_cast<__nv_bfloat162 *>(a.h2 + (out_row0 + r) * a.C + c) = v;
                    }
                }
            }
        }
    }
}

// One CTA (256 threads) per image.  Dynamic: the image's patches are the contiguous
// idx range of its cell ids (ascending); only in-image output pixels are pooled.
// Pooling: thread (slice rs, vector v) sums 8 channels (one 16-B load per row) of
// rows rs, rs + RS, ... in order; the RS slice partials are then added in slice
// order per channel -- a fixed summation tree (deterministic).
constexpr int kSeThreads = 256;
__global__ void __launch_bounds__(kSeThreads) se_kernel(const SeArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ float sm[];
    const int cv = a.C / 8;
    const int RS = cv >= kSeThreads ? 1 : kSeThreads / cv;  // row slices
    float *part = sm;                  // [RS][C]
    float *pooled = nullptr, *z = nullptr;
    __shared__ int range[2];
    __shared__ int npix_s[kSeThreads];
    const int n = blockIdx.x;
    int t0 = 0, t1 = 0;
    if (a.count) {
        // the image's patches [t0, t1) in the ascending ids: the first id of image >= n and >= n + 1,
        // found by the whole CTA in two probe rounds (256 evenly spaced positions, then every
        // position between the two bracketing probes) instead of a one-thread binary search
        // (~28 dependent L2 round trips)
        __shared__ int s_lo[2], s_hi[2];
        const int cnt = __ldcg(a.count);
        if (threadIdx.x < 2) {
            s_lo[threadIdx.x] = 0;
            s_hi[threadIdx.x] = cnt;
        }
        __syncthreads();
        {
            const long p = (long)cnt * threadIdx.x / kSeThreads;  // round 1: evenly spaced probes
            const int img = p < cnt ? __ldcg(a.idx + p) / a.G : 0x7fffffff;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                if (p < cnt && img < n + b) atomicMax(&s_lo[b], (int)p);  // last probe below the bound
                if (p < cnt && img >= n + b) atomicMin(&s_hi[b], (int)p);  // first probe at or above it
            }
        }
        __syncthreads();
        __shared__ int s_first[2];
        if (threadIdx.x < 2) s_first[threadIdx.x] = s_hi[threadIdx.x];
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 2; ++b) {  // round 2: every position of the bracket (< cnt / 256 + 1 of them)
            for (int p = s_lo[b] + (int)threadIdx.x; p < s_hi[b]; p += kSeThreads)
                if (__ldcg(a.idx + p) / a.G >= n + b) atomicMin(&s_first[b], p);
        }
        __syncthreads();
        t0 = s_first[0];
        t1 = s_first[1];
        if (t0 == t1) return;  // no active cell: the block leaves the image untouched
    }
    const int ss = a.S * a.S;
    const int64_t row0 = a.count ? (int64_t)t0 * ss : (int64_t)n * a.HW;
    const int nrows = a.count ? (t1 - t0) * ss : a.HW;
    const int rs = threadIdx.x / cv, v = threadIdx.x - rs * cv;
    int np = 0;
    if (rs < RS) {
        for (int vv = v; vv < cv; vv += (RS == 1 ? kSeThreads : cv)) {
            float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            int cntp = 0;
            // the thread's rows r = rs, rs + RS, ... eight at a time: their id loads, then their
            // h2 loads, are in flight together (one round trip each per 8 rows instead of per
            // row); the sums still run in row order (bitwise the row-by-row loop)
            constexpr int kU = 8;
            for (int rb = rs; rb < nrows; rb += kU * RS) {
                bool ok[kU];
                int cellv[kU];
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    const int r = rb + k * RS;
                    ok[k] = r < nrows;
                    cellv[k] = 0;
                    if (a.count && ok[k]) cellv[k] = __ldcg(a.idx + t0 + r / ss);
                }
                uint4 q[kU];
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    const int r = rb + k * RS;
                    if (a.count && ok[k]) {  // clipped edge cells: only in-image pixels
                        const int j = r - (r / ss) * ss, cell = cellv[k] - n * a.G;
                        const int gy = cell / a.Gw, gx = cell - gy * a.Gw;
                        const int py = j / a.S, px = j - py * a.S;
                        ok[k] = gy * a.S + py < a.H && gx * a.S + px < a.W;
                    }
                    q[k] = ok[k] ? __ldca(reinterpret_cast<const uint4 *>(a.h2 + (row0 + r) * a.C) + vv)  // (PDL)
                                 : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    if (!ok[k]) continue;
                    const uint32_t u[4] = {q[k].x, q[k].y, q[k].z, q[k].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        acc[2 * e] += __uint_as_float(u[e] << 16);
                        acc[2 * e + 1] += __uint_as_float(u[e] & 0xffff0000u);
                    }
                    ++cntp;
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) part[rs * a.C + 8 * vv + e] = acc[e];
            np = cntp;
        }
    }
    npix_s[threadIdx.x] = (rs < RS && v == 0) ? np : 0;
    __syncthreads();
    if (threadIdx.x == 0) {  // pixels pooled: the slices of vector 0, in order
        int t = 0;
        for (int k = 0; k < RS; ++k) t += npix_s[k * cv];
        range[0] = t;
    }
    __syncthreads();
    const float inv = 1.f / (float)range[0];
    for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
        float s = 0.f;
        for (int k = 0; k < RS; ++k) s += part[k * a.C + c];
        a.pooled[(int64_t)n * a.C + c] = s * inv;
    }
    (void)pooled;
    (void)z;
}

// The excitation of all images at once, two small fp32 GEMMs (se_fc_kernel twice):
// out[n][j] = act(b[j] + sum_k in[n][k] w[j][k]), act = ReLU (W1) or sigmoid (W2);
// one CTA per 32 images x 32 outputs, K staged in 64-wide chunks, fixed-order sums.
// Images without active cells (a dynamic block) are skipped (their scale is unused).
__global__ void __launch_bounds__(256) se_fc_kernel(const float *in, const float *__restrict__ w,
                                                    const float *__restrict__ b, float *__restrict__ out, int n_img,
                                                    int K, int N, int sigmoid_act) {
    pdl_wait();
    pdl_trigger();
    __shared__ float sa[32][65], sb[32][65];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int j0 = blockIdx.x * 32, n0 = blockIdx.y * 32;
    float acc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
    for (int k0 = 0; k0 < K; k0 += 64) {
        for (int e = threadIdx.x; e < 32 * 64; e += 256) {
            const int r = e / 64, kk = e % 64, k = k0 + kk;
            sa[r][kk] = (n0 + r < n_img && k < K) ? in[(int64_t)(n0 + r) * K + k] : 0.f;
            sb[r][kk] = (j0 + r < N && k < K) ? w[(int64_t)(j0 + r) * K + k] : 0.f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < 64; ++kk) {
            const float a0 = sa[ty][kk], a1 = sa[ty + 16][kk], b0 = sb[tx][kk], b1 = sb[tx + 16][kk];
            acc[0][0] = fmaf(a0, b0, acc[0][0]);
            acc[0][1] = fmaf(a0, b1, acc[0][1]);
            acc[1][0] = fmaf(a1, b0, acc[1][0]);
            acc[1][1] = fmaf(a1, b1, acc[1][1]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
            const int n = n0 + ty + 16 * i, j = j0 + tx + 16 * jj;
            if (n < n_img && j < N) {
                const float v = acc[i][jj] + b[j];
                out[(int64_t)n * N + j] = sigmoid_act ? 1.f / (1.f + __expf(-v)) : fmaxf(v, 0.f);
            }
        }
}

// h2[row][:] *= scale[image(row)][:] (bf16 RNE), 8 channels per thread
__global__ void __launch_bounds__(256) se_apply_kernel(__nv_bfloat16 *h2, const float *scale, const int32_t *idx,
                                                       const int32_t *count, int rows_dense, int C, int S, int G,
                                                       int HW) {
    pdl_wait();
    pdl_trigger();
    const int ss = S * S;
    const int rows = count ? (*count) * ss : rows_dense;
    const int cv = C / 8;
    const int64_t total = (int64_t)rows * cv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / cv), v = (int)(i - (int64_t)r * cv);
        const int n = count ? __ldcg(idx + r / ss) / G : r / HW;
        uint4 *p = reinterpret_cast<uint4 *>(h2 + (int64_t)r * C) + v;
        uint4 q = *p;
        uint32_t u[4] = {q.x, q.y, q.z, q.w};
        const float *sc = scale + (int64_t)n * C + 8 * v;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float lo = __uint_as_float(u[e] << 16) * sc[2 * e];
            const float hi = __uint_as_float(u[e] & 0xffff0000u) * sc[2 * e + 1];
            const __nv_bfloat162 b = __floats2bfloat162_rn(lo, hi);
            u[e] = *reinterpret_cast<const uint32_t *>(&b);
        }
        *p = make_uint4(u[0], u[1], u[2], u[3]);
    }
}

// RegNet stem: x_pad [n][2h][2w + 8][8] (image at column offset 4, channels 3..7 zero),
// w [64][3][3][8] OHWI, b [64] -> y [n][h][w][64]; one thread per PAIR of horizontally
// adjacent output pixels (every weight read from shared memory feeds two pixels).
__global__ void __launch_bounds__(128) regnet_stem_kernel(const __nv_bfloat16 *__restrict__ x,
                                                          const __nv_bfloat16 *__restrict__ w,
                                                          const float *__restrict__ b, __nv_bfloat16 *__restrict__ y,
                                                          int n_img, int h, int wo, int co_real) {
    pdl_wait();
    pdl_trigger();
    __shared__ float2 ws[27][32];  // (channel 2j, 2j+1) pairs
    __shared__ float bs[64];
    for (int i = threadIdx.x; i < 27 * 64; i += blockDim.x) {
        const int o = i % 64, k = i / 64, t = k / 3, c = k % 3;
        reinterpret_cast<float *>(&ws[k][0])[o] = __bfloat162float(w[(o * 9 + t) * 8 + c]);
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) bs[i] = b[i];
    __syncthreads();
    const int hi = 2 * h, wp = 2 * wo + 8;
    const int wq = (wo + 1) / 2;  // pixel pairs per row
    const int64_t total = (int64_t)n_img * h * wq;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total; p += (int64_t)gridDim.x * blockDim.x) {
        const int oq = (int)(p % wq);
        const int64_t q = p / wq;
        const int oy = (int)(q % h), n = (int)(q / h);
        const int ox0 = 2 * oq;
        const bool two = ox0 + 1 < wo;
        float xin[2][27];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int iy = 2 * oy + t / 3 - 1;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int ix = 2 * (ox0 + u) + t % 3 - 1;  // padded column ix + 4
                uint4 v = make_uint4(0, 0, 0, 0);
                if (iy >= 0 && iy < hi && (u == 0 || two))
                    v = __ldg(reinterpret_cast<const uint4 *>(x + (((int64_t)n * hi + iy) * wp + ix + 4) * 8));
                xin[u][3 * t] = __uint_as_float(v.x << 16);
                xin[u][3 * t + 1] = __uint_as_float(v.x & 0xffff0000u);
                xin[u][3 * t + 2] = __uint_as_float(v.y << 16);
            }
        }
        uint32_t o32[2][32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int o = 2 * j;
            float s[2][2];
            const float bb0 = o < co_real ? bs[o] : 0.f, bb1 = o < co_real ? bs[o + 1] : 0.f;
            s[0][0] = s[1][0] = bb0;
            s[0][1] = s[1][1] = bb1;
            if (o < co_real) {
#pragma unroll
                for (int k = 0; k < 27; ++k) {
                    const float2 wv = ws[k][j];
                    s[0][0] = fmaf(wv.x, xin[0][k], s[0][0]);
                    s[0][1] = fmaf(wv.y, xin[0][k], s[0][1]);
                    s[1][0] = fmaf(wv.x, xin[1][k], s[1][0]);
                    s[1][1] = fmaf(wv.y, xin[1][k], s[1][1]);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const __nv_bfloat162 v = __floats2bfloat162_rn(fmaxf(s[u][0], 0.f), fmaxf(s[u][1], 0.f));
                o32[u][j] = *reinterpret_cast<const uint32_t *>(&v);
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u == 1 && !two) break;
            uint4 *yp = reinterpret_cast<uint4 *>(y + (((int64_t)n * h + oy) * wo + ox0 + u) * 64);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                yp[k] = make_uint4(o32[u][4 * k], o32[u][4 * k + 1], o32[u][4 * k + 2], o32[u][4 * k + 3]);
        }
    }
}

// ----------------------------------------------------------------- host ----

// Tile geometry of gconv_kernel: dynamic -- upt patches per tile (whole patches of
// at most 128 output rows); dense -- trows output rows of one image whose staged
// input box fits kGcMaxIn rows.  Returns the grid size (0: nothing to do, -1: no fit).
long gconv_tiles(bool dyn, GconvArgs &a, int max_rows) {
    if (dyn) {
        a.upt = 128 / (a.S * a.S);
        while (a.upt > 1 && a.upt * a.hs * a.hs > kGcMaxIn) --a.upt;
        if (a.upt < 1 || a.upt * a.hs * a.hs > kGcMaxIn) return -1;
        const long cap = max_rows / (a.S * a.S);
        return (cap + a.upt - 1) / a.upt;
    }
    a.trows = a.Wo > 128 ? 0 : 128 / a.Wo;
    if (a.trows > a.Ho) a.trows = a.Ho;
    while (a.trows > 0 && (a.stride * (a.trows - 1) + 3) * (a.stride * (a.Wo - 1) + 3) > kGcMaxIn) --a.trows;
    if (a.trows < 1) return -1;
    return (long)a.n_img * ((a.Ho + a.trows - 1) / a.trows);
}

cudaError_t launch_gconv(bool dyn, const GconvArgs &a0, int max_rows, int num_sms, cudaStream_t st) {
    (void)num_sms;
    GconvArgs a = a0;
    const long grid = gconv_tiles(dyn, a, max_rows);
    if (grid < 0) return cudaErrorInvalidValue;
    if (grid == 0) return cudaSuccess;
    const int smem = kGcMaxIn * 128 + 64 * 9 * 16 * 2 + 128 * 9 * 4 + 3 * 128 * 4;
    static bool configured[2] = {false, false};
    if (!configured[dyn]) {
        cudaError_t e = cudaFuncSetAttribute(dyn ? (const void *)gconv_kernel<true> : (const void *)gconv_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured[dyn] = true;
    }
    return dyn ? launch_k(gconv_kernel<true>, dim3((unsigned)grid), dim3(kGcThreads), smem, st, a)
               : launch_k(gconv_kernel<false>, dim3((unsigned)grid), dim3(kGcThreads), smem, st, a);
}

cudaError_t launch_se(const SeArgs &a, cudaStream_t st) {
    if (a.n_img == 0) return cudaSuccess;
    const int cv = a.C / 8;
    const int RS = cv >= kSeThreads ? 1 : kSeThreads / cv;
    const size_t smem = (size_t)RS * a.C * 4;
    static size_t configured = 48 * 1024;
    if (smem > configured) {
        if (cudaFuncSetAttribute(se_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return cudaErrorInvalidValue;
        configured = smem;
    }
    cudaError_t e = launch_k(se_kernel, dim3((unsigned)a.n_img), dim3(kSeThreads), smem, st, a);
    if (e != cudaSuccess) return e;
    // z = ReLU(pooled W1^T + b1), then scale = sigmoid(z W2^T + b2)
    const dim3 g1((unsigned)((a.w_se + 31) / 32), (unsigned)((a.n_img + 31) / 32));
    e = launch_k(se_fc_kernel, g1, dim3(256), 0, st, static_cast<const float *>(a.pooled), a.w1, a.b1, a.z, a.n_img,
                 a.C, a.w_se, 0);
    if (e != cudaSuccess) return e;
    const dim3 g2((unsigned)((a.C + 31) / 32), (unsigned)((a.n_img + 31) / 32));
    return launch_k(se_fc_kernel, g2, dim3(256), 0, st, static_cast<const float *>(a.z), a.w2, a.b2, a.scale,
                    a.n_img, a.w_se, a.C, 1);
}

cudaError_t launch_se_apply(__nv_bfloat16 *h2, const float *scale, const int32_t *idx, const int32_t *count,
                            int max_rows, int C, int S, int G, int HW, int num_sms, cudaStream_t st) {
    const long total = (long)max_rows * (C / 8);
    long grid = (total + 255) / 256;
    if (grid > 8L * num_sms) grid = 8L * num_sms;
    if (grid == 0) return cudaSuccess;
    return launch_k(se_apply_kernel, dim3((unsigned)grid), dim3(256), 0, st, h2, scale, idx, count, max_rows, C, S,
                    G, HW);
}

cudaError_t launch_regnet_stem(const void *x, const void *w, const float *b, void *y, int n_img, int h, int wo,
                               int co_real, int num_sms, cudaStream_t st) {
    const long total = (long)n_img * h * ((wo + 1) / 2);
    long grid = (total + 127) / 128;
    if (grid > 16L * num_sms) grid = 16L * num_sms;
    if (grid == 0) return cudaSuccess;
    return launch_k(regnet_stem_kernel, dim3((unsigned)grid), dim3(128), 0, st, static_cast<const __nv_bfloat16 *>(x),
                    static_cast<const __nv_bfloat16 *>(w), b, static_cast<__nv_bfloat16 *>(y), n_img, h, wo, co_real);
}

}  // namespace lasnet

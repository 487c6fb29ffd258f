// mask_compact.cu -- steps 1 and 2 of the LASNet block.
//
// Step 1, masker (P:109 pooling + 1x1 conv; App. B P:560-563 2->1 channel
// reduction): one warp per coarse cell; lanes own 16-byte NHWC channel vectors
// (a warp reads 512 contiguous bytes of a pixel per instruction), 8 loads per
// lane in flight.  sum_p sum_c w_c x[p,c] accumulates in fp64 with exact
// products (bf16 x fp32 fits a double), then a warp shuffle reduction;
// logit = sum / |Omega| + b, decision logit > 0.  HBM-bound: every x byte once.
// The fused variant (bottom) also does step 2 in the same launch.
//
// Step 2, compaction (App. B): single-pass stream compaction with
// decoupled look-back.  Each 256-thread CTA owns 4096 cells (16 per thread,
// one uint4 load), scans them with warp ballots/shuffles, publishes its
// aggregate, looks back over predecessors 32 at a time, and writes ascending
// cell ids.  The last tile writes the device count.
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"

namespace lasnet {

// ---------------------------------------------------------------- masker ---

// bf16 bits -> the exact double, with integer ops (normal numbers) -- keeps the
// F2F conversion pipe out of the hot loop; zero/subnormal/inf/nan via the slow path.
__device__ __forceinline__ double bf16_to_f64(uint32_t b) {
    const uint32_t e = (b >> 7) & 0xFFu;
    if (__builtin_expect(e == 0u || e == 0xFFu, 0)) return (double)__uint_as_float(b << 16);
    const unsigned long long bits = ((unsigned long long)(b & 0x8000u) << 48) |
                                    ((unsigned long long)(e + 896u) << 52) | ((unsigned long long)(b & 0x7Fu) << 45);
    return __longlong_as_double((long long)bits);
}

template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
    static constexpr int kPerVec = 8;
    __device__ static void fma8(const uint4 &v, const float *w, double &acc) {
        const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc = fma((double)w[2 * i], bf16_to_f64(q[i] & 0xFFFFu), acc);
            acc = fma((double)w[2 * i + 1], bf16_to_f64(q[i] >> 16), acc);
        }
    }
    __device__ static void ffma8(const uint4 &v, const float *w, float &acc, float &mag) {
        const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float lo = __uint_as_float(q[i] << 16), hi = __uint_as_float(q[i] & 0xFFFF0000u);
            acc = fmaf(w[2 * i], lo, acc);
            acc = fmaf(w[2 * i + 1], hi, acc);
            mag = fmaf(fabsf(w[2 * i]), fabsf(lo), mag);  // |.| are free operand modifiers
            mag = fmaf(fabsf(w[2 * i + 1]), fabsf(hi), mag);
        }
    }
};
template <> struct Elem<float> {
    static constexpr int kPerVec = 4;
    __device__ static void fma8(const uint4 &v, const float *w, double &acc) {
        acc = fma((double)w[0], (double)__uint_as_float(v.x), acc);
        acc = fma((double)w[1], (double)__uint_as_float(v.y), acc);
        acc = fma((double)w[2], (double)__uint_as_float(v.z), acc);
        acc = fma((double)w[3], (double)__uint_as_float(v.w), acc);
    }
    __device__ static void ffma8(const uint4 &v, const float *w, float &acc, float &mag) {
        const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc = fmaf(w[i], f[i], acc);
            mag = fmaf(fabsf(w[i]), fabsf(f[i]), mag);
        }
    }
};

// Masker geometry (host-computed).  A cell's work is split into "items": one
// 16-byte channel vector per lane for one pixel (nvec >= 32 vectors per pixel:
// item = (pixel, vector slot), lane l reads vector 32*slot + l), or, for narrow
// pixels (nvec < 32), one vector of each of ppw = 32/nvec pixels.  A group of
// wpc warps shares one cell and each warp issues all of its <= 16 loads at
// once, so every warp needs a single memory round trip; cpb = 8/wpc cells per
// 256-thread CTA.  <= 64 registers keep 4 CTAs (32 warps) per SM resident.
struct MaskGeo {
    int nvec;  // 16-B vectors per pixel
    int ppw;   // pixels per item (nvec < 32), else 1
    int nvl;   // vector slots per pixel (nvec >= 32), else 1
    int wpc;   // warps per cell (1, 2, 4, 8)
    int cpb;   // cells per CTA = 8 / wpc
};

constexpr int kMaskThreads = 256;
constexpr int kMaxItems = 8;  // loads in flight per lane

// Partial sum of this warp's pixels of cell (n, gy, gx).  EXACT: fp64 with exact
// products (bf16 x fp32 fits a double).  Otherwise fp32 FFMA plus sum|w x| and
// the longest addition chain for the error bound (Higham: |fl(s)-s| <= gamma_n sum|terms|).
// Warp k of the cell's group takes pixels p0, p0 + pstride, ...; each pixel is
// SLOTS 16-B vectors per lane (wide pixels) or one vector (narrow pixels).  The
// pixel walk is incremental (no integer division in the loop) and every lane
// issues up to 8 loads before consuming any.
template <typename T, bool EXACT, int SLOTS>
__device__ __forceinline__ void warp_items_s(const T *__restrict__ x, const float *__restrict__ wm, const MaskGeo &mg,
                                             int H, int W, int C, int S, int n, int gy, int gx, int k, int lane,
                                             double &dacc, float &facc, float &fmag, int &nterms) {
    constexpr int PV = Elem<T>::kPerVec;
    constexpr int PPC = kMaxItems / SLOTS;  // pixels per chunk
    const int y0 = gy * S, x0 = gx * S;
    const int cw = min(x0 + S, W) - x0;
    const int npix = (min(y0 + S, H) - y0) * cw;
    const bool wide = mg.nvec >= 32;
    const int vlane = wide ? lane : lane % mg.nvec;
    const int psub = wide ? 0 : lane / mg.nvec;
    if (!wide && psub >= mg.ppw) return;  // idle lane (zeros join the shuffles)
    const int p0 = wide ? k : k * mg.ppw + psub;
    const int pstride = wide ? mg.wpc : mg.wpc * mg.ppw;
    const uint4 *xv = reinterpret_cast<const uint4 *>(x);
    const long rowpitch = (long)W * (C / PV);  // uint4 per image row
    const uint4 *base = xv + ((long)n * H + y0) * rowpitch + (long)x0 * (C / PV) + vlane;
    int p = p0, py = p0 / cw, px = p0 - (p0 / cw) * cw;
    while (p < npix) {
        uint4 q[kMaxItems];
        int np = 0;
        {
            int qy = py, qx = px, qp = p;
#pragma unroll
            for (int i = 0; i < PPC; ++i) {
                if (qp < npix) {
                    const uint4 *pix = base + qy * rowpitch + (long)qx * (C / PV);
#pragma unroll
                    for (int sl = 0; sl < SLOTS; ++sl)  // a partial last slot (nvec % 32) loads zeros
                        q[i * SLOTS + sl] = (!wide || sl * 32 + vlane < mg.nvec) ? __ldca(pix + sl * 32)
                                                                                  : make_uint4(0u, 0u, 0u, 0u);
                    ++np;
                }
                qp += pstride;
                qx += pstride;
                while (qx >= cw) {
                    qx -= cw;
                    ++qy;
                }
            }
            p = qp;
            py = qy;
            px = qx;
        }
#pragma unroll
        for (int i = 0; i < PPC; ++i) {
            if (i >= np) break;
#pragma unroll
            for (int sl = 0; sl < SLOTS; ++sl) {
                const bool live = !wide || sl * 32 + vlane < mg.nvec;
                const float4 *wp = reinterpret_cast<const float4 *>(wm + (live ? sl * 32 + vlane : 0) * PV);
                float w[PV];
#pragma unroll
                for (int e = 0; e < PV / 4; ++e) {
                    const float4 f = live ? __ldg(wp + e) : make_float4(0.f, 0.f, 0.f, 0.f);  // L1-resident
                    w[4 * e] = f.x;
                    w[4 * e + 1] = f.y;
                    w[4 * e + 2] = f.z;
                    w[4 * e + 3] = f.w;
                }
                if constexpr (EXACT) {
                    Elem<T>::fma8(q[i * SLOTS + sl], w, dacc);
                } else {
                    Elem<T>::ffma8(q[i * SLOTS + sl], w, facc, fmag);
                    nterms += live ? PV : 0;
                }
            }
        }
    }
}

template <typename T, bool EXACT, int SLOTS>
__device__ __forceinline__ void warp_items(const T *__restrict__ x, const float *__restrict__ w_s, const MaskGeo &mg,
                                           int H, int W, int C, int S, int n, int gy, int gx, int k, int lane,
                                           double &dacc, float &facc, float &fmag, int &nterms) {
    warp_items_s<T, EXACT, SLOTS>(x, w_s, mg, H, W, C, S, n, gy, gx, k, lane, dacc, facc, fmag, nterms);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        if constexpr (EXACT) {
            dacc += __shfl_xor_sync(0xffffffffu, dacc, off);
        } else {
            facc += __shfl_xor_sync(0xffffffffu, facc, off);
            fmag += __shfl_xor_sync(0xffffffffu, fmag, off);
            nterms = max(nterms, __shfl_xor_sync(0xffffffffu, nterms, off));
        }
    }
}

// The exact fp64 pass, kept out of line: it runs for logits requests and for the
// rare cells the fp32 bound cannot decide, and must not cost the fast path registers.
template <typename T, int SLOTS>
__device__ __noinline__ double warp_items_exact(const T *__restrict__ x, const float *__restrict__ w_s,
                                                const MaskGeo mg, int H, int W, int C, int S, int n, int gy, int gx,
                                                int k, int lane) {
    double d = 0.0;
    float fa = 0.f, fm = 0.f;
    int nt = 0;
    warp_items<T, true, SLOTS>(x, w_s, mg, H, W, C, S, n, gy, gx, k, lane, d, fa, fm, nt);
    return d;
}

__device__ __forceinline__ int cell_npix(int H, int W, int S, int gy, int gx) {
    return (min(gy * S + S, H) - gy * S) * (min(gx * S + S, W) - gx * S);
}

// All 256 threads of the CTA call this together: decides the CTA's cpb cells
// [cell0, cell0 + cpb).  want_logits: exact fp64 everywhere.  Otherwise each cell
// is decided from the fp32 sum when the error bound separates it from 0 (so the
// decision equals exact arithmetic), and re-summed in fp64 when it does not.
// Returns, in thread 0 of each group's leading warp, the decision (and logit).
template <typename T, int SLOTS>
__device__ __forceinline__ void cta_decide(const T *__restrict__ x, const float *__restrict__ w_s, const MaskGeo &mg, float bm,
                                           int H, int W, int C, int S, int Gh, int Gw, long ncells, long cell0,
                                           bool want_logits, uint8_t *dec, double *logits) {
    __shared__ float r_f[8], r_m[8];
    __shared__ int r_n[8];
    __shared__ double r_d[8];
    __shared__ int s_need[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / mg.wpc, k = warp - grp * mg.wpc;
    const long cell = cell0 + grp;
    const bool valid = grp < mg.cpb && cell < ncells;
    const int G = Gh * Gw;
    int n = 0, gy = 0, gx = 0;
    if (valid) {
        n = (int)(cell / G);
        const int g = (int)(cell - (long)n * G);
        gy = g / Gw;
        gx = g - gy * Gw;
    }
    bool need_exact = want_logits;
    if (!want_logits) {
        double d = 0.0;
        float fa = 0.f, fm = 0.f;
        int nt = 0;
        if (valid) warp_items<T, false, SLOTS>(x, w_s, mg, H, W, C, S, n, gy, gx, k, lane, d, fa, fm, nt);
        if (lane == 0) {
            r_f[warp] = fa;
            r_m[warp] = fm;
            r_n[warp] = nt;
        }
        __syncthreads();
        if (valid && k == 0 && lane == 0) {
            float sa = 0.f, sm = 0.f;
            int chain = 0;
            for (int j = 0; j < mg.wpc; ++j) {  // fixed order
                sa += r_f[warp + j];
                sm += r_m[warp + j];
                chain = max(chain, r_n[warp + j]);
            }
            const double n_chain = (double)chain + 6.0 + mg.wpc;  // lane chain + shuffles + group adds
            const double u = 5.9604644775390625e-8;               // 2^-24
            const double err = (double)sm * (n_chain * u / (1.0 - n_chain * u)) * 1.0001 + 1e-37;
            const int npix = cell_npix(H, W, S, gy, gx);
            const double z = (double)sa + (double)bm * (double)npix;  // scaled logit
            const bool sure = fabs(z) > err * 1.0001 + 1e-300;
            s_need[grp] = !sure;
            if (sure) dec[cell] = z > 0.0 ? 1 : 0;
        }
        __syncthreads();
        need_exact = valid && s_need[grp];
        if (!__syncthreads_or(need_exact)) return;
    }
    double d = 0.0;
    if (need_exact) d = warp_items_exact<T, SLOTS>(x, w_s, mg, H, W, C, S, n, gy, gx, k, lane);
    if (lane == 0) r_d[warp] = d;
    __syncthreads();
    if (need_exact && k == 0 && lane == 0) {
        double sd = 0.0;
        for (int j = 0; j < mg.wpc; ++j) sd += r_d[warp + j];
        const double logit = sd / (double)cell_npix(H, W, S, gy, gx) + (double)bm;
        dec[cell] = logit > 0.0 ? 1 : 0;
        if (logits) logits[cell] = logit;
    }
}

template <typename T, int SLOTS>
__global__ void __launch_bounds__(kMaskThreads, 3) masker_kernel(const T *__restrict__ x, const float *__restrict__ wm,
                                                              float bm, int n_img, int H, int W, int C, int S, int Gh,
                                                              int Gw, MaskGeo mg, uint8_t *__restrict__ mask,
                                                              double *__restrict__ logits) {
    pdl_wait();
    pdl_trigger();
    const long ncells = (long)n_img * Gh * Gw;
    cta_decide<T, SLOTS>(x, wm, mg, bm, H, W, C, S, Gh, Gw, ncells, (long)blockIdx.x * mg.cpb, logits != nullptr,
                         mask, logits);
}

MaskGeo mask_geo(int C, int PV, int S) {
    MaskGeo g;
    g.nvec = C / PV;
    g.ppw = g.nvec < 32 ? 32 / g.nvec : 1;
    // vector slots per lane: ceil(nvec / 32) rounded up to a power of two (the kernel's
    // SLOTS template); lanes past nvec in the last slot load nothing
    g.nvl = 1;
    while (g.nvec >= 32 && g.nvl * 32 < g.nvec) g.nvl *= 2;
    const int items = g.nvec >= 32 ? S * S * g.nvl : (S * S + g.ppw - 1) / g.ppw;  // loads per lane per cell
    // warps per cell: LASNET_MASK_MAXITEMS (default 8 = loads per lane per round
    // trip) bounds a warp's share; 1 warp per cell walks the cell in several round trips
    static const int max_items = [] {
        const char *e = getenv("LASNET_MASK_MAXITEMS");
        return e ? atoi(e) : 2 * kMaxItems;
    }();
    g.wpc = 1;
    while (g.wpc < 8 && (items + g.wpc - 1) / g.wpc > max_items) g.wpc *= 2;
    g.cpb = 8 / g.wpc;
    return g;
}

cudaError_t launch_masker(int dtype_bf16, const void *x, const float *wm, float bm, int n_img, int H,
                          int W, int C, int S, uint8_t *mask, double *logits, cudaStream_t st) {
    const int Gh = (H + S - 1) / S, Gw = (W + S - 1) / S;
    const long ncells = (long)n_img * Gh * Gw;
    if (ncells == 0) return cudaSuccess;
    const MaskGeo mg = mask_geo(C, dtype_bf16 ? 8 : 4, S);
    const long grid = (ncells + mg.cpb - 1) / mg.cpb;
    const int slots = mg.nvec >= 32 ? mg.nvl : 1;
    cudaError_t e = cudaSuccess;
#define LASNET_MASKER(TT, SL)                                                                                  \
    e = launch_k(masker_kernel<TT, SL>, dim3((unsigned)grid), dim3(kMaskThreads), 0, st, static_cast<const TT *>(x), \
                 wm, bm, n_img, H, W, C, S, Gh, Gw, mg, mask, logits)
    if (dtype_bf16) {
        if (slots == 1) LASNET_MASKER(__nv_bfloat16, 1);
        else if (slots == 2) LASNET_MASKER(__nv_bfloat16, 2);
        else if (slots == 4) LASNET_MASKER(__nv_bfloat16, 4);
        else LASNET_MASKER(__nv_bfloat16, 8);
    } else {
        if (slots == 1) LASNET_MASKER(float, 1);
        else if (slots == 2) LASNET_MASKER(float, 2);
        else if (slots == 4) LASNET_MASKER(float, 4);
        else LASNET_MASKER(float, 8);
    }
#undef LASNET_MASKER
    return e;
}

// ------------------------------------------------------------ compaction ---

constexpr int kCompactThreads = 256;
constexpr int kCellsPerThread = 16;
constexpr int kCellsPerTile = kCompactThreads * kCellsPerThread;  // 4096
constexpr uint32_t kFlagAgg = 1u, kFlagPrefix = 2u;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kCompactThreads) compact_kernel(const uint8_t *mask, int ncells,
                                                                  int32_t *__restrict__ idx,
                                                                  int32_t *__restrict__ count,
                                                                  unsigned long long *status) {
    __shared__ int warp_tot[kCompactThreads / 32];
    __shared__ int tile_prefix;
    pdl_wait();
    pdl_trigger();
    const int tile = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long base = (long)tile * kCellsPerTile + (long)tid * kCellsPerThread;

    uint8_t m[kCellsPerThread];
    if (base + kCellsPerThread <= ncells && (reinterpret_cast<uintptr_t>(mask + base) & 15) == 0) {
        const uint4 v = *reinterpret_cast<const uint4 *>(mask + base);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) m[i] = (base + i < ncells) ? mask[base + i] : 0;
    }
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) cnt += m[i] != 0;

    // block-wide exclusive scan of cnt
    int incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int warp_off = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kCompactThreads / 32; ++w) {
        if (w < warp) warp_off += warp_tot[w];
        agg += warp_tot[w];
    }
    const int excl = warp_off + incl - cnt;

    // decoupled look-back (warp 0)
    if (warp == 0) {
        int prefix = 0;
        if (tile == 0) {
            if (lane == 0) {
                __threadfence();
                atomicExch(status, ((unsigned long long)kFlagPrefix << 32) | (unsigned)agg);
            }
        } else {
            if (lane == 0) {
                atomicExch(status + tile, ((unsigned long long)kFlagAgg << 32) | (unsigned)agg);
            }
            int pred = tile - 1;
            while (true) {
                const int j = pred - lane;
                unsigned long long s = j >= 0 ? ld_volatile_u64(status + j)
                                              : ((unsigned long long)kFlagPrefix << 32);
                while (__any_sync(0xffffffffu, (uint32_t)(s >> 32) == 0u)) {
                    if ((uint32_t)(s >> 32) == 0u) s = ld_volatile_u64(status + j);
                }
                const unsigned pmask = __ballot_sync(0xffffffffu, (uint32_t)(s >> 32) == kFlagPrefix);
                const int first_p = pmask ? __ffs(pmask) - 1 : 32;
                int v = lane <= first_p ? (int)(uint32_t)(s & 0xffffffffu) : 0;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                prefix += v;
                if (pmask) break;
                pred -= 32;
            }
            if (lane == 0) {
                __threadfence();
                atomicExch(status + tile, ((unsigned long long)kFlagPrefix << 32) | (unsigned)(prefix + agg));
            }
        }
        if (lane == 0) {
            tile_prefix = prefix;
            if (tile == gridDim.x - 1) *count = prefix + agg;
        }
    }
    __syncthreads();
    int pos = tile_prefix + excl;
#pragma unroll
    for (int i = 0; i < 16; ++i)
        if (m[i]) idx[pos++] = (int32_t)(base + i);
}

size_t compact_workspace_bytes(int ncells) {
    const long tiles = ((long)ncells + kCellsPerTile - 1) / kCellsPerTile;
    return (size_t)(tiles > 0 ? tiles : 1) * sizeof(unsigned long long);
}

// Returns the number of kernels launched.
int launch_compact(const uint8_t *mask, int ncells, int32_t *idx, int32_t *count, void *ws, cudaStream_t st,
                   cudaError_t *err) {
    if (ncells == 0) {
        *err = cudaMemsetAsync(count, 0, sizeof(int32_t), st);
        return 0;
    }
    const int tiles = (ncells + kCellsPerTile - 1) / kCellsPerTile;
    cudaError_t e = cudaMemsetAsync(ws, 0, (size_t)tiles * sizeof(unsigned long long), st);
    if (e != cudaSuccess) {
        *err = e;
        return 0;
    }
    *err = launch_k(compact_kernel, dim3(tiles), dim3(kCompactThreads), 0, st, mask, ncells, idx, count,
                    static_cast<unsigned long long *>(ws));
    return 1;
}


// ------------------------------------------- fused masker + compaction ----
// Steps 1+2 in one launch (App. B: "the masker generates the indices of
// activated patches instead of sparse mask").  Every CTA decides 16 cells (one
// warp each) and writes the mask bytes; the last CTA to finish (done counter)
// compacts the whole mask into ascending ids with block-wide scans, writes the
// count and resets the counter -- the workspace is left zeroed, so no per-call
// memset.  (A decoupled look-back is slower here: all CTAs finish together and
// the prefix chain becomes serial.)
constexpr int kFusedWarps = 8;

#ifdef LASNET_TRACE
// [0] earliest CTA start, [1] latest cell decision, [2] last CTA begins compaction, [3] compaction done
__device__ unsigned long long g_mtrace[4];
__device__ __forceinline__ unsigned long long mtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define MTRACE_MIN(k) atomicMin(&g_mtrace[k], mtimer())
#define MTRACE_MAX(k) atomicMax(&g_mtrace[k], mtimer())
extern "C" int lasnet_mtrace_read(unsigned long long *h) { return (int)cudaMemcpyFromSymbol(h, g_mtrace, 32); }
extern "C" int lasnet_mtrace_clear(void) {
    unsigned long long z[4] = {~0ull, 0, 0, 0};
    return (int)cudaMemcpyToSymbol(g_mtrace, z, 32);
}
#else
#define MTRACE_MIN(k) do { } while (0)
#define MTRACE_MAX(k) do { } while (0)
#endif

struct FusedWs {
    unsigned int done, pad[3];
    uint8_t decisions[16];  // used when the caller passes no mask buffer (ncells bytes)
};

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ uint4 ld_cg_u4(const void *p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <typename T, int SLOTS>
__global__ void __launch_bounds__(kMaskThreads, 3) masker_compact_kernel(
    const T *__restrict__ x, const float *__restrict__ wm, float bm, int n_img, int H, int W, int C, int S, int Gh,
    int Gw, MaskGeo mg, uint8_t *mask, double *__restrict__ logits, int32_t *__restrict__ idx,
    int32_t *__restrict__ count, FusedWs *ws) {
    __shared__ int s_last;
    __shared__ int s_warp[kFusedWarps];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long ncells = (long)n_img * Gh * Gw;
    uint8_t *dec = mask ? mask : ws->decisions;
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) MTRACE_MIN(0);
    cta_decide<T, SLOTS>(x, wm, mg, bm, H, W, C, S, Gh, Gw, ncells, (long)blockIdx.x * mg.cpb, logits != nullptr,
                         dec, logits);
    if (threadIdx.x == 0) MTRACE_MAX(1);
    __syncthreads();
    if (threadIdx.x == 0) {
        // release: this CTA's decisions (ordered before by bar.sync) become visible
        // before the counter moves; acquire: the last CTA then sees everyone's
        s_last = atom_add_acq_rel_gpu(&ws->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x == 0) MTRACE_MAX(2);
    // ---- last CTA: compaction of all ncells decisions (16 per thread per pass)
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    constexpr int kPass = 32 * kFusedWarps * 16;
    for (long c0 = 0; c0 < ncells; c0 += kPass) {
        const long base = c0 + (long)threadIdx.x * 16;
        uint8_t m[16];
        if (base + 16 <= ncells && ((reinterpret_cast<uintptr_t>(dec + base) & 15) == 0)) {
            const uint4 v = ld_cg_u4(dec + base);
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) m[i] = (uint8_t)(wv[i >> 2] >> (8 * (i & 3)));
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                m[i] = 0;
                if (base + i < ncells) {
                    unsigned int b;
                    asm volatile("ld.global.cg.u8 %0, [%1];" : "=r"(b) : "l"(dec + base + i));
                    m[i] = (uint8_t)b;
                }
            }
        }
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) cnt += m[i] != 0;
        int incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        int woff = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kFusedWarps; ++w) {
            woff += w < warp ? s_warp[w] : 0;
            tot += s_warp[w];
        }
        int pos = s_base + woff + incl - cnt;
#pragma unroll
        for (int i = 0; i < 16; ++i)
            if (m[i]) idx[pos++] = (int32_t)(base + i);
        __syncthreads();
        if (threadIdx.x == 0) s_base += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *count = s_base;
        ws->done = 0u;  // kernel completion orders this before the next launch
        MTRACE_MAX(3);
    }
}

size_t mask_compact_workspace_bytes(long ncells) {
    return sizeof(FusedWs) + (size_t)(ncells > 16 ? ncells - 16 : 0);
}

cudaError_t launch_mask_compact(int dtype_bf16, const void *x, const float *wm, float bm, int n_img, int H, int W,
                                int C, int S, uint8_t *mask, double *logits, int32_t *idx, int32_t *count, void *ws,
                                cudaStream_t st) {
    const int Gh = (H + S - 1) / S, Gw = (W + S - 1) / S;
    const long ncells = (long)n_img * Gh * Gw;
    if (ncells == 0) return cudaMemsetAsync(count, 0, sizeof(int32_t), st);
    const MaskGeo mg = mask_geo(C, dtype_bf16 ? 8 : 4, S);
    const long grid = (ncells + mg.cpb - 1) / mg.cpb;
    FusedWs *w = static_cast<FusedWs *>(ws);
    const int slots = mg.nvec >= 32 ? mg.nvl : 1;
    cudaError_t e = cudaSuccess;
#define LASNET_FUSED(TT, SL)                                                                                      \
    e = launch_k(masker_compact_kernel<TT, SL>, dim3((unsigned)grid), dim3(kMaskThreads), 0, st,                      \
                 static_cast<const TT *>(x), wm, bm, n_img, H, W, C, S, Gh, Gw, mg, mask, logits, idx, count, w)
    if (dtype_bf16) {
        if (slots == 1) LASNET_FUSED(__nv_bfloat16, 1);
        else if (slots == 2) LASNET_FUSED(__nv_bfloat16, 2);
        else if (slots == 4) LASNET_FUSED(__nv_bfloat16, 4);
        else LASNET_FUSED(__nv_bfloat16, 8);
    } else {
        if (slots == 1) LASNET_FUSED(float, 1);
        else if (slots == 2) LASNET_FUSED(float, 2);
        else if (slots == 4) LASNET_FUSED(float, 4);
        else LASNET_FUSED(float, 8);
    }
#undef LASNET_FUSED
    return e;
}

}  // namespace lasnet

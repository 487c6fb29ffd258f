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
#include <cuda_bf16.h>
#include <cuda_runtime.h>

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
    __device__ static void ffma8(const uint4 &v, const float *w, const float *wa, float &acc, float &mag) {
        const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float lo = __uint_as_float(q[i] << 16), hi = __uint_as_float(q[i] & 0xFFFF0000u);
            acc = fmaf(w[2 * i], lo, acc);
            acc = fmaf(w[2 * i + 1], hi, acc);
            mag = fmaf(wa[2 * i], fabsf(lo), mag);
            mag = fmaf(wa[2 * i + 1], fabsf(hi), mag);
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
    __device__ static void ffma8(const uint4 &v, const float *w, const float *wa, float &acc, float &mag) {
        const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            acc = fmaf(w[i], f[i], acc);
            mag = fmaf(wa[i], fabsf(f[i]), mag);
        }
    }
};

// One warp computes the masker logit of one coarse cell:
//   logit = (1/|Omega|) * sum_{p in Omega} sum_c w_c x[p,c] + b
// EXACT = true: fp64 accumulation of exact products (bf16 x fp32 fits a double).
// EXACT = false: fp32 FFMA accumulation of the same sum together with
//   sum |w_c x[p,c]|; returns a bound on the fp32 rounding error through *err
//   (Higham: |fl(s) - s| <= gamma_n * sum|terms|, n = longest addition chain).
// Lanes own 16-byte channel vectors; when a pixel has fewer than 32 vectors
// the warp covers several pixels per step.  8 loads per lane are in flight.
template <typename T, bool EXACT>
__device__ __forceinline__ double cell_sum(const T *__restrict__ x, const float *__restrict__ wm, int H, int W, int C,
                                           int S, int n, int gy, int gx, int lane, int &npix_out, double *err) {
    constexpr int PV = Elem<T>::kPerVec;
    const int y0 = gy * S, x0 = gx * S;
    const int cw = min(x0 + S, W) - x0;
    const int npix = (min(y0 + S, H) - y0) * cw;
    npix_out = npix;
    const int nvec = C / PV;
    const uint4 *xv = reinterpret_cast<const uint4 *>(x);
    const long img = (long)n * H * W;
    double acc = 0.0;
    float facc = 0.f, fmag = 0.f;
    int nterms = 0;
    const int ppw = nvec <= 32 ? 32 / nvec : 1;         // pixels per warp step
    const int v0 = nvec <= 32 ? lane % nvec : lane;     // first vector of this lane
    const int psub = nvec <= 32 ? lane / nvec : 0;
    const int vstep = nvec <= 32 ? nvec : 32;
    if (psub < ppw) {
        for (int v = v0; v < nvec; v += vstep) {
            float w[PV], wa[PV];
#pragma unroll
            for (int k = 0; k < PV; ++k) {
                w[k] = __ldg(wm + v * PV + k);
                wa[k] = fabsf(w[k]);
            }
            for (int p0 = psub; p0 < npix; p0 += 8 * ppw) {
                uint4 q[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int p = p0 + u * ppw;
                    if (p < npix) {
                        const int yy = y0 + p / cw, xx = x0 + p % cw;
                        q[u] = __ldg(xv + ((img + (long)yy * W + xx) * C) / PV + v);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (p0 + u * ppw < npix) {
                        if constexpr (EXACT) {
                            Elem<T>::fma8(q[u], w, acc);
                        } else {
                            Elem<T>::ffma8(q[u], w, wa, facc, fmag);
                            nterms += PV;
                        }
                    }
                }
            }
            if (nvec <= 32) break;
        }
    }
    if constexpr (EXACT) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        return acc;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        facc += __shfl_xor_sync(0xffffffffu, facc, off);
        fmag += __shfl_xor_sync(0xffffffffu, fmag, off);
        nterms = max(nterms, __shfl_xor_sync(0xffffffffu, nterms, off));
    }
    // chain length: per-lane sequential terms + 5 shuffle levels (+1 for the FFMA product)
    const double n_chain = (double)nterms + 6.0;
    const double u = 5.9604644775390625e-8;  // 2^-24
    *err = (double)fmag * (n_chain * u / (1.0 - n_chain * u)) * 1.0001 + 1e-37;
    return (double)facc;
}

// Decision and logit of one cell.  want_logit: exact fp64 logit.  Otherwise the
// decision is taken from the fp32 sum when its error bound separates it from 0
// (so it equals the decision of exact arithmetic) and recomputed in fp64 when not.
template <typename T>
__device__ __forceinline__ bool cell_decide(const T *__restrict__ x, const float *__restrict__ wm, float bm, int H,
                                            int W, int C, int S, int n, int gy, int gx, int lane, bool want_logit,
                                            double &logit) {
    int npix;
    if (!want_logit) {
        double err;
        const double s32 = cell_sum<T, false>(x, wm, H, W, C, S, n, gy, gx, lane, npix, &err);
        const double z = s32 + (double)bm * (double)npix;  // scaled logit, fp64
        if (fabs(z) > err * 1.0001 + 1e-300) {
            logit = z / (double)npix;
            return z > 0.0;
        }
    }
    const double s64 = cell_sum<T, true>(x, wm, H, W, C, S, n, gy, gx, lane, npix, nullptr);
    logit = s64 / (double)npix + (double)bm;
    return logit > 0.0;
}

template <typename T>
__global__ void __launch_bounds__(256) masker_kernel(const T *__restrict__ x, const float *__restrict__ wm,
                                                     float bm, int n_img, int H, int W, int C, int S,
                                                     int Gh, int Gw, uint8_t *__restrict__ mask,
                                                     double *__restrict__ logits) {
    const int lane = threadIdx.x & 31;
    const long cell = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long ncells = (long)n_img * Gh * Gw;
    if (cell >= ncells) return;
    const int G = Gh * Gw;
    const int n = (int)(cell / G);
    const int g = (int)(cell - (long)n * G);
    const int gy = g / Gw, gx = g - gy * Gw;
    double logit;
    const bool act = cell_decide<T>(x, wm, bm, H, W, C, S, n, gy, gx, lane, logits != nullptr, logit);
    if (lane == 0) {
        mask[cell] = act ? 1 : 0;
        if (logits) logits[cell] = logit;
    }
}

cudaError_t launch_masker(int dtype_bf16, const void *x, const float *wm, float bm, int n_img, int H,
                          int W, int C, int S, uint8_t *mask, double *logits, cudaStream_t st) {
    const int Gh = (H + S - 1) / S, Gw = (W + S - 1) / S;
    const long ncells = (long)n_img * Gh * Gw;
    if (ncells == 0) return cudaSuccess;
    const int warps = 8;
    const long grid = (ncells + warps - 1) / warps;
    if (dtype_bf16)
        masker_kernel<__nv_bfloat16><<<(unsigned)grid, warps * 32, 0, st>>>(
            static_cast<const __nv_bfloat16 *>(x), wm, bm, n_img, H, W, C, S, Gh, Gw, mask, logits);
    else
        masker_kernel<float><<<(unsigned)grid, warps * 32, 0, st>>>(static_cast<const float *>(x), wm, bm,
                                                                    n_img, H, W, C, S, Gh, Gw, mask, logits);
    return cudaGetLastError();
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

__global__ void __launch_bounds__(kCompactThreads) compact_kernel(const uint8_t *__restrict__ mask, int ncells,
                                                                  int32_t *__restrict__ idx,
                                                                  int32_t *__restrict__ count,
                                                                  unsigned long long *status) {
    __shared__ int warp_tot[kCompactThreads / 32];
    __shared__ int tile_prefix;
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
    compact_kernel<<<tiles, kCompactThreads, 0, st>>>(mask, ncells, idx, count,
                                                      static_cast<unsigned long long *>(ws));
    *err = cudaGetLastError();
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
constexpr int kFusedWarps = 16;

struct FusedWs {
    unsigned int done, pad[3];
    uint8_t decisions[16];  // used when the caller passes no mask buffer (ncells bytes)
};

__device__ __forceinline__ uint4 ld_cg_u4(const void *p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

template <typename T>
__global__ void __launch_bounds__(32 * kFusedWarps) masker_compact_kernel(
    const T *__restrict__ x, const float *__restrict__ wm, float bm, int n_img, int H, int W, int C, int S, int Gh,
    int Gw, uint8_t *mask, double *__restrict__ logits, int32_t *__restrict__ idx, int32_t *__restrict__ count,
    FusedWs *ws) {
    __shared__ int s_last;
    __shared__ int s_warp[kFusedWarps];
    __shared__ int s_base;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long ncells = (long)n_img * Gh * Gw;
    const long cell = (long)blockIdx.x * kFusedWarps + warp;
    uint8_t *dec = mask ? mask : ws->decisions;
    if (cell < ncells) {
        const int G = Gh * Gw;
        const int n = (int)(cell / G);
        const int g = (int)(cell - (long)n * G);
        const int gy = g / Gw, gx = g - gy * Gw;
        double logit;
        const bool act = cell_decide<T>(x, wm, bm, H, W, C, S, n, gy, gx, lane, logits != nullptr, logit);
        if (lane == 0) {
            dec[cell] = act ? 1 : 0;
            if (logits) logits[cell] = logit;
            __threadfence();  // publish before the done-counter increment
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
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
        ws->done = 0u;
        __threadfence();
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
    const long grid = (ncells + kFusedWarps - 1) / kFusedWarps;
    FusedWs *w = static_cast<FusedWs *>(ws);
    if (dtype_bf16)
        masker_compact_kernel<__nv_bfloat16><<<(unsigned)grid, 32 * kFusedWarps, 0, st>>>(
            static_cast<const __nv_bfloat16 *>(x), wm, bm, n_img, H, W, C, S, Gh, Gw, mask, logits, idx, count, w);
    else
        masker_compact_kernel<float><<<(unsigned)grid, 32 * kFusedWarps, 0, st>>>(
            static_cast<const float *>(x), wm, bm, n_img, H, W, C, S, Gh, Gw, mask, logits, idx, count, w);
    return cudaGetLastError();
}

}  // namespace lasnet

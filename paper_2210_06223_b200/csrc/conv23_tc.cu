// conv23_tc.cu -- steps 4 and 5 of the LASNet block fused in one persistent
// tcgen05 kernel: the 3x3 conv on the gathered patch batch and the last
// 1x1 conv with the scatter-add into the residual map.
//
// Per 128-row tile (patch-aligned in dynamic mode, image-row-aligned dense):
//   conv2  A = 4-D TMA im2col box of h1, B = W2 (TMA), K = 9*c_mid -> TMEM acc2
//   epi2   (warps 0-3) acc2 + b2, ReLU, bf16 -> the K-major 128-B-swizzled smem
//          tile H2 (never written to HBM)
//   conv3  A = H2 (smem), B = W3 chunk of 128 output channels (TMA), K = c_mid
//          -> TMEM acc3 (double-buffered per chunk)
//   epi3   (warps 4-11) acc3 + b3 + residual x (cp.async prefetched one chunk
//          ahead) -> ReLU -> bf16 -> 16-B coalesced stores to y (in place)
// conv2 and conv3 have separate smem rings, TMA producers and MMA-issuing
// warps, so the HBM-bound conv3 epilogue of tile i overlaps the L2-bound conv2
// K-loop of tile i+1 instead of stalling it.  Warps: 0-3 epi2, 4-11 epi3,
// 12 conv2 producer, 13 conv2 MMA + TMEM allocator, 14 conv3 MMA, 15 conv3 producer.
//
// (Weight multicast over 2- / 4-CTA clusters and 2-SM pair UMMAs were built and measured
// slower -- lockstep and cross-CTA arrivals cost more than the weight traffic they save,
// and removed in round 2.)
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "rowmap.cuh"
#include "sm100_ptx.cuh"

namespace lasnet {

using namespace ptx;

#ifdef LASNET_TRACE
// CTA 0 timeline per local tile: [0] conv2 loads start [1] conv2 acc ready
// [2] H2 staged [3] conv3 MMAs done [4] last chunk stored
__device__ unsigned long long g_trace23[64 * 8];
__device__ __forceinline__ unsigned long long gtimer23() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define T23(i, k) \
    do { if (blockIdx.x == 0 && (i) < 64) g_trace23[(i) * 8 + (k)] = gtimer23(); } while (0)
// per conv3 chunk: [0] W3 load issued [1] MMA acc free [2] W3 landed [3] MMAs committed
// [4] epi3 residual landed [5] epi3 acc ready [6] epi3 stored
__device__ unsigned long long g_trace23c[64 * 16];
#define T23C(c, k) \
    do { if (blockIdx.x == 0 && (c) < 64) g_trace23c[(c) * 16 + (k)] = gtimer23(); } while (0)
#else
#define T23(i, k) do { } while (0)
#define T23C(c, k) do { } while (0)
#endif

namespace c23 {
constexpr int kBM = 128, kBK = 64;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
#ifndef LASNET_C23_STAGES
#define LASNET_C23_STAGES 3
#endif
#ifndef LASNET_C23_H2BUFS
#define LASNET_C23_H2BUFS 1
#endif
constexpr int kStages = LASNET_C23_STAGES;  // conv2 ring depth
constexpr int kH2Bufs = LASNET_C23_H2BUFS;  // H2 tiles (double-buffering lets epi2 of tile i+1 overlap conv3 of tile i)
constexpr int kStageBytes = 2 * kABytes;  // A 16 KB + B (<= 128 rows) 16 KB
constexpr int kNC3 = 128;                 // max conv3 output channels per MMA chunk (64 when c_out % 128 != 0)
constexpr int kAcc3 = 2;                  // conv3 accumulator buffers (128 TMEM columns each)
constexpr int kChunkBytes = kBM * 128;    // one 64-column bf16 chunk of a 128-row tile
#ifndef LASNET_C23_EPI3_WARPS
#define LASNET_C23_EPI3_WARPS 8
#endif
// epi3 warps: 8, each 32 rows x 32 columns of a 64-column part (16 warps of 16 columns measured
// slower: configs[1] block conv23 51.2 -> 52.9 us, unlike conv_tc's conv3 epilogue)
constexpr int kEpi3Warps = LASNET_C23_EPI3_WARPS;
constexpr int kThreads = (8 + kEpi3Warps) * 32;
constexpr int kEpi2Warp0 = 0, kEpi3Warp0 = 4, kProdWarp = 4 + kEpi3Warps, kMmaWarp = kProdWarp + 1,
              kMma3Warp = kProdWarp + 2, kProd3Warp = kProdWarp + 3;
constexpr int kStages3 = 2;                // conv3 weight ring (<= 16 KB stages: kNC3 rows x 64 K)
constexpr int kB3Bytes = kNC3 * 128;
// smem layout (offsets from the 1024-aligned base); biases are read through L1
constexpr int kStagesOff = 0;
constexpr int kH2Off = kStages * kStageBytes;                 // 2 x up to 32 KB (c_mid <= 128), double-buffered
constexpr int kResBufs = 3;  // residual prefetched kResBufs-1 64-column chunks ahead (epi3 waits on its HBM latency)
constexpr int kResOff = kH2Off + kH2Bufs * 2 * kChunkBytes;   // kResBufs x 16 KB (one 64-col chunk)
constexpr int kRing3Off = kResOff + kResBufs * kChunkBytes;
constexpr int kBiasOff = kRing3Off + kStages3 * kB3Bytes;     // b2 (<= 128 floats), b3 (<= 2048 floats)
constexpr int kMaxCout = 512;
constexpr int kBarOff = kBiasOff + (128 + kMaxCout) * 4;      // barriers
constexpr int smem_bytes(int, int) { return 1024 + kBarOff + 256; }  // + 1 KB to round the dynamic smem base up to 1 KB
}  // namespace c23

// output pixel of row r of a conv23 tile (or -1): patch rows in dynamic mode, image rows dense
template <bool DENSE>
__device__ __forceinline__ int tile_pixel(const ConvArgs &args, int tile, int r, int rows_per_tile, int M) {
    if (r >= rows_per_tile) return -1;
    if (DENSE) {
        const int per_img = args.cols_w * args.rows_h;
        int n0, y0, x0;
        dense_tile_origin(args, tile, n0, y0, x0);
        const int im = r / per_img, rr = r - im * per_img, yy = y0 + rr / args.cols_w, xx = x0 + rr % args.cols_w;
        const int n = n0 + im;
        return (n < args.n_img && yy < args.H && xx < args.W) ? (n * args.H + yy) * args.W + xx : -1;
    }
    return out_pixel(args, tile * rows_per_tile + r, M);
}

// Dynamic tiles: tile t holds patches [t0, t0 + nv).  Fixed: units_per_tile each.
// Balanced (args.balance): the count is spread over T = whole rounds of the grid
// (q or q + 1 patches per tile), so the last round is not a partial one.
struct DynTiles {
    int upt, cnt, q, rem;
    bool bal;
    __device__ __forceinline__ void range(int t, int &t0, int &nv) const {
        if (bal) {
            t0 = t * q + min(t, rem);
            nv = q + (t < rem ? 1 : 0);
        } else {
            t0 = t * upt;
            nv = min(upt, cnt - t0);
        }
    }
};

template <bool DENSE>
__global__ void __launch_bounds__(c23::kThreads, 1) conv23_kernel(const __grid_constant__ ConvArgs args) {
    using namespace c23;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    const uint32_t sbase = (raw_u32 + 1023u) & ~1023u;  // 128-B swizzle atoms need a 1 KB aligned base
    uint8_t *sgen = smem_raw + (sbase - raw_u32);
    const uint32_t h2s = sbase + kH2Off;
    const uint32_t bar = sbase + kBarOff;
    const uint32_t bar_full = bar, bar_empty = bar + 8 * kStages;
    const uint32_t bar_t2full = bar + 16 * kStages, bar_t2empty = bar_t2full + 16;
    const uint32_t bar_t3full = bar_t2empty + 16, bar_t3empty = bar_t3full + 8 * kAcc3;
    const uint32_t bar_h2full = bar_t3empty + 8 * kAcc3, bar_h2empty = bar_h2full + 16;  // [2] each
    const uint32_t bar_full3 = bar_h2empty + 16, bar_empty3 = bar_full3 + 8 * kStages3;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sgen + kBarOff + 16 * kStages + 32 + 16 * kAcc3 + 32 +
                                                       16 * kStages3);
    const int KC = args.N;   // c_mid: conv2 N and conv3 K (64 or 128)
    const int CO = args.n3;  // c_out
    float *b2_s = reinterpret_cast<float *>(sgen + kBiasOff);  // biases staged once in smem
    float *b3_s = b2_s + 128;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);  // the MMA commit
        }
        for (int s = 0; s < kStages3; ++s) {
            mbar_init(bar_full3 + 8 * s, 1);
            mbar_init(bar_empty3 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_t2full + 8 * a, 1);
            mbar_init(bar_t2empty + 8 * a, 128);  // epi2 threads
        }
        for (int a = 0; a < kAcc3; ++a) {
            mbar_init(bar_t3full + 8 * a, 1);
            mbar_init(bar_t3empty + 8 * a, 32 * kEpi3Warps);  // epi3 threads
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_h2full + 8 * a, 128);
            mbar_init(bar_h2empty + 8 * a, 1);
        }
        fence_mbar_init();
    }
    if (warp == kProdWarp && lane == 0) {
        tma_prefetch_desc(&args.tmap_a);
        tma_prefetch_desc(&args.tmap_b);
        tma_prefetch_desc(&args.tmap_b3);
    }
    if (warp == kMmaWarp) {
        tmem_alloc<512>(smem_u32(tmem_slot));
    }
    for (int c = tid; c < args.N; c += kThreads) b2_s[c] = args.bias[c];
    for (int c = tid; c < args.n3; c += kThreads) b3_s[c] = args.bias3[c];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();  // h1, idx and count of the previous kernels are complete from here on
    pdl_trigger();
    // TMEM columns: acc2[2] at 0 / KC, acc3[kAcc3] at 256 + 64 k
    const uint32_t acc3_col = 256;

    // tile geometry
    int num_tiles, rows_per_tile;
    if (DENSE) {
        num_tiles = args.dense_tiles;
        rows_per_tile = args.box_rows;
    } else {
        num_tiles = (*args.count + args.units_per_tile - 1) / args.units_per_tile;
        rows_per_tile = args.units_per_tile * args.S * args.S;
    }
    DynTiles dt{args.units_per_tile, DENSE ? 0 : *args.count, 0, 0, false};
    if (!DENSE && args.balance && num_tiles > (int)gridDim.x) {
        // only when every tile of the rounded-up count gets at least one patch (q >= 1):
        // an empty tile would still stream the weights and issue its MMAs
        const int t_bal = (num_tiles + gridDim.x - 1) / gridDim.x * gridDim.x;
        if (dt.cnt >= t_bal) {
            num_tiles = t_bal;
            dt.bal = true;
            dt.q = dt.cnt / num_tiles;
            dt.rem = dt.cnt - dt.q * num_tiles;
        }
    }
    const int M = DENSE ? 0 : (*args.count) * args.S * args.S;  // valid h2 rows (dynamic)
    const int kb2 = 9 * KC / kBK;                                 // conv2 K-blocks
    const int kpt = KC / kBK;                                     // K-blocks per tap
    const int kb3 = KC / kBK;                                     // conv3 K-blocks
    const int NC3 = CO % kNC3 == 0 ? kNC3 : 64;                   // conv3 MMA N
    const int nch = CO / NC3;                                     // conv3 MMA chunks
    const int nsub = CO / 64;                                     // 64-column epilogue sub-chunks
    // local tile i of this CTA: blockIdx.x + i * gridDim.x
    const int ntl = (int)blockIdx.x < num_tiles ? (num_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    auto tile_of = [&](int i) { return (int)blockIdx.x + i * (int)gridDim.x; };

    if (warp == kProdWarp && !DENSE && args.direct) {
        // ------------------- conv2 TMA producer, direct from the dense h1 --
        // lane u owns patch u of the tile: one {64, S, S} box per K-block at the
        // cell's halo origin (TMA zero-fills the halo outside the image)
        int it = 0;
        const int ss128 = args.S * args.S * 128;
        const int cnt = *args.count;
        // the next tile's cell ids are loaded while this tile's boxes are issued
        auto ids_of = [&](int i) {
            if (i >= ntl) return -1;
            int t0, nv;
            dt.range(tile_of(i), t0, nv);
            return lane < nv ? __ldcg(args.idx + t0 + lane) : -1;  // (written by the previous kernel)
        };
        int next = ids_of(0);
        for (int i = 0; i < ntl; ++i) {
            int t0, nval;
            dt.range(tile_of(i), t0, nval);
            const int cell = next;
            next = ids_of(i + 1);
            int n = 0, y0 = 0, x0 = 0;
            if (cell >= 0) {
                int gy, gx;
                cell_decode(args, cell, n, gy, gx);
                y0 = gy * args.S - 1;
                x0 = gx * args.S - 1;
            }
            for (int kb = 0; kb < kb2; ++kb, ++it) {
                const int st = it % kStages;
                const uint32_t sa = sbase + st * kStageBytes, fb = bar_full + 8 * st;
                const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3, c0 = (kb - tap * kpt) * kBK;
                if (lane == 0) {
                    mbar_wait(bar_empty + 8 * st, ((it / kStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(fb, nval * ss128 + KC * 128);
                    tma_load_2d(sa + kABytes, &args.tmap_b, fb, kb * kBK, 0);
                }
                __syncwarp();
                if (lane < nval) tma_load_5d(sa + lane * ss128, &args.tmap_a, fb, 0, x0 + dx, y0 + dy, n, c0 >> 6);
            }
        }
    } else if (warp == kProdWarp) {
        // ------------------------------------------ conv2 TMA producer --
        int it = 0;
        for (int i = 0; i < ntl; ++i) {
            const int tile = tile_of(i);
            if (lane == 0) {
                int n0 = 0, y0 = 0, x0 = 0;
                if (DENSE) dense_tile_origin(args, tile, n0, y0, x0);
                T23(i, 0);
                for (int kb = 0; kb < kb2; ++kb, ++it) {
                    const int st = it % kStages;
                    mbar_wait(bar_empty + 8 * st, ((it / kStages) & 1) ^ 1);
                    const uint32_t sa = sbase + st * kStageBytes, fb = bar_full + 8 * st;
                    const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3, c0 = (kb - tap * kpt) * kBK;
                    mbar_arrive_expect_tx(fb, args.box_rows * 128 + KC * 128);
                    int t0 = 0, nv;
                    if (!DENSE) dt.range(tile, t0, nv);
                    tma_load_2d(sa + kABytes, &args.tmap_b, fb, kb * kBK, 0);
                    // h1 is channel-chunk-major: [c_mid/64][P][S+2][S+2][64] (dense: [c_mid/64][N][H][W][64])
                    if (DENSE) tma_load_5d(sa, &args.tmap_a, fb, 0, x0 + dx - 1, y0 + dy - 1, n0, c0 >> 6);
                    else if (args.conv_stride == 2)  // stride-2 3x3 (projection block): parity view of the windows
                        tma_load_5d(sa, &args.tmap_s[((dy & 1) << 1) | (dx & 1)], fb, 0, dx >> 1, dy >> 1, t0, c0 >> 6);
                    else tma_load_5d(sa, &args.tmap_a, fb, 0, dx, dy, t0, c0 >> 6);
                }
            }
            __syncwarp();
        }
    } else if (warp == kProd3Warp) {
        // ------------------------------------- conv3 weight TMA producer --
        if (lane == 0) {
            int it = 0;
            for (int i = 0; i < ntl; ++i)
                for (int nc = 0; nc < nch; ++nc)
                    for (int kb = 0; kb < kb3; ++kb, ++it) {
                        const int st = it % kStages3;
                        mbar_wait(bar_empty3 + 8 * st, ((it / kStages3) & 1) ^ 1);
                        if (kb == 0) T23C(i * nch + nc, 0);
                        const uint32_t fb = bar_full3 + 8 * st;
                        mbar_arrive_expect_tx(fb, NC3 * 128);
                        tma_load_2d(sbase + kRing3Off + st * kB3Bytes, &args.tmap_b3, fb, kb * kBK, nc * NC3);
                    }
        }
    } else if (warp == kMmaWarp) {
        // ---------------------------------------------- conv2 MMA issuer --
        if (lane == 0) {
            const uint32_t idesc2 = idesc_bf16_f32(kBM, KC);
            int it = 0;
            for (int i = 0; i < ntl; ++i) {
                const int acc = i & 1;
                mbar_wait(bar_t2empty + 8 * acc, ((i >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem_base + acc * KC;
                for (int kb = 0; kb < kb2; ++kb, ++it) {
                    const int st = it % kStages;
                    mbar_wait(bar_full + 8 * st, (it / kStages) & 1);
                    tc_fence_after();
                    const uint32_t sa = sbase + st * kStageBytes;
                    const uint64_t ad = smem_desc_sw128(sa), bd = smem_desc_sw128(sa + kABytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc2, (kb | kk) != 0);
                    mma_commit(bar_empty + 8 * st);
                }
                mma_commit(bar_t2full + 8 * acc);
            }
        }
        __syncwarp();
    } else if (warp == kMma3Warp) {
        // ---------------------------------------------- conv3 MMA issuer --
        if (lane == 0) {
            const uint32_t idesc3 = idesc_bf16_f32(kBM, NC3);
            int it = 0, c3 = 0;
            for (int i = 0; i < ntl; ++i) {
                const int hb = i % kH2Bufs;
                const uint32_t h2b = h2s + hb * 2 * kChunkBytes;
                // H2 of tile i staged by epi2 (pair: both CTAs')
                mbar_wait(bar_h2full + 8 * hb, (i / kH2Bufs) & 1);
                tc_fence_after();
                for (int nc = 0; nc < nch; ++nc, ++c3) {
                    const int buf = c3 % kAcc3;
                    mbar_wait(bar_t3empty + 8 * buf, ((c3 / kAcc3) & 1) ^ 1);
                    T23C(c3, 1);
                    tc_fence_after();
                    const uint32_t d = tmem_base + acc3_col + buf * kNC3;  // kNC3 columns per buffer
                    for (int kb = 0; kb < kb3; ++kb, ++it) {
                        const int st = it % kStages3;
                        mbar_wait(bar_full3 + 8 * st, (it / kStages3) & 1);
                        if (kb == kb3 - 1) T23C(c3, 2);
                        tc_fence_after();
                        const uint64_t ad = smem_desc_sw128(h2b + kb * kChunkBytes);
                        const uint64_t bd = smem_desc_sw128(sbase + kRing3Off + st * kB3Bytes);
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            mma_bf16(d, ad + 2 * kk, bd + 2 * kk, idesc3, (kb | kk) != 0);
                        mma_commit(bar_empty3 + 8 * st);
                    }
                    mma_commit(bar_t3full + 8 * buf);
                    T23C(c3, 3);
                }
                // buffer reusable once these MMAs have read it
                mma_commit(bar_h2empty + 8 * hb);
                T23(i, 3);
            }
        }
        __syncwarp();
    } else if (warp < kEpi3Warp0) {
        // ---------------------------------------- epi2: acc2 -> H2 (smem) --
        const int r = warp * 32 + lane;
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        for (int i = 0; i < ntl; ++i) {
            const int acc = i & 1;
            mbar_wait(bar_t2full + 8 * acc, (i >> 1) & 1);
            if (r == 0) T23(i, 1);
            mbar_wait(bar_h2empty + 8 * (i % kH2Bufs), ((i / kH2Bufs) & 1) ^ 1);  // conv3 MMAs of tile i-kH2Bufs read it
            tc_fence_after();
            for (int c = 0; c < KC; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + lane_base + acc * KC + c, v);
                tmem_ld_wait();
                const uint32_t rowbase = h2s + (i % kH2Bufs) * 2 * kChunkBytes + (c >> 6) * kChunkBytes + r * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int col = c + 8 * q + 2 * e;
                        const float lo = fmaxf(__uint_as_float(v[8 * q + 2 * e]) + b2_s[col], 0.f);
                        const float hi = fmaxf(__uint_as_float(v[8 * q + 2 * e + 1]) + b2_s[col + 1], 0.f);
                        pk[e] = pack_bf16x2(lo, hi);
                    }
                    const uint32_t saddr = rowbase + ((((c & 63) >> 3) + q) ^ (r & 7)) * 16;
                    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(pk[0]), "r"(pk[1]),
                                 "r"(pk[2]), "r"(pk[3])
                                 : "memory");
                }
            }
            tc_fence_before();
            fence_proxy_async_smem();  // generic smem writes -> visible to tcgen05.mma
            mbar_arrive(bar_t2empty + 8 * acc);
            mbar_arrive(bar_h2full + 8 * (i % kH2Bufs));
            if (r == 0) T23(i, 2);
        }
    } else if (warp >= kEpi3Warp0 && warp < kProdWarp) {
        // ------------------------------- epi3: acc3 + b3 + x -> ReLU -> y --
        // kEpi3Warps warps per 64-column part: rows 32*quarter.., columns kColsW*cg..
        constexpr int kColsW = 64 / (kEpi3Warps / 4);
        const int ew = warp - kEpi3Warp0;
        const int quarter = ew & 3, cg = ew >> 2;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const __nv_bfloat16 *X = static_cast<const __nv_bfloat16 *>(args.resid);
        __nv_bfloat16 *Y = static_cast<__nv_bfloat16 *>(args.out);
        // output pixel of tile-row r of local tile i (or -1)
        auto pixel_of = [&](int i) -> int {
            if (!DENSE && dt.bal) {
                int t0, nv;
                dt.range(tile_of(i), t0, nv);
                return r < nv * args.S * args.S ? out_pixel(args, t0 * args.S * args.S + r, M) : -1;
            }
            return tile_pixel<DENSE>(args, tile_of(i), r, rows_per_tile, M);
        };
        constexpr int kChunks = kColsW / 8;       // 16-B chunks of this warp's columns
        constexpr int kRowsPerIt = 32 / kChunks;  // rows per store instruction
        constexpr int kIt = 32 / kRowsPerIt;      // store instructions per 32 rows
        const int c16 = lane % kChunks, rl0 = lane / kChunks;
        auto chunk_addr = [&](uint32_t buf, int rl) -> uint32_t {
            const int row = quarter * 32 + rl;
            return buf + row * 128 + (((cg * kChunks + c16) ^ (row & 7)) << 4);
        };
        // element offsets (pixel * out_ld + this lane's 8 columns) of the rows this lane moves in the
        // coalesced pattern (rows k*8 + lane/4 of the warp's 32); constant over the chunks of a tile
        auto row_offsets = [&](int i, long long (&o)[kIt]) {
            const int pix = i < ntl ? pixel_of(i) : -1;
#pragma unroll
            for (int k = 0; k < kIt; ++k) {
                const int p = __shfl_sync(0xffffffffu, pix, k * kRowsPerIt + rl0);
                o[k] = p >= 0 ? (long long)p * args.out_ld + cg * kColsW + c16 * 8 : -1;
            }
        };
        auto prefetch = [&](const long long (&o)[kIt], int nc, uint32_t buf) {
#pragma unroll
            for (int k = 0; k < kIt; ++k)
                cp_async_16(chunk_addr(buf, k * kRowsPerIt + rl0), o[k] >= 0 ? X + o[k] + nc * 64 : X,
                            o[k] >= 0 ? 16u : 0u);
            cp_async_commit();
        };
        const uint32_t res0 = sbase + kResOff;
        constexpr int D = kResBufs - 1;  // prefetch distance in chunks (D <= nch: at most one tile ahead)
        // the prefetch runs at most one tile ahead (cur / nxt row offsets): D <= nsub
        long long cur[kIt], nxt[kIt];
        row_offsets(0, cur);
        row_offsets(1, nxt);
        int pf_i = 0, pf_nc = 0, pf_n = 0;  // next chunk to prefetch
        auto issue_prefetch = [&](int i_now) {
            if (pf_i < ntl) {
                long long o[kIt];
#pragma unroll
                for (int k = 0; k < kIt; ++k) o[k] = pf_i == i_now ? cur[k] : nxt[k];
                prefetch(o, pf_nc, res0 + (pf_n % kResBufs) * kChunkBytes);
            } else {
                cp_async_commit();
            }
            ++pf_n;
            if (++pf_nc == nsub) pf_nc = 0, ++pf_i;
        };
        for (int d = 0; d < D; ++d) issue_prefetch(0);
        int sc = 0;  // 64-column sub-chunk counter
        const int spc = NC3 / 64;  // sub-chunks per MMA chunk
        for (int i = 0; i < ntl; ++i) {
            for (int nc = 0; nc < nsub; ++nc, ++sc) {
                const int c3 = sc / spc, part = sc - c3 * spc;  // MMA chunk, 64-col part of it
                const int buf = c3 % kAcc3;
                const uint32_t sres = res0 + (sc % kResBufs) * kChunkBytes;
                issue_prefetch(i);  // sub-chunk sc + D into the buffer sub-chunk sc - 1 used
                cp_async_wait<D>();  // sub-chunk sc has landed
                __syncwarp();
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 4);
                if (part == 0) mbar_wait(bar_t3full + 8 * buf, (c3 / kAcc3) & 1);
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 5);
                tc_fence_after();
                const int col0 = nc * 64 + cg * kColsW;
                uint32_t v[kColsW];
                tmem_ld_cols(tmem_base + lane_base + acc3_col + buf * kNC3 + part * 64 + cg * kColsW, v);
                tmem_ld_wait();
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 7);
                if (part == spc - 1) {
                    tc_fence_before();
                    // accumulator drained into registers
                    mbar_arrive(bar_t3empty + 8 * buf);
                }
                // all smem loads first (smem latency is long under UMMA/TMA traffic), then math, then stores
                uint32_t rv[kChunks][4];
#pragma unroll
                for (int q = 0; q < kChunks; ++q)
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(rv[q][0]), "=r"(rv[q][1]), "=r"(rv[q][2]), "=r"(rv[q][3])
                                 : "r"(sres + r * 128 + (((cg * kChunks + q) ^ (r & 7)) << 4)));
                float4 bsv[kColsW / 4];
#pragma unroll
                for (int j = 0; j < kColsW / 4; ++j) bsv[j] = reinterpret_cast<const float4 *>(b3_s + col0)[j];
                const float *bias = reinterpret_cast<const float *>(bsv);
                uint32_t pk[kChunks][4];
#pragma unroll
                for (int q = 0; q < kChunks; ++q)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = 8 * q + 2 * e;
                        const float lo = fmaxf(__uint_as_float(v[c]) + bias[c] + bf16lo(rv[q][e]), 0.f);
                        const float hi = fmaxf(__uint_as_float(v[c + 1]) + bias[c + 1] + bf16hi(rv[q][e]), 0.f);
                        pk[q][e] = pack_bf16x2(lo, hi);
                    }
#pragma unroll
                for (int q = 0; q < kChunks; ++q)
                    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(
                                     sres + r * 128 + (((cg * kChunks + q) ^ (r & 7)) << 4)),
                                 "r"(pk[q][0]), "r"(pk[q][1]), "r"(pk[q][2]), "r"(pk[q][3])
                                 : "memory");
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 8);
                __syncwarp();
                uint4 o[kIt];
#pragma unroll
                for (int k = 0; k < kIt; ++k)
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(o[k].x), "=r"(o[k].y), "=r"(o[k].z), "=r"(o[k].w)
                                 : "r"(chunk_addr(sres, k * kRowsPerIt + rl0)));
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 9);
#pragma unroll
                for (int k = 0; k < kIt; ++k)
                    if (cur[k] >= 0) *reinterpret_cast<uint4 *>(Y + cur[k] + nc * 64) = o[k];
                __syncwarp();
                if (warp == kEpi3Warp0 && lane == 0) T23C(sc, 6);
            }
            if (warp == kEpi3Warp0 && lane == 0) T23(i, 4);
#pragma unroll
            for (int k = 0; k < kIt; ++k) cur[k] = nxt[k];
            row_offsets(i + 2, nxt);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

#ifdef LASNET_TRACE
extern "C" int lasnet_trace23_read(unsigned long long *h) {
    return (int)cudaMemcpyFromSymbol(h, g_trace23, sizeof(unsigned long long) * 512);
}
extern "C" int lasnet_trace23_clear(void) {
    static unsigned long long z[1024];
    cudaMemcpyToSymbol(g_trace23c, z, sizeof(z));
    return (int)cudaMemcpyToSymbol(g_trace23, z, sizeof(unsigned long long) * 512);
}
extern "C" int lasnet_trace23c_read(unsigned long long *h) {
    return (int)cudaMemcpyFromSymbol(h, g_trace23c, sizeof(unsigned long long) * 1024);
}
#endif

template <bool DENSE>
static cudaError_t launch23(const ConvArgs &a, int max_tiles, int num_sms, cudaStream_t st) {
    const int smem = c23::smem_bytes(a.N, a.n3);
    static int cfg = 0;
    if (smem > cfg) {
        cudaError_t e = cudaFuncSetAttribute(conv23_kernel<DENSE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        cfg = smem;
    }
    const int grid = max_tiles < num_sms ? (max_tiles > 0 ? max_tiles : 1) : num_sms;  // at most one CTA per SM
    return launch_k(conv23_kernel<DENSE>, dim3(grid), dim3(c23::kThreads), smem, st, a);
}

cudaError_t launch_conv23(bool dense, const ConvArgs &a, int max_tiles, int num_sms, cudaStream_t st) {
    if (!(a.N == 64 || a.N == 128) || a.n3 % 64 != 0 || a.n3 > c23::kMaxCout || a.n3 < 64 * (c23::kResBufs - 1))
        return cudaErrorInvalidValue;
    return dense ? launch23<true>(a, max_tiles, num_sms, st) : launch23<false>(a, max_tiles, num_sms, st);
}

}  // namespace lasnet

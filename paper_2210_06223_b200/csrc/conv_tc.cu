// conv_tc.cu -- tcgen05 (5th-gen tensor core) implicit-GEMM convolutions of the
// LASNet bottleneck, bf16 x bf16 -> fp32 (TMEM) -> bf16, all operands moved by TMA.
//
// One persistent, warp-specialised kernel template serves the six modes of
// rowmap.cuh.  Per CTA (1 per SM, 192 threads):
//   warps 0-3  epilogue: tcgen05.ld the fp32 accumulator (thread = GEMM row =
//              TMEM lane), + bias [+ residual], ReLU, bf16 RNE into a 128-B-
//              swizzled smem staging tile, then one thread TMA-stores it
//   warp 4     producer: one thread issues every TMA load -- the weight tile B
//              (2-D box) and the activation tile A, whose box shape does the
//              gather/im2col:
//                conv1 dyn   one 4-D box {64, S+2, S+2|1, 1} of x per patch
//                            (or per halo row), OOB halo pixels zero-filled
//                conv2 dyn   one 4-D box {64, S, S, patches} of h1 per tap
//                conv2 dense one 4-D box {64, W, rows, imgs} of h1 per tap,
//                            the zero padding is TMA's OOB fill
//                others      one 2-D box {64, 128} of a contiguous row matrix
//              and, for conv3, the residual tile of x into the staging buffer
//              (per-patch 4-D boxes in dynamic mode: the scatter is the store)
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
// Pipelines: ST smem stages (full/empty mbarriers), two TMEM accumulators
// (tmem_full/tmem_empty) and two staging buffers (stage_full/stage_empty), so
// loads, MMAs, epilogue math and TMA stores of consecutive tiles overlap.
// Dynamic modes derive their tile count from the device-resident active count:
// no host synchronisation (the index list spreads work evenly).
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "rowmap.cuh"
#include "sm100_ptx.cuh"

namespace lasnet {

using namespace ptx;

constexpr int kBM = 128;       // UMMA M (rows per tile = TMEM lanes)
constexpr int kBK = 64;        // K elements per stage = one 128-B swizzle row
constexpr int kThreads = 192;  // 4 epilogue + 1 producer + 1 MMA warps
constexpr int kABytes = kBM * kBK * 2;
constexpr int kChunkBytes = kBM * 128;  // one 64-column bf16 chunk of a 128-row tile

template <int BN> struct TileCfg {
    static constexpr int kStages = BN == 128 ? 4 : 6;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStagingBytes = (BN / 64) * kChunkBytes;
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kStagingOff = kStages * kStageBytes;
    static constexpr int kBarOff = kStagingOff + 2 * kStagingBytes;
    static constexpr int kBiasOff = kBarOff + 256;
    static constexpr int smem_bytes(int n) { return 1024 + kBiasOff + n * 4; }
};

// Tile geometry shared by all roles.
struct TileGeo {
    int num_tiles;    // total tiles (M tiles x N tiles)
    int n_tiles_n;    // N / BN
    int units_total;  // dynamic modes: units (boxes) overall
};

template <int MODE>
__device__ __forceinline__ TileGeo tile_geo(const ConvArgs &a, int BN) {
    TileGeo g;
    g.n_tiles_n = a.N / BN;
    int mt;
    if (MODE == CONV1_DYN) {
        g.units_total = (*a.count) * a.units_per_patch;
        mt = (g.units_total + a.units_per_tile - 1) / a.units_per_tile;
    } else if (MODE == CONV2_DYN || MODE == CONV3_DYN) {
        g.units_total = *a.count;  // units = patches
        mt = (g.units_total + a.units_per_tile - 1) / a.units_per_tile;
    } else if (MODE == CONV2_DENSE) {
        g.units_total = 0;
        mt = a.dense_tiles;
    } else {
        g.units_total = 0;
        mt = (a.m_dense + kBM - 1) / kBM;
    }
    g.num_tiles = mt * g.n_tiles_n;
    return g;
}

// CONV2_DENSE tile -> (first image, first image row) of its box.
__device__ __forceinline__ void dense2_tile(const ConvArgs &a, int mt, int &n0, int &y0) {
    if (a.rows_h < a.H) {
        const int tpi = (a.H + a.rows_h - 1) / a.rows_h;
        n0 = mt / tpi;
        y0 = (mt - n0 * tpi) * a.rows_h;
    } else {
        n0 = mt * a.imgs_box;
        y0 = 0;
    }
}

template <int MODE, int BN>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ ConvArgs args) {
    using Cfg = TileCfg<BN>;
    constexpr int ST = Cfg::kStages;
    constexpr bool kResid = (MODE == CONV3_DYN || MODE == CONV3_DENSE);
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    const uint32_t sbase = (raw_u32 + 1023u) & ~1023u;
    uint8_t *sgen = smem_raw + (sbase - raw_u32);

    const uint32_t staging = sbase + Cfg::kStagingOff;      // 2 x kStagingBytes
    const uint32_t bar_full = sbase + Cfg::kBarOff;         // ST
    const uint32_t bar_empty = bar_full + ST * 8;           // ST
    const uint32_t bar_tfull = bar_empty + ST * 8;          // 2
    const uint32_t bar_tempty = bar_tfull + 16;             // 2
    const uint32_t bar_sfull = bar_tempty + 16;             // 2 (conv3: residual landed)
    const uint32_t bar_sempty = bar_sfull + 16;             // 2 (staging free again)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sgen + Cfg::kBarOff + ST * 16 + 64);
    float *bias_s = reinterpret_cast<float *>(sgen + Cfg::kBiasOff);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    for (int i = tid; i < args.N; i += kThreads) bias_s[i] = args.bias[i];
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(bar_full + 8 * s, 1);   // producer arrive.expect_tx
            mbar_init(bar_empty + 8 * s, 1);  // tcgen05.commit
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);     // tcgen05.commit
            mbar_init(bar_tempty + 8 * a, 128);  // every epilogue thread
            mbar_init(bar_sfull + 8 * a, 1);     // producer arrive.expect_tx (residual)
            mbar_init(bar_sempty + 8 * a, 1);    // store thread, after the TMA store read smem
        }
        fence_mbar_init();
    }
    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&args.tmap_a);
        tma_prefetch_desc(&args.tmap_b);
        tma_prefetch_desc(&args.tmap_out);
        if (kResid) tma_prefetch_desc(&args.tmap_res);
    }
    if (warp == 5) tmem_alloc<Cfg::kTmemCols>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const TileGeo geo = tile_geo<MODE>(args, BN);
    const int num_kb = args.K / kBK;
    const int kpt = args.a_ld / kBK;  // K-blocks per 3x3 tap (conv2)

    if (warp == 4) {
        // ------------------------------------------------------- producer --
        if (lane == 0) {
            int it = 0, lt = 0;
            for (int tile = blockIdx.x; tile < geo.num_tiles; tile += gridDim.x, ++lt) {
                const int mt = tile / geo.n_tiles_n;
                const int n0 = (tile - mt * geo.n_tiles_n) * BN;
                int u0 = 0, nu = 0;  // first unit and unit count of this tile (dynamic modes)
                if (MODE == CONV1_DYN || MODE == CONV2_DYN || MODE == CONV3_DYN) {
                    u0 = mt * args.units_per_tile;
                    nu = min(args.units_per_tile, geo.units_total - u0);
                }
                int d2n = 0, d2y = 0;
                if (MODE == CONV2_DENSE) dense2_tile(args, mt, d2n, d2y);
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int stage = it % ST;
                    mbar_wait(bar_empty + 8 * stage, ((it / ST) & 1) ^ 1);
                    const uint32_t sa = sbase + stage * Cfg::kStageBytes;
                    const uint32_t sb = sa + kABytes;
                    const uint32_t fb = bar_full + 8 * stage;
                    int a_bytes;
                    if (MODE == CONV1_DYN) {
                        a_bytes = nu * args.unit_rows * 128;
                    } else if (MODE == CONV2_DYN || MODE == CONV3_DYN) {
                        a_bytes = args.box_rows * 128;  // one box (garbage rows past count are never stored)
                    } else if (MODE == CONV2_DENSE) {
                        a_bytes = args.box_rows * 128;
                    } else {
                        a_bytes = kABytes;
                    }
                    mbar_arrive_expect_tx(fb, a_bytes + Cfg::kBBytes);
                    tma_load_2d(sb, &args.tmap_b, fb, kb * kBK, n0);
                    if (MODE == CONV1_DYN) {
                        const int c0 = kb * kBK;
                        for (int u = 0; u < nu; ++u) {
                            const int unit = u0 + u;
                            const int t = unit / args.units_per_patch;
                            const int jy = (unit - t * args.units_per_patch) * args.unit_halo_rows;
                            int n, gy, gx;
                            cell_coords(args, t, n, gy, gx);
                            tma_load_4d(sa + u * args.unit_rows * 128, &args.tmap_a, fb, c0, gx * args.S - 1,
                                        gy * args.S - 1 + jy, n);
                        }
                    } else if (MODE == CONV2_DYN) {
                        const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                        tma_load_4d(sa, &args.tmap_a, fb, (kb - tap * kpt) * kBK, dx, dy, u0);
                    } else if (MODE == CONV2_DENSE) {
                        const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                        tma_load_4d(sa, &args.tmap_a, fb, (kb - tap * kpt) * kBK, dx - 1, d2y + dy - 1, d2n);
                    } else if (MODE == CONV3_DYN) {
                        tma_load_2d(sa, &args.tmap_a, fb, kb * kBK, u0 * args.S * args.S);
                    } else {
                        tma_load_2d(sa, &args.tmap_a, fb, kb * kBK, mt * kBM);
                    }
                }
                if (kResid) {
                    // residual tile of x -> staging buffer lt&1 (the epilogue adds it in place);
                    // issued after the K loads so MMA(lt) overlaps the epilogue of lt-1
                    const int b = lt & 1;
                    mbar_wait(bar_sempty + 8 * b, ((lt >> 1) & 1) ^ 1);
                    const uint32_t sdst = staging + b * Cfg::kStagingBytes;
                    if (MODE == CONV3_DYN) {
                        const int box_bytes = args.S * args.S * 128;
                        mbar_arrive_expect_tx(bar_sfull + 8 * b, nu * (BN / 64) * box_bytes);
                        for (int p = 0; p < nu; ++p) {
                            int n, gy, gx;
                            cell_coords(args, u0 + p, n, gy, gx);
                            for (int c = 0; c < BN / 64; ++c)
                                tma_load_4d(sdst + c * kChunkBytes + p * box_bytes, &args.tmap_res, bar_sfull + 8 * b,
                                            n0 + c * 64, gx * args.S, gy * args.S, n);
                        }
                    } else {
                        mbar_arrive_expect_tx(bar_sfull + 8 * b, (BN / 64) * kChunkBytes);
                        for (int c = 0; c < BN / 64; ++c)
                            tma_load_2d(sdst + c * kChunkBytes, &args.tmap_res, bar_sfull + 8 * b, n0 + c * 64,
                                        mt * kBM);
                    }
                }
            }
        }
    } else if (warp == 5) {
        // ---------------------------------------------------- MMA issuer --
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN);
            int it = 0, lt = 0;
            for (int tile = blockIdx.x; tile < geo.num_tiles; tile += gridDim.x, ++lt) {
                const int acc = lt & 1;
                mbar_wait(bar_tempty + 8 * acc, ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int stage = it % ST;
                    mbar_wait(bar_full + 8 * stage, (it / ST) & 1);
                    tc_fence_after();
                    const uint32_t sa = sbase + stage * Cfg::kStageBytes;
                    const uint64_t adesc = smem_desc_sw128(sa);
                    const uint64_t bdesc = smem_desc_sw128(sa + kABytes);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                    mma_commit(bar_empty + 8 * stage);
                }
                mma_commit(bar_tfull + 8 * acc);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------- epilogue --
        const int r = tid;  // tile row == TMEM lane
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        int lt = 0;
        for (int tile = blockIdx.x; tile < geo.num_tiles; tile += gridDim.x, ++lt) {
            const int mt = tile / geo.n_tiles_n;
            const int n0 = (tile - mt * geo.n_tiles_n) * BN;
            const int acc = lt & 1, b = lt & 1;
            const uint32_t sbuf = staging + b * Cfg::kStagingBytes;
            bool zero = false;  // conv1: halo pixel outside the image stores 0 (R6)
            if (MODE == CONV1_DYN) {
                const int u = r / args.unit_rows, q = r - u * args.unit_rows;
                const int unit = mt * args.units_per_tile + u;
                if (u < args.units_per_tile && unit < geo.units_total) {
                    const int t = unit / args.units_per_patch;
                    const int hs = args.S + 2;
                    const int j = (unit - t * args.units_per_patch) * args.unit_rows + q;  // halo index
                    const int jy = j / hs, jx = j - jy * hs;
                    int n, gy, gx;
                    cell_coords(args, t, n, gy, gx);
                    const int hy = gy * args.S - 1 + jy, hx = gx * args.S - 1 + jx;
                    zero = hy < 0 || hy >= args.H || hx < 0 || hx >= args.W;
                }
            }
            if (kResid) {
                mbar_wait(bar_sfull + 8 * b, (lt >> 1) & 1);
            } else {
                mbar_wait(bar_sempty + 8 * b, ((lt >> 1) & 1) ^ 1);
            }
            mbar_wait(bar_tfull + 8 * acc, (lt >> 1) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem_base + lane_base + acc * BN + c, v);
                tmem_ld_wait();
                // 32 columns = 4 x 16-B chunks of row r inside 64-column chunk c/64
                const uint32_t rowbase = sbuf + (c >> 6) * kChunkBytes + r * 128;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t saddr = rowbase + ((((c & 63) >> 3) + q) ^ (r & 7)) * 16;
                    float f[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[8 * q + e]) + bias_s[n0 + c + 8 * q + e];
                    if (kResid) {
                        uint32_t rv[4];
                        asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(rv[0]), "=r"(rv[1]), "=r"(rv[2]), "=r"(rv[3])
                                     : "r"(saddr));
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            f[2 * e] += bf16lo(rv[e]);
                            f[2 * e + 1] += bf16hi(rv[e]);
                        }
                    }
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float lo = fmaxf(f[2 * e], 0.f), hi = fmaxf(f[2 * e + 1], 0.f);
                        if (zero) lo = hi = 0.f;
                        pk[e] = pack_bf16x2(lo, hi);
                    }
                    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(pk[0]), "r"(pk[1]),
                                 "r"(pk[2]), "r"(pk[3])
                                 : "memory");
                }
            }
            tc_fence_before();
            mbar_arrive(bar_tempty + 8 * acc);
            fence_proxy_async_smem();  // staging writes -> visible to the TMA store
            named_bar_sync(1, 128);
            if (r == 0) {
                if (MODE == CONV3_DYN) {
                    const int u0 = mt * args.units_per_tile;
                    const int nu = min(args.units_per_tile, geo.units_total - u0);
                    const int box_bytes = args.S * args.S * 128;
                    for (int p = 0; p < nu; ++p) {
                        int n, gy, gx;
                        cell_coords(args, u0 + p, n, gy, gx);
                        for (int c = 0; c < BN / 64; ++c)
                            tma_store_4d(&args.tmap_out, sbuf + c * kChunkBytes + p * box_bytes, n0 + c * 64,
                                         gx * args.S, gy * args.S, n);
                    }
                } else if (MODE == CONV2_DENSE) {
                    int d2n, d2y;
                    dense2_tile(args, mt, d2n, d2y);
                    for (int c = 0; c < BN / 64; ++c)
                        tma_store_4d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, 0, d2y, d2n);
                } else {
                    int row0;
                    if (MODE == CONV1_DYN) row0 = mt * args.units_per_tile * args.unit_rows;
                    else if (MODE == CONV2_DYN) row0 = mt * args.units_per_tile * args.S * args.S;
                    else row0 = mt * kBM;
                    for (int c = 0; c < BN / 64; ++c)
                        tma_store_2d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, row0);
                }
                bulk_commit();
                // the previous tile's store has finished reading its staging buffer
                bulk_wait_read<1>();
                if (lt >= 1) mbar_arrive(bar_sempty + 8 * (b ^ 1));
            }
        }
        if (r == 0) bulk_wait_all<0>();
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<Cfg::kTmemCols>(tmem_base);
    }
}

// ----------------------------------------------------------------- host ----

template <int MODE, int BN>
static cudaError_t launch_mode_bn(const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    auto kern = conv_tc_kernel<MODE, BN>;
    const int smem = TileCfg<BN>::smem_bytes(a.N);
    static int configured = 0;  // per instantiation: largest dynamic smem enabled so far
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const long tiles = (long)max_tiles_m * (a.N / BN);
    const int grid = (int)(tiles < num_sms ? (tiles > 0 ? tiles : 1) : num_sms);
    kern<<<grid, kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_mode(const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    if (a.N == 64) return launch_mode_bn<MODE, 64>(a, max_tiles_m, num_sms, st);
    if (a.N % 128 == 0) return launch_mode_bn<MODE, 128>(a, max_tiles_m, num_sms, st);
    return cudaErrorInvalidValue;
}

// max_tiles_m: capacity bound on the M tiles (grid sizing only; dynamic modes
// derive the true tile count from the device count).
cudaError_t launch_conv_tc(int mode, const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    if (a.K % kBK != 0) return cudaErrorInvalidValue;
    switch (mode) {
        case CONV1_DYN: return launch_mode<CONV1_DYN>(a, max_tiles_m, num_sms, st);
        case CONV2_DYN: return launch_mode<CONV2_DYN>(a, max_tiles_m, num_sms, st);
        case CONV3_DYN: return launch_mode<CONV3_DYN>(a, max_tiles_m, num_sms, st);
        case CONV1_DENSE: return launch_mode<CONV1_DENSE>(a, max_tiles_m, num_sms, st);
        case CONV2_DENSE: return launch_mode<CONV2_DENSE>(a, max_tiles_m, num_sms, st);
        case CONV3_DENSE: return launch_mode<CONV3_DENSE>(a, max_tiles_m, num_sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lasnet

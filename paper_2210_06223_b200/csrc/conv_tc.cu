// conv_tc.cu -- tcgen05 (5th-gen tensor core) implicit-GEMM convolutions of the
// LASNet bottleneck, bf16 x bf16 -> fp32 (TMEM) -> bf16, all operands moved by TMA.
//
// One persistent, warp-specialised kernel template serves the six modes of
// rowmap.cuh.  Per CTA (1 per SM):
//   warps 0-3  epilogue: tcgen05.ld the fp32 accumulator (thread = GEMM row =
//              TMEM lane), + bias [+ residual], ReLU, bf16 RNE into a 128-B-
//              swizzled smem staging tile.  conv1/conv2: one thread TMA-stores
//              the tile (contiguous h1/h2 rows).  conv3: each warp prefetches
//              the residual rows of x for the NEXT tile with cp.async, and
//              writes its 32 output pixels with coalesced 16-B stores -- the
//              scatter-add is this epilogue
//   warp 4     TMA producer: the weight tile B (2-D box) every K-block and the
//              activation tile A where a box does the job:
//                conv2 dyn   one 4-D box {64, S, S, patches} of h1 per tap (im2col)
//                conv2 dense one 4-D box {64, W, rows, imgs} of h1 per tap, the
//                            zero padding is TMA's out-of-bounds fill
//                conv1 dense, conv3   one 2-D box {64, 128} of contiguous rows
//   warps 6-9  (conv1 dyn only) cp.async gather of the halo rows of x: small
//              scattered rows are where TMA's per-box cost dominates, 16-B
//              LDGSTS keep the HBM pipe full
//   warps 6-9  (conv1 dense + masker, the paper's masker-conv1 fusion P:153-160)
//              read each A stage of x from smem (thread = pixel row) and
//              accumulate the fp32 masker partial sum_c wm_c x[p,c] and its
//              magnitude sum_c |wm_c x[p,c]| (error bound of the decision)
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
// Pipelines: ST smem stages (full/empty mbarriers), two TMEM accumulators
// (tmem_full/tmem_empty) and two staging buffers, so loads, MMAs, epilogue math
// and stores of consecutive tiles overlap.  Dynamic modes derive their tile
// count from the device-resident active count: no host synchronisation
// (the index list spreads work evenly over the SMs).
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "launch.cuh"
#include "rowmap.cuh"
#include "sm100_ptx.cuh"

namespace lasnet {

using namespace ptx;

#ifdef LASNET_TRACE
// Debug timeline of CTA 0 (trace builds only): per local tile, globaltimer ns at
// [0] producer tile start [1] producer K loads issued [2] MMA acc free
// [3] MMA last commit [4] epilogue acc ready [5] epilogue staged [6] store issued
__device__ unsigned long long g_trace[64 * 8];
__device__ unsigned long long g_ktrace[128 * 4];  // per K-block: gather issue, TMA issue, MMA full, MMA commit
__device__ int g_trace_mode = -1;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define KTRACE(it, k) \
    do { if (blockIdx.x == 0 && (it) < 128 && MODE == g_trace_mode) g_ktrace[(it) * 4 + (k)] = gtimer(); } while (0)
#define TRACE(lt, k) \
    do { if (blockIdx.x == 0 && (lt) < 64 && MODE == g_trace_mode) g_trace[(lt) * 8 + (k)] = gtimer(); } while (0)
#else
#define TRACE(lt, k) do { } while (0)
#define KTRACE(it, k) do { } while (0)
#endif

constexpr int kBM = 128;       // UMMA M (rows per tile = TMEM lanes)
constexpr int kBK = 64;        // K elements per stage = one 128-B swizzle row
constexpr int kABytes = kBM * kBK * 2;
constexpr int kChunkBytes = kBM * 128;  // one 64-column bf16 chunk of a 128-row tile

// Per-mode configuration.  Warp roles: [0, E) epilogue, E TMA producer,
// E+1 MMA issuer, E+2 .. E+9 cp.async gather (conv1 dyn only).
// PAIR: the two CTAs of a cluster pair run 2-SM UMMAs (cta_group::2, M = 256):
// each stages its own 128 A rows but only HALF of the BN weight rows of every
// K-block, so the weight bytes each SM pulls through L2 halve (the TMA/L2 path,
// ~43 B/clk/SM, bounds a 128 x 256 tile that re-streams all of B: 64 B/clk).
template <int MODE, int BN, bool PAIR = false> struct Cfg {
    static constexpr bool kResid = MODE == CONV3_DYN || MODE == CONV3_DENSE;
    static constexpr bool kGather = MODE == CONV1_DYN || MODE == CONV2_GATHER;
    static constexpr bool kMasker = MODE == CONV1_DENSE_MASK;
    // conv2 gather at BN = 256: the h2 tile is staged and stored in two 128-column halves through
    // one 32 KB buffer, which frees room for a 4th stage (its cp.async A gather is bound by the bytes
    // in flight per SM)
    static constexpr bool kHalfStage =
        (MODE == CONV2_GATHER || MODE == CONV1_DENSE || MODE == CONV1_DENSE_MASK || MODE == CONV1_DYN) && BN == 256 &&
        !PAIR;  // (PROJ_SC measured: 7^2 shortcut 64 -> 54 us, 28^2 96 -> 116 us: not taken)
#ifndef LASNET_RESID_EPI_WARPS
#define LASNET_RESID_EPI_WARPS 16
#endif
#ifndef LASNET_EPI_WARPS
#define LASNET_EPI_WARPS 8
#endif
    // conv3 (residual epilogue): its epilogue bounds the kernel (the MMAs of a 128-column tile
    // take ~1.5 us, the residual / ReLU / scatter of its 128 rows ~2.5 us): 16 warps, 32 columns
    // each (8 warps: conv3_dyn 0.944 -> 0.846 ms per LAS-R101 forward with 16); conv1 / conv2:
    // 8 warps (4: LAS-R101 5.30 -> 5.26 ms with 8)
    // (each warp drains >= 32 columns: 64-column tiles take at most 8 warps)
    static constexpr int kEpiWarpsWant = kResid ? LASNET_RESID_EPI_WARPS : (MODE == STEM ? 4 : LASNET_EPI_WARPS);
    static constexpr int kEpiWarps = kEpiWarpsWant * 32 / 4 > BN ? 4 * BN / 32 : kEpiWarpsWant;
    static_assert(BN / (kEpiWarps / 4) >= 32, "an epilogue warp drains at least 32 TMEM columns");
    static constexpr int kProdWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1, kGatherWarp0 = kEpiWarps + 2;
    static constexpr int kGatherThreads = 256;
    static constexpr int kMaskerWarp0 = kEpiWarps + 2, kMaskerThreads = 256;
    static constexpr int kThreads =
        32 * (kEpiWarps + 2) + (kGather ? kGatherThreads : 0) + (kMasker ? kMaskerThreads : 0);
    // stem: B is the 64-channel weight (its BN = 128 spans two output rows' accumulators)
    static constexpr int kBBytes = (MODE == STEM ? 64 : (PAIR ? BN / 2 : BN)) * kBK * 2;
    // Pairs serve the 256-column conv2 tiles only.  Measured and dropped: pairs for conv1 + masker
    // (the odd CTA's masker warps need the stage-full event relayed from the even CTA: 43 -> 62 us
    // at stage 3, with one or two relay hops), for conv3 and 128-column tiles (slower), and for
    // the cp.async-fed conv2 gather (45 -> 65 us).
    static_assert(!PAIR || MODE == CONV2_DYN || MODE == CONV2_DENSE, "pairs: conv2 only");
    // stem: the whole packed weight (7 K-blocks of 64 x 64, 56 KB) stays resident in smem,
    // loaded once per CTA; its stages carry A only (it was L2-throughput bound re-streaming it)
    static constexpr bool kBRes = MODE == STEM;
    static constexpr int kBResBytes = kBRes ? 7 * kBBytes : 0;
    static constexpr int kStageBytes = kABytes + (kBRes ? 0 : kBBytes);
    // kHalfStage: 64-column chunks per staging pass (the masker's weights keep their smem: one chunk)
    static constexpr int kStagingChunks = kHalfStage ? (kMasker ? 1 : 2) : BN / 64;
    static constexpr int kStagingBytes = kStagingChunks * kChunkBytes;
    // conv1 dyn: HBM gather -> deep pipeline, 1 staging buffer (TMA store drains fast)
    // conv3: short K (2-8 blocks) -> 3 stages, 3 staging buffers (residual prefetched 2 tiles ahead)
    // BN = 256 (conv1 at c_mid >= 256): A is read once per M tile instead
    // of once per 128-column N tile, and each UMMA moves 96 instead of 128 smem bytes
    // per clock; 3 stages of 48 KB + one 64 KB staging tile
    static_assert(BN != 256 || !kResid, "BN = 256 only without the residual epilogue");
    // dense conv1 at 128 columns: 5 stages and one staging tile (more bytes in flight)
    static constexpr bool kDeep128 = (MODE == CONV1_DENSE || MODE == CONV1_DENSE_MASK) && BN == 128 && !PAIR;
    static constexpr int kStaging = BN == 256 || kDeep128 ? 1 : (kGather ? 1 : (kResid ? 3 : 2));
    // pairs: stages of 32 KB (BN 256) / 24 KB (BN 128) -> deeper rings in the same smem
    // stem: resident weights, 16 KB A-only stages
    static constexpr int kStages =
        MODE == STEM ? 6
        : kHalfStage ? 4
        : kDeep128 ? 5
        : PAIR ? (BN == 256 ? 4 : (kResid ? 4 : 6))
               : (BN == 256 ? 3 : (kGather ? (BN == 128 ? 6 : 8) : (kResid ? 3 : (BN == 128 ? 4 : 6))));
    static constexpr int kTmemCols = 2 * BN;
    static constexpr int kStageOff = kBResBytes;  // [resident B][stages][staging][barriers][bias (+wm)]
    static constexpr int kStagingOff = kStageOff + kStages * kStageBytes;
    static constexpr int kBarOff = kStagingOff + kStaging * kStagingBytes;
    static constexpr int kBiasOff = kBarOff + 256;
    // bias [n] then (masker) wm [k]
    static constexpr bool kWmSmem = kMasker;
    // + 1 KB: the dynamic smem base is only guaranteed 16-B aligned (a CTA co-resident
    // with another kernel's CTA may start anywhere); the kernel rounds it up to 1 KB
    static constexpr bool kBiasSmem = !kHalfStage;  // (kHalfStage: bias read through L1, smem is full)
    static constexpr int smem_bytes(int n, int k) {
        return 1024 + kBiasOff + (kBiasSmem ? n * 4 : 0) + (kWmSmem ? k * 4 : 0);
    }
};

template <int MODE, int BN> __host__ __device__ constexpr int threads_of() { return Cfg<MODE, BN>::kThreads; }

// Persistent tile walk.  One CTA: unit u = tile u.  Pair: unit u = (M-tile pair,
// N tile); rank r of the cluster takes M tile 2 * pair + r (a tile past the end,
// odd M-tile count, still runs: zero-filled / never-stored rows).
struct TileWalk {
    int first, step, units, nn, rank;
    bool pair;
    __device__ __forceinline__ int tile(int u) const {
        if (!pair) return u;
        const int pm = u / nn;
        return (2 * pm + rank) * nn + (u - pm * nn);
    }
    // i-th tile of this CTA (i >= 0), -1 past the end (a pair's odd-count tail tile is returned
    // even though it lies past num_tiles: it runs on zero-filled rows and stores nothing)
    __device__ __forceinline__ int at(int i) const {
        const int u = first + i * step;
        return u < units ? tile(u) : -1;
    }
};

// Tile geometry shared by all roles.
struct TileGeo {
    int num_tiles;  // total tiles (M tiles x N tiles)
    int n_tiles_n;  // N / BN
};

template <int MODE>
__device__ __forceinline__ TileGeo tile_geo(const ConvArgs &a, int BN) {
    TileGeo g;
    g.n_tiles_n = a.N / BN;
    int mt;
    if (MODE == CONV2_DYN || MODE == CONV2_GATHER) {
        mt = (*a.count + a.units_per_tile - 1) / a.units_per_tile;  // patch-aligned tiles
    } else if (MODE == CONV2_DENSE || MODE == STEM || ((MODE == CONV3_DENSE || MODE == PROJ_SC) && a.view4)) {
        mt = a.dense_tiles;
        if (MODE == STEM) g.n_tiles_n = 1;  // one 64-channel weight, BN / 64 output rows per tile
    } else {
        mt = (gemm_rows(MODE, a) + kBM - 1) / kBM;
    }
    g.num_tiles = mt * g.n_tiles_n;
    return g;
}

template <int MODE, int BN, bool PAIR = false>
__global__ void __launch_bounds__(threads_of<MODE, BN>(), 1) conv_tc_kernel(const __grid_constant__ ConvArgs args) {
    using C = Cfg<MODE, BN, PAIR>;
    constexpr int ST = C::kStages, NSTG = C::kStaging, EPI = C::kEpiWarps * 32;
    constexpr bool kResid = C::kResid;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_u32 = smem_u32(smem_raw);
    const uint32_t sbase = (raw_u32 + 1023u) & ~1023u;  // 128-B swizzle atoms need a 1 KB aligned base
    uint8_t *sgen = smem_raw + (sbase - raw_u32);

    const uint32_t staging = sbase + C::kStagingOff;  // NSTG x kStagingBytes
    const uint32_t bar_full = sbase + C::kBarOff;     // ST
    const uint32_t bar_empty = bar_full + ST * 8;     // ST
    const uint32_t bar_tfull = bar_empty + ST * 8;    // 2
    const uint32_t bar_tempty = bar_tfull + 16;       // 2
    const uint32_t bar_sempty = bar_tempty + 16;      // 2 (TMA-store modes: staging free again)
    const uint32_t bar_bres = bar_sempty + 16;        // 1 (stem: resident weights landed)
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sgen + C::kBarOff + ST * 16 + 64);
    float *bias_s = reinterpret_cast<float *>(sgen + C::kBiasOff);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int rank = PAIR ? (int)cluster_ctarank() : 0;
    const bool lead = rank == 0;

    if (C::kBiasSmem)
        for (int i = tid; i < args.N; i += C::kThreads) bias_s[i] = args.bias[i];
    // masker weight (CONV1_DENSE_MASK); N % 64 == 0 keeps it 16-B aligned
    const int wm_off = C::kBiasSmem ? args.N : 0;  // the masker weight follows the bias (if that is in smem)
    const float *wm_s = C::kWmSmem ? bias_s + wm_off : args.wm;
    if (C::kWmSmem)
        for (int i = tid; i < args.K; i += C::kThreads) bias_s[wm_off + i] = args.wm[i];
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            // TMA producer's arrive.expect_tx (+ one noinc arrival per gather thread for conv1 dyn)
            mbar_init(bar_full + 8 * s, C::kGather ? C::kGatherThreads + 1 : 1);
            mbar_init(bar_empty + 8 * s, C::kMasker ? 1 + C::kMaskerThreads / 32 : 1);  // tcgen05.commit (+ every masker warp)
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);     // tcgen05.commit (pair: the lead's, multicast)
            mbar_init(bar_tempty + 8 * a, PAIR ? 2 * C::kEpiWarps : EPI);  // every epilogue thread (pair: warp of both CTAs)
            mbar_init(bar_sempty + 8 * a, 1);    // store thread, after the TMA store read smem
        }
        mbar_init(bar_bres, 1);
        fence_mbar_init();
    }
    if (warp == C::kProdWarp && lane == 0) {
        if (!C::kGather && MODE != STEM) tma_prefetch_desc(&args.tmap_a);
        tma_prefetch_desc(&args.tmap_b);
        if (!kResid && MODE != STEM) tma_prefetch_desc(&args.tmap_out);
    }
    if (warp == C::kMmaWarp) {
        if (PAIR) tmem_alloc_pair<C::kTmemCols>(smem_u32(tmem_slot));
        else tmem_alloc<C::kTmemCols>(smem_u32(tmem_slot));
    }
    tc_fence_before();
    if (PAIR) cluster_sync();  // the peer's barriers are initialised before any remote arrive / TMA
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    pdl_wait();     // inputs of the previous kernel (x, h1, idx/count) are complete from here on
    pdl_trigger();

    const TileGeo geo = tile_geo<MODE>(args, BN);
    TileWalk walk;
    walk.pair = PAIR;
    walk.rank = rank;
    walk.nn = geo.n_tiles_n;
    if (PAIR) {
        const int mt_all = geo.num_tiles / geo.n_tiles_n;
        walk.first = blockIdx.x >> 1;
        walk.step = gridDim.x >> 1;
        walk.units = (mt_all + 1) / 2 * geo.n_tiles_n;
    } else {
        walk.first = blockIdx.x;
        walk.step = gridDim.x;
        walk.units = geo.num_tiles;
    }
    // stem: a tile is TWO output rows (2 oy0, 2 oy0 + 1 -> accumulator columns 0-63 / 64-127);
    // its K loop walks the 9 input rows they need, each staged once and used by both rows'
    // MMAs (kernel row j for the first, j - 2 for the second): 9 instead of 14 row loads
    // stem: a tile = R = BN / 64 output rows; its K loop walks the 2 R + 5 input rows they need, each
    // staged once and used by every row whose 7-row window covers it (kernel row kb - 2 j of row j)
    constexpr int kStemRows = BN / 64;
    const int num_kb = MODE == STEM ? 2 * kStemRows + 5 : args.K / kBK;
    const int num_kb_b = args.K / kBK;  // resident weight K-blocks (stem: 7 kernel rows)
    const int kpt = args.a_ld / kBK;  // K-blocks per 3x3 tap (conv2)

    if (warp == C::kProdWarp) {
        // --------------------------------------------------- TMA producer --
        if (lane == 0) {
            if (C::kBRes) {
                mbar_arrive_expect_tx(bar_bres, (uint32_t)(num_kb_b * C::kBBytes));
                for (int kb = 0; kb < num_kb_b; ++kb)
                    tma_load_2d(sbase + kb * C::kBBytes, &args.tmap_b, bar_bres, kb * kBK, 0);
            }
            int it = 0, lt = 0;
            for (int i = 0;; ++i, ++lt) {
                const int tile = walk.at(i);
                if (tile < 0) break;
                const int mt = tile / geo.n_tiles_n;
                const int n0 = (tile - mt * geo.n_tiles_n) * BN;
                const int u0 = MODE == CONV2_DYN ? mt * args.units_per_tile : 0;  // first patch (conv2 dyn)
                int d2n = 0, d2y = 0, d2x = 0;
                if (MODE == CONV2_DENSE || ((MODE == CONV3_DENSE || MODE == PROJ_SC) && args.view4))
                    dense_tile_origin(args, mt, d2n, d2y, d2x);
                TRACE(lt, 0);
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int stage = it % ST;
                    mbar_wait(bar_empty + 8 * stage, ((it / ST) & 1) ^ 1);
                    const uint32_t sa = sbase + C::kStageOff + stage * C::kStageBytes;
                    const uint32_t sb = sa + kABytes;
                    const uint32_t fb = bar_full + 8 * stage;
                    int a_bytes = kABytes;  // conv1 dyn: A arrives by cp.async (not counted here)
                    if (C::kGather) a_bytes = 0;
                    else if (MODE == STEM) a_bytes = args.cols_w * 128;  // 4 boxes of cols_w / 4 columns
                    else if (MODE == CONV2_DYN || MODE == CONV2_DENSE || ((MODE == CONV3_DENSE || MODE == PROJ_SC) && args.view4))
                        a_bytes = args.box_rows * 128;
                    if (PAIR) {
                        // own A rows + own half of the B rows; both CTAs' bytes complete on the lead's barrier
                        if (lead) mbar_arrive_expect_tx(fb, 2 * (a_bytes + C::kBBytes));
                        tma_load_2d_pair(sb, &args.tmap_b, fb, kb * kBK, n0 + rank * (BN / 2));
                        if (MODE == CONV2_DYN) {
                            const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                            if (args.conv_stride == 2)
                                tma_load_5d_pair(sa, &args.tmap_s[((dy & 1) << 1) | (dx & 1)], fb, 0, dx >> 1, dy >> 1,
                                                 u0, kb - tap * kpt);
                            else
                                tma_load_5d_pair(sa, &args.tmap_a, fb, 0, dx, dy, u0, kb - tap * kpt);
                        } else if (MODE == CONV2_DENSE) {
                            const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                            if (args.conv_stride == 2) {
                                const int v = ((dy != 1) << 1) | (dx != 1);
                                tma_load_5d_pair(sa, &args.tmap_s[v], fb, 0, d2x - (dx == 0), d2y - (dy == 0), d2n,
                                                 kb - tap * kpt);
                            } else {
                                tma_load_5d_pair(sa, &args.tmap_a, fb, 0, d2x + dx - 1, d2y + dy - 1, d2n, kb - tap * kpt);
                            }
                        } else if (args.a2_kb && kb >= args.a2_kb) {
                            tma_load_2d_pair(sa, &args.tmap_s[0], fb, (kb - args.a2_kb) * kBK, mt * kBM);
                        } else {
                            tma_load_2d_pair(sa, &args.tmap_a, fb, kb * kBK, mt * kBM);
                        }
                        continue;
                    }
                    mbar_arrive_expect_tx(fb, a_bytes + (C::kBRes ? 0 : C::kBBytes));
                    if (!C::kBRes) tma_load_2d(sb, &args.tmap_b, fb, kb * kBK, n0);
                    KTRACE(it, 1);
                    if (MODE == CONV2_DYN) {
                        const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                        if (args.conv_stride == 2)  // stride-2 3x3: parity view (dy&1, dx&1) of the windows
                            tma_load_5d(sa, &args.tmap_s[((dy & 1) << 1) | (dx & 1)], fb, 0, dx >> 1, dy >> 1, u0,
                                        kb - tap * kpt);
                        else
                            tma_load_5d(sa, &args.tmap_a, fb, 0, dx, dy, u0, kb - tap * kpt);  // h1 [c/64][P][hs][hs][64]
                    } else if (MODE == CONV2_DENSE) {
                        const int tap = kb / kpt, dy = tap / 3, dx = tap - dy * 3;
                        if (args.conv_stride == 2) {
                            // input (2 o + d - 1): view of parity (d != 1), coordinate o - (d == 0)
                            const int v = ((dy != 1) << 1) | (dx != 1);
                            tma_load_5d(sa, &args.tmap_s[v], fb, 0, d2x - (dx == 0), d2y - (dy == 0), d2n, kb - tap * kpt);
                        } else {
                            tma_load_5d(sa, &args.tmap_a, fb, 0, d2x + dx - 1, d2y + dy - 1, d2n, kb - tap * kpt);  // [c/64][N][H][W][64]
                        }
                    } else if (MODE == STEM) {
                        // K-block kb = kernel row dy: 4 boxes of W/4 output columns each (residue k of
                        // ox mod 4), every box row the 8 input pixels x 8 channels of one output pixel
                        // tile = (image, output row pair, column block of cols_w columns); K-block kb =
                        // input row 2 oy0 + kb - 3 (out of the image: TMA zero fill)
                        const int xb = mt % args.tiles_x, row = mt / args.tiles_x;
                        const int groups = (args.H + kStemRows - 1) / kStemRows;
                        const int n = row / groups, oy0 = kStemRows * (row - n * groups);
                        const int q = args.cols_w / 4;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tma_load_4d(sa + k * q * 128, &args.tmap_s[k], fb, 0, xb * q, 2 * oy0 + kb - 3, n);
                    } else if ((MODE == CONV3_DENSE || MODE == PROJ_SC) && args.view4) {
                        // the strided projection shortcut: A = a 4-D view of x at every stride-th pixel
                        // (dense tiles of rows_h x cols_w output pixels of imgs_box images): no subsample copy
                        tma_load_4d(sa, &args.tmap_a, fb, kb * kBK, d2x, d2y, d2n);
                    } else if (!C::kGather) {
                        if (args.a2_kb && kb >= args.a2_kb)  // second A source (projection shortcut input)
                            tma_load_2d(sa, &args.tmap_s[0], fb, (kb - args.a2_kb) * kBK, mt * kBM);
                        else
                            tma_load_2d(sa, &args.tmap_a, fb, kb * kBK, mt * kBM);
                    }
                }
                TRACE(lt, 1);
            }
        }
    } else if (C::kGather && warp >= C::kGatherWarp0) {
        if constexpr (MODE == CONV2_GATHER) {
            // ------------------------- cp.async im2col gather from the dense h1 --
            // thread -> (row group prow, 16-B chunk pch); tile rows prow + 32 i, i < 4: row =
            // (patch t, pixel j of its S x S cell); K-block kb = (tap, 64-channel chunk cb) reads
            // h1 pixel (cell origin + (py + dy - 1, px + dx - 1)) of chunk cb, 0 outside the image
            // (conv2's zero padding, R6).  The next tile's idx loads are in flight during this
            // tile's K-loop.
            constexpr int RPT = 128 * 8 / C::kGatherThreads;
            constexpr int RSTEP = 128 / RPT;
            const int pt = tid - 32 * C::kGatherWarp0;
            const int prow = pt >> 3, pch = pt & 7;
            const __nv_bfloat16 *H1 = static_cast<const __nv_bfloat16 *>(args.a_src);
            const int cnt = *args.count, ss = args.S * args.S, rows_pt = args.units_per_tile * ss;
            auto load_cells = [&](int tile, int (&cell)[RPT]) {
                const int mt = tile / geo.n_tiles_n;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int row = prow + RSTEP * i;
                    const int t = mt * args.units_per_tile + args.fd_SS.div(row);
                    cell[i] = (tile < geo.num_tiles && row < rows_pt && t < cnt) ? ld_nc_volatile(args.idx + t) : -1;
                }
            };
            // base pixel (image row origin) and (y0, x0) = the output pixel's window origin
            auto decode = [&](const int (&cell)[RPT], int (&img)[RPT], int (&y0)[RPT], int (&x0)[RPT]) {
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    img[i] = -1;
                    y0[i] = x0[i] = 0;
                    if (cell[i] >= 0) {
                        int n, gy, gx;
                        cell_decode(args, cell[i], n, gy, gx);
                        const int row = prow + RSTEP * i;
                        const int j = row - args.fd_SS.div(row) * ss;
                        const int py = args.fd_S.div(j);
                        img[i] = n;
                        y0[i] = gy * args.S + py - 1;
                        x0[i] = gx * args.S + (j - py * args.S) - 1;
                    }
                }
            };
            int cell[RPT], img[RPT], y0[RPT], x0[RPT];
            int ncell[RPT], nimg[RPT], ny0[RPT], nx0[RPT];
            auto tile_at = [&](int i) -> int { const int t = walk.at(i); return t < 0 ? geo.num_tiles : t; };
            load_cells(tile_at(0), cell);
            decode(cell, img, y0, x0);
            int it = 0;
            for (int i = 0; walk.at(i) >= 0; ++i) {
                load_cells(tile_at(i + 1), ncell);  // next tile: loads in flight during this K-loop
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int stage = it % ST;
                    const int tap = kb / kpt, cb = kb - tap * kpt, dy = tap / 3, dx = tap - dy * 3;
                    mbar_wait(bar_empty + 8 * stage, ((it / ST) & 1) ^ 1);
                    const uint32_t sa = sbase + C::kStageOff + stage * C::kStageBytes;
                    const __nv_bfloat16 *cbase = H1 + (size_t)cb * args.m_dense * 64 + pch * 8;
#pragma unroll
                    for (int i = 0; i < RPT; ++i) {
                        const int row = prow + RSTEP * i;
                        const int yy = y0[i] + dy, xx = x0[i] + dx;
                        const bool ok = img[i] >= 0 && yy >= 0 && yy < args.H && xx >= 0 && xx < args.W;
                        const __nv_bfloat16 *g = ok ? cbase + (size_t)((img[i] * args.H + yy) * args.W + xx) * 64 : H1;
                        cp_async_16(sa + row * 128 + ((pch ^ (row & 7)) << 4), g, ok ? 16u : 0u);
                    }
                    cp_async_arrive_noinc(bar_full + 8 * stage);
                    if (kb == (num_kb >> 1)) decode(ncell, nimg, ny0, nx0);  // mid-loop: off the tile boundary
                }
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    img[i] = nimg[i];
                    y0[i] = ny0[i];
                    x0[i] = nx0[i];
                }
            }
        } else {
        // ------------------------------------------ cp.async halo gather --
        // thread -> (row group prow, 16-B chunk pch); rows prow + 32 i, i < 4.
        // The idx loads of tile t+1 are issued before the K-loop of tile t and
        // decoded after it, so row mapping never sits on the critical path.
        constexpr int RPT = 128 * 8 / C::kGatherThreads;  // rows per thread
        constexpr int RSTEP = 128 / RPT;
        const int pt = tid - 32 * C::kGatherWarp0;
        const int prow = pt >> 3, pch = pt & 7;
        const __nv_bfloat16 *X = static_cast<const __nv_bfloat16 *>(args.a_src);
        const int M = gemm_rows(MODE, args);
        const int hs = args.hs, hs2 = hs * hs;
        auto load_cells = [&](int tile, int (&cell)[RPT], int (&jj)[RPT]) {
            const int r0 = (tile / geo.n_tiles_n) * kBM + prow;
            int t = args.fd_hs2.div(r0), j = r0 - t * hs2;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = r0 + RSTEP * i;
                cell[i] = -1;
                if (tile < geo.num_tiles && r < M) cell[i] = ld_nc_volatile(args.idx + t);  // stays before the K-loop
                jj[i] = j;
                j += RSTEP;
                while (j >= hs2) {
                    j -= hs2;
                    ++t;
                }
            }
        };
        auto decode = [&](const int (&cell)[RPT], const int (&jj)[RPT], int (&src)[RPT]) {
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                src[i] = -1;
                if (cell[i] >= 0) {
                    int n, gy, gx;
                    cell_decode(args, cell[i], n, gy, gx);
                    const int jy = args.fd_hs.div(jj[i]);
                    const int hy = gy * args.S_in - 1 + jy, hx = gx * args.S_in - 1 + (jj[i] - jy * hs);
                    if (hy >= 0 && hy < args.H && hx >= 0 && hx < args.W) src[i] = (n * args.H + hy) * args.W + hx;
                }
            }
        };
        int cell[RPT], jj[RPT], src[RPT], src_next[RPT];
        load_cells(blockIdx.x, cell, jj);
        decode(cell, jj, src);
        int it = 0;
        for (int tile = blockIdx.x; tile < geo.num_tiles; tile += gridDim.x) {
            load_cells(tile + gridDim.x, cell, jj);  // next tile: loads in flight during this K-loop
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int stage = it % ST;
                mbar_wait(bar_empty + 8 * stage, ((it / ST) & 1) ^ 1);
                if (pt == 0) KTRACE(it, 3);
                const uint32_t sa = sbase + C::kStageOff + stage * C::kStageBytes;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int row = prow + RSTEP * i;
                    const bool ok = src[i] >= 0;
                    const __nv_bfloat16 *g = ok ? X + (size_t)src[i] * args.a_ld + kb * kBK + pch * 8 : X;
                    cp_async_16(sa + row * 128 + ((pch ^ (row & 7)) << 4), g, ok ? 16u : 0u);
                }
                cp_async_arrive_noinc(bar_full + 8 * stage);
                if (pt == 0) KTRACE(it, 0);
                if (kb == (num_kb >> 1)) decode(cell, jj, src_next);  // mid-loop: off the tile boundary
            }
#pragma unroll
            for (int i = 0; i < RPT; ++i) src[i] = src_next[i];
        }
        }  // CONV1_DYN gather
    } else if (C::kMasker && warp >= C::kMaskerWarp0) {
        // -------------------------------------- masker partials (fused) --
        // 8 warps, two threads per A row (pixel): thread 2r + h reads the 16-B chunks
        // 4h .. 4h+3 of row r's 128-B swizzled row of EVERY K-block (a quarter-warp
        // = 4 rows x 2 halves touches 8 distinct chunk slots: conflict-free) while
        // the MMA consumes the same stage.  Every masker warp waits on every stage,
        // so the mbarrier parity it waits for is always the current one whatever
        // the stage count (a K-block split by parity would skip phases when the
        // stage count is odd and read a stage before it is refilled).  fp32 FFMA
        // sums: the partial a = sum_c wm_c x[p,c] over its half of the channels and
        // the magnitude m = sum_c |wm_c x[p,c]|, two chains each; every channel
        // term passes through at most c_in/16 + 10 fp32 roundings, which
        // decide_gather.cu's certified bound accounts for.  Fixed channel order.
        const int mt = tid - 32 * C::kMaskerWarp0;
        const int r = mt >> 1, h = mt & 1;
        int it = 0;
        for (int i = 0;; ++i) {
            const int tile = walk.at(i);
            if (tile < 0) break;
            float acc0 = 0.f, acc1 = 0.f, mag0 = 0.f, mag1 = 0.f;
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int stage = it % ST;
                mbar_wait(bar_full + 8 * stage, (it / ST) & 1);
                const uint32_t row = sbase + C::kStageOff + stage * C::kStageBytes + r * 128;
                uint32_t q[4][4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(q[jj][0]), "=r"(q[jj][1]), "=r"(q[jj][2]), "=r"(q[jj][3])
                                 : "r"(row + (((4 * h + jj) ^ (r & 7)) << 4)));
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_empty + 8 * stage);  // this warp's reads are done
                const float4 *w4 = reinterpret_cast<const float4 *>(wm_s + kb * kBK + 32 * h);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const float4 wa = C::kWmSmem ? w4[2 * jj] : __ldg(w4 + 2 * jj);
                    const float4 wb = C::kWmSmem ? w4[2 * jj + 1] : __ldg(w4 + 2 * jj + 1);
                    const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
                    float cs = 0.f, ms = 0.f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float lo = bf16lo(q[jj][e]), hi = bf16hi(q[jj][e]);
                        cs = fmaf(wv[2 * e], lo, cs);
                        cs = fmaf(wv[2 * e + 1], hi, cs);
                        ms = fmaf(fabsf(wv[2 * e]), fabsf(lo), ms);
                        ms = fmaf(fabsf(wv[2 * e + 1]), fabsf(hi), ms);
                    }
                    if (jj & 1) { acc1 += cs; mag1 += ms; } else { acc0 += cs; mag0 += ms; }
                }
            }
            const int m = (tile / geo.n_tiles_n) * kBM + r;
            if (tile % geo.n_tiles_n == 0 && m < args.m_dense)
                reinterpret_cast<float2 *>(args.mpart)[2 * m + h] = make_float2(acc0 + acc1, mag0 + mag1);
        }
    } else if (warp == C::kMmaWarp) {
        // ---------------------------------------------------- MMA issuer --
        if (lane == 0 && lead) {
            constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * kBM : kBM, BN);
            if (C::kBRes) mbar_wait(bar_bres, 0);
            int it = 0, lt = 0;
            for (int i = 0; walk.at(i) >= 0; ++i, ++lt) {
                const int acc = lt & 1;
                if (PAIR) mbar_wait_cluster(bar_tempty + 8 * acc, ((lt >> 1) & 1) ^ 1);
                else mbar_wait(bar_tempty + 8 * acc, ((lt >> 1) & 1) ^ 1);
                tc_fence_after();
                TRACE(lt, 2);
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < num_kb; ++kb, ++it) {
                    const int stage = it % ST;
                    mbar_wait(bar_full + 8 * stage, (it / ST) & 1);
                    KTRACE(it, 2);
                    if (C::kGather) fence_proxy_async_smem();  // cp.async (generic) -> tcgen05 (async)
                    tc_fence_after();
                    const uint32_t sa = sbase + C::kStageOff + stage * C::kStageBytes;
                    const uint64_t adesc = smem_desc_sw128(sa);
                    if (MODE == STEM) {  // input row kb: kernel row kb - 2 j of output row j (TMEM columns 64 j..)
                        constexpr uint32_t idesc64 = idesc_bf16_f32(kBM, 64);
#pragma unroll
                        for (int j = 0; j < kStemRows; ++j) {
                            const int kr = kb - 2 * j;
                            if (kr < 0 || kr > 6) continue;
                            const uint64_t bd = smem_desc_sw128(sbase + kr * C::kBBytes);
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk)
                                mma_bf16(d_tmem + 64 * j, adesc + 2 * kk, bd + 2 * kk, idesc64, (kr | kk) != 0);
                        }
                        mma_commit(bar_empty + 8 * stage);
                        continue;
                    }
                    const uint64_t bdesc = smem_desc_sw128(C::kBRes ? sbase + kb * C::kBBytes : sa + kABytes);
                    if (PAIR) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            mma_bf16_pair(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                        mma_commit_pair_mc(bar_empty + 8 * stage, 3);
                        continue;
                    }
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        mma_bf16(d_tmem, adesc + 2 * kk, bdesc + 2 * kk, idesc, (kb | kk) != 0);
                    mma_commit(bar_empty + 8 * stage);
                }
                if (PAIR) mma_commit_pair_mc(bar_tfull + 8 * acc, 3);
                else mma_commit(bar_tfull + 8 * acc);
                TRACE(lt, 3);
            }
        }
        __syncwarp();
    } else if (warp < C::kEpiWarps) {
        // ------------------------------------------------------- epilogue --
        // warp -> TMEM lane quarter (warp % 4) and column range [c_lo, c_hi)
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // tile row == TMEM lane
        constexpr int kCols = BN / (C::kEpiWarps / 4);
        const int c_lo = (warp >> 2) * kCols;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const int M = gemm_rows(MODE, args);
        const __nv_bfloat16 *X = static_cast<const __nv_bfloat16 *>(args.resid);
        __nv_bfloat16 *Y = static_cast<__nv_bfloat16 *>(args.out);
        // conv3: output pixel of a GEMM row, in two halves so the idx load can be
        // issued early: row_cell (volatile load of idx[patch]) then cell_pixel.
        auto row_cell = [&](int tl) -> int {
            if (tl >= geo.num_tiles) return -2;
            const int m = (tl / geo.n_tiles_n) * kBM + r;
            if (m >= M) return -2;
            if (MODE != CONV3_DYN) return -1;
            return ld_nc_volatile(args.idx + args.fd_SS.div(m));
        };
        auto cell_pixel = [&](int tl, int cell) -> int {
            if (cell == -2) return -1;
            const int m = (tl / geo.n_tiles_n) * kBM + r;
            if (MODE != CONV3_DYN) return m;
            int n, gy, gx;
            cell_decode(args, cell, n, gy, gx);
            const int j = m - args.fd_SS.div(m) * args.S * args.S;
            const int py = args.fd_S.div(j);
            const int yy = gy * args.S + py, xx = gx * args.S + (j - py * args.S);
            return (yy < args.H && xx < args.W) ? (n * args.H + yy) * args.W + xx : -1;  // R7 clip
        };
        // conv3: rows x 16-B chunks of this warp's [32 rows] x [kCols columns] block
        constexpr int kChunks = kCols / 8;
        constexpr int kRowsPerIt = 32 / kChunks;
        auto chunk_addr = [&](uint32_t buf, int rl, int c16) -> uint32_t {
            const int row = quarter * 32 + rl;
            const int col = c_lo + c16 * 8;  // column within the tile
            return buf + (col >> 6) * kChunkBytes + row * 128 + ((((col & 63) >> 3) ^ (row & 7)) << 4);
        };
        auto prefetch_resid = [&](int tl, int mypix, uint32_t buf) {
            if (tl < geo.num_tiles && X != nullptr) {  // no residual tensor: nothing to stage
                const int n0 = (tl % geo.n_tiles_n) * BN;
#pragma unroll
                for (int i = 0; i < 32 / kRowsPerIt; ++i) {
                    const int rl = i * kRowsPerIt + lane / kChunks, c16 = lane % kChunks;
                    const int pix = __shfl_sync(0xffffffffu, mypix, rl);
                    const bool ok = pix >= 0 && X != nullptr;  // no residual tensor: zero-fill
                    const __nv_bfloat16 *g = ok ? X + (size_t)pix * args.out_ld + n0 + c_lo + c16 * 8 : Y;
                    cp_async_16(chunk_addr(buf, rl, c16), g, ok ? 16u : 0u);
                }
            }
            cp_async_commit();
        };
        int lt = 0;
        // tile of the local unit u (past the end: an invalid tile, nothing staged or stored)
        auto tile_at = [&](int i) -> int { const int t = walk.at(i); return t < 0 ? geo.num_tiles : t; };
        int pix_ring[NSTG];  // output pixel of this thread's row for tiles lt .. lt+NSTG-2 (rotated)
#pragma unroll
        for (int k = 0; k < NSTG; ++k) pix_ring[k] = -1;
        if (kResid) {  // residual of the first NSTG-1 tiles
#pragma unroll
            for (int k = 0; k < NSTG - 1; ++k) {
                const int tl = tile_at(k);
                pix_ring[k] = cell_pixel(tl, row_cell(tl));
                prefetch_resid(tl, pix_ring[k], staging + k * C::kStagingBytes);
            }
        }
        for (int i = 0;; ++i, ++lt) {
            const int tile = walk.at(i);
            if (tile < 0) break;
            const int mt = tile / geo.n_tiles_n;
            const int n0 = (tile - mt * geo.n_tiles_n) * BN;
            const int acc = lt & 1, b = lt % NSTG;
            const uint32_t sbuf = staging + b * C::kStagingBytes;
            bool zero = false;  // conv1: halo pixel outside the image stores 0 (R6)
            if (MODE == CONV1_DYN) zero = mt * kBM + r < M && halo_pixel(args, mt * kBM + r, M) < 0;
            bool relu = !args.no_relu;
            if ((MODE == CONV3_DENSE || MODE == PROJ_SC) && args.relu_mask != nullptr) {
                // dynamic projection shortcut: ReLU(R) on inactive cells, R itself on active ones
                int n = -1, yy = 0, xx = 0;
                if (args.view4) {  // dense tile geometry (rows_h x cols_w pixels of imgs_box images)
                    int t0n, t0y, t0x;
                    dense_tile_origin(args, mt, t0n, t0y, t0x);
                    const int per_img = args.cols_w * args.rows_h, im = r / per_img, rr = r - im * per_img;
                    yy = t0y + rr / args.cols_w;
                    xx = t0x + rr % args.cols_w;
                    n = t0n + im;
                    if (n >= args.n_img || yy >= args.H || xx >= args.W || r >= args.box_rows) n = -1;
                } else {
                    const int m = mt * kBM + r;
                    if (m < M) {
                        n = args.fd_HW.div(m);
                        const int rem = m - n * (int)args.fd_HW.d;
                        yy = args.fd_W.div(rem);
                        xx = rem - yy * args.W;
                    }
                }
                if (n >= 0) {
                    const int cell = (n * args.Gh + args.fd_S.div(yy)) * args.Gw + args.fd_S.div(xx);
                    relu = __ldg(args.relu_mask + cell) == 0;
                }
            }
            if constexpr (C::kHalfStage) {
                // BN / CP passes of CP columns through the one staging buffer: pass p stages columns
                // [CP p, CP p + CP) (warp: its 32 rows x CP / 2 columns) and TMA-stores them
                constexpr int CP = 64 * C::kStagingChunks, NP = BN / CP;
                mbar_wait(bar_tfull + 8 * acc, (lt >> 1) & 1);
                tc_fence_after();
                const int row0 = MODE == CONV2_GATHER ? mt * args.units_per_tile * args.S * args.S : mt * kBM;
#pragma unroll 1
                for (int p = 0; p < NP; ++p) {
                    const int qp = NP * lt + p;  // pass counter: the buffer's use
                    mbar_wait(bar_sempty, (qp & 1) ^ 1);
#pragma unroll 1
                    for (int cc = 0; cc < CP / 2; cc += 32) {
                        const int c = CP * p + (warp >> 2) * (CP / 2) + cc, hc = c - CP * p;
                        uint32_t v[32];
                        tmem_ld32(tmem_base + lane_base + acc * BN + c, v);
                        tmem_ld_wait();
                        const uint32_t rowbase = staging + (hc >> 6) * kChunkBytes + r * 128;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint32_t saddr = rowbase + ((((hc & 63) >> 3) + q) ^ (r & 7)) * 16;
                            const float4 b0 = __ldg(reinterpret_cast<const float4 *>(args.bias + n0 + c + 8 * q));
                            const float4 b1 = __ldg(reinterpret_cast<const float4 *>(args.bias + n0 + c + 8 * q + 4));
                            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                            uint32_t pk[4];
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float lo = __uint_as_float(v[8 * q + 2 * e]) + bb[2 * e];
                                float hi = __uint_as_float(v[8 * q + 2 * e + 1]) + bb[2 * e + 1];
                                if (relu) lo = fmaxf(lo, 0.f), hi = fmaxf(hi, 0.f);
                                if (zero) lo = hi = 0.f;
                                pk[e] = pack_bf16x2(lo, hi);
                            }
                            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(pk[0]), "r"(pk[1]),
                                         "r"(pk[2]), "r"(pk[3])
                                         : "memory");
                        }
                    }
                    if (p == NP - 1) {  // every TMEM read of this tile is done
                        tc_fence_before();
                        mbar_arrive(bar_tempty + 8 * acc);
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(1, EPI);
                    if (tid == 0) {
                        for (int c2 = 0; c2 < C::kStagingChunks; ++c2) {
                            const uint32_t src = staging + c2 * kChunkBytes;
                            if (MODE == CONV2_GATHER || ((MODE == PROJ_SC) && !args.view4)) {
                                tma_store_2d(&args.tmap_out, src, n0 + CP * p + 64 * c2, row0);
                            } else if ((MODE == PROJ_SC)) {  // the 4-D output view of the dense tile
                                int d2n, d2y, d2x;
                                dense_tile_origin(args, mt, d2n, d2y, d2x);
                                tma_store_4d(&args.tmap_out, src, n0 + CP * p + 64 * c2, d2x, d2y, d2n);
                            } else {  // conv1: h1 [c_mid/64][rows][64]
                                tma_store_3d(&args.tmap_out, src, 0, mt * kBM, ((n0 + CP * p) >> 6) + c2);
                            }
                        }
                        bulk_commit();
                        bulk_wait_read<0>();  // the buffer is free once this store has read it
                        mbar_arrive(bar_sempty);
                    }
                }
                continue;
            }
            int cell_ahead = -2;
            if (kResid) {
                cell_ahead = row_cell(tile_at(i + NSTG - 1));  // idx load in flight during this tile
                cp_async_wait<NSTG - 2>();  // this tile's residual has landed
                __syncwarp();
            } else {
                // staging buffer b is free once the store of tile lt - NSTG has read it
                mbar_wait(bar_sempty + 8 * b, ((lt / NSTG) & 1) ^ 1);
            }
            mbar_wait(bar_tfull + 8 * acc, (lt >> 1) & 1);
            tc_fence_after();
            if (tid == 0) TRACE(lt, 4);
#pragma unroll 1
            for (int c = c_lo; c < c_lo + kCols; c += 32) {
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
                    for (int e = 0; e < 8; ++e)  // (stem: columns 64-127 are the second row's 64 channels)
                        f[e] = __uint_as_float(v[8 * q + e]) + bias_s[(n0 + c + 8 * q + e) & (MODE == STEM ? 63 : 0x7fffffff)];
                    if (kResid && X != nullptr) {
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
                        float lo = f[2 * e], hi = f[2 * e + 1];
                        if (relu) lo = fmaxf(lo, 0.f), hi = fmaxf(hi, 0.f);
                        if (zero) lo = hi = 0.f;
                        pk[e] = pack_bf16x2(lo, hi);
                    }
                    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(pk[0]), "r"(pk[1]),
                                 "r"(pk[2]), "r"(pk[3])
                                 : "memory");
                }
            }
            tc_fence_before();
            if (PAIR) {  // the lead's MMA waits for the epilogue warps of both CTAs
                __syncwarp();
                if (lane == 0) {
                    if (lead) mbar_arrive(bar_tempty + 8 * acc);
                    else mbar_arrive_cluster(bar_tempty + 8 * acc, 0);
                }
            } else {
                mbar_arrive(bar_tempty + 8 * acc);
            }
            if (kResid && MODE == CONV3_DENSE && args.tma_y) {
                // dense rows: the staged (128-B swizzled) tile is y's rows [mt*128, +128) --
                // one TMA store per 64-column chunk (rows past the end are clipped); the
                // buffer the next prefetch reuses was read by the previous tile's store
                fence_proxy_async_smem();
                named_bar_sync(1, EPI);
                if (tid == 0) {
                    if (args.view4) {  // y through the 4-D output view of the dense tile
                        int t0n, t0y, t0x;
                        dense_tile_origin(args, mt, t0n, t0y, t0x);
                        for (int c = 0; c < BN / 64; ++c)
                            tma_store_4d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, t0x, t0y, t0n);
                    } else {
                        for (int c = 0; c < BN / 64; ++c)
                            tma_store_2d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, mt * kBM);
                    }
                    bulk_commit();
                    bulk_wait_read<1>();
                }
                named_bar_sync(1, EPI);
            } else if (kResid) {
                // scatter-add store: the warp's 32 rows x kCols columns, 16-B chunks,
                // kRowsPerIt rows per instruction (full 128-B lines)
                __syncwarp();
                const int mypix = pix_ring[0];
#pragma unroll
                for (int i = 0; i < 32 / kRowsPerIt; ++i) {
                    const int rl = i * kRowsPerIt + lane / kChunks, c16 = lane % kChunks;
                    const int pix = __shfl_sync(0xffffffffu, mypix, rl);
                    uint32_t o[4];
                    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3])
                                 : "r"(chunk_addr(sbuf, rl, c16)));
                    if (pix >= 0)
                        *reinterpret_cast<uint4 *>(Y + (size_t)pix * args.out_ld + n0 + c_lo + c16 * 8) =
                            make_uint4(o[0], o[1], o[2], o[3]);
                }
                __syncwarp();
            }
            if (kResid) {
                // residual prefetch for tile lt+NSTG-1 into the buffer tile lt-1 used
                const int ahead = tile_at(i + NSTG - 1);
                const int slot = (lt + NSTG - 1) % NSTG;
#pragma unroll
                for (int k = 0; k + 1 < NSTG - 1; ++k) pix_ring[k] = pix_ring[k + 1];
                pix_ring[NSTG - 2] = cell_pixel(ahead, cell_ahead);
                prefetch_resid(ahead, pix_ring[NSTG - 2], staging + slot * C::kStagingBytes);
                if (tid == 0) TRACE(lt, 6);
                continue;
            }
            fence_proxy_async_smem();  // staging writes -> visible to the TMA store
            named_bar_sync(1, EPI);
            if (tid == 0) TRACE(lt, 5);
            if (tid == 0) {
                if (MODE == CONV2_DENSE || (MODE == PROJ_SC && args.view4)) {  // 4-D output view of the dense tile
                    int d2n, d2y, d2x;
                    dense_tile_origin(args, mt, d2n, d2y, d2x);
                    for (int c = 0; c < BN / 64; ++c)
                        tma_store_4d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, d2x, d2y, d2n);
                } else if (MODE == STEM) {  // the tile's rows in residue order back to output columns
                    const int xb = mt % args.tiles_x, row = mt / args.tiles_x;
                    const int groups = (args.H + kStemRows - 1) / kStemRows;
                    const int n = row / groups, oy0 = kStemRows * (row - n * groups);
                    const int q = args.cols_w / 4;
                    for (int r2 = 0; r2 < kStemRows; ++r2)  // 64-column chunk r2 = output row oy0 + r2 (rows >= H: clipped)
                        for (int k = 0; k < 4; ++k)
                            tma_store_4d(&args.tmap_s[4 + k], sbuf + r2 * kChunkBytes + k * q * 128, 0, xb * q,
                                         oy0 + r2, n);
                } else if (MODE == CONV1_DYN || MODE == CONV1_DENSE || MODE == CONV1_DENSE_MASK) {  // h1: [c_mid/64][rows][64]
                    for (int c = 0; c < BN / 64; ++c)
                        tma_store_3d(&args.tmap_out, sbuf + c * kChunkBytes, 0, mt * kBM, (n0 >> 6) + c);
                } else {
                    const int row0 = (MODE == CONV2_DYN || MODE == CONV2_GATHER) ? mt * args.units_per_tile * args.S * args.S
                                                                                 : mt * kBM;
                    for (int c = 0; c < BN / 64; ++c)
                        tma_store_2d(&args.tmap_out, sbuf + c * kChunkBytes, n0 + c * 64, row0);
                }
                bulk_commit();
                TRACE(lt, 6);
                if (NSTG == 1) {
                    bulk_wait_read<0>();  // single buffer: free it as soon as this store has read it
                    mbar_arrive(bar_sempty);
                } else {
                    bulk_wait_read<1>();  // the previous tile's store has read its buffer
                    if (lt >= 1) mbar_arrive(bar_sempty + 8 * ((lt - 1) % NSTG));
                }
            }
        }
        if (tid == 0 && (!kResid || (MODE == CONV3_DENSE && args.tma_y))) bulk_wait_all<0>();
    }

    tc_fence_before();
    // pair: no CTA leaves while its peer may still arrive on its barriers or its MMAs write its TMEM
    if (PAIR) cluster_sync();
    else __syncthreads();
    if (warp == C::kMmaWarp) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair<C::kTmemCols>(tmem_base);
        else tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// ----------------------------------------------------------------- host ----

template <int MODE, int BN, bool PAIR>
static cudaError_t launch_mode_bn(const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    auto kern = conv_tc_kernel<MODE, BN, PAIR>;
    const int smem = Cfg<MODE, BN, PAIR>::smem_bytes(a.N, a.K);
    static int configured = 0;  // per instantiation: largest dynamic smem enabled so far
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    if (PAIR) {  // whole pairs, at most one CTA per SM
        const long units = (long)(max_tiles_m + 1) / 2 * (a.N / BN);
        const int cap = num_sms / 2;
        const int pairs = (int)(units < cap ? (units > 0 ? units : 1) : cap);
        return launch_k_cluster(kern, dim3(2 * pairs), dim3(threads_of<MODE, BN>()), smem, st, 2, a);
    }
    const long tiles = (long)max_tiles_m * (a.N / BN);
    const int grid = (int)(tiles < num_sms ? (tiles > 0 ? tiles : 1) : num_sms);
    return launch_k(kern, dim3(grid), dim3(threads_of<MODE, BN>()), smem, st, a);
}

// LASNET_TC_PAIR=0: no 2-SM pairs (the 256-column conv2 tiles run one CTA per tile)
static bool pairs_enabled() {
    static const bool on = [] {
        const char *e = getenv("LASNET_TC_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

// conv2 (dynamic) without pairs stays on 128-column tiles: 256-column tiles measured no faster
// (stage-3 blocks of LAS-R101: 1.121 vs 1.115 ms over 26 launches); LASNET_CONV2_BN=256 opts in
static bool conv2_bn256() {
    static const bool on = [] {
        const char *e = getenv("LASNET_CONV2_BN");
        return e && atoi(e) == 256;
    }();
    return on;
}

// N tile of a conv_tc launch and whether it runs on CTA pairs; the host encodes the
// weight (B) box with bn / 2 rows for a pair (each CTA stages half of the N rows).
int conv_tc_plan(int mode, int n, int *pair) {
    *pair = 0;
    if (n % 128 != 0) return 64;  // 64-column N tiles
    if ((mode == CONV2_DYN || mode == CONV2_DENSE) && n % 256 == 0 && pairs_enabled()) {
        *pair = 1;
        return 256;
    }
    // 256-column tiles: A (the gathered rows / the im2col taps) is staged once per M
    // tile instead of once per 128-column N tile
    if (n % 256 == 0 && (mode == CONV1_DYN || mode == CONV1_DENSE || mode == CONV1_DENSE_MASK || mode == CONV2_GATHER ||
                         mode == PROJ_SC ||
                         (mode == CONV2_DYN && conv2_bn256())))
        return 256;
    return 128;
}

template <int MODE>
static cudaError_t launch_mode(const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    int pair = 0;
    const int bn = conv_tc_plan(MODE, a.N, &pair);
    if (pair != a.pair_tc) return cudaErrorInvalidValue;  // the host encoded B for the other plan
    constexpr bool kResid = MODE == CONV3_DYN || MODE == CONV3_DENSE;
    if constexpr (MODE == CONV2_DYN || MODE == CONV2_DENSE) {
        if (pair && bn == 256) return launch_mode_bn<MODE, 256, true>(a, max_tiles_m, num_sms, st);
    }
    if (bn == 64) return launch_mode_bn<MODE, 64, false>(a, max_tiles_m, num_sms, st);
    if constexpr (!kResid) {
        if (bn == 256) return launch_mode_bn<MODE, 256, false>(a, max_tiles_m, num_sms, st);
    }
    if (bn == 128) return launch_mode_bn<MODE, 128, false>(a, max_tiles_m, num_sms, st);
    return cudaErrorInvalidValue;
}

// max_tiles_m: capacity bound on the M tiles (grid sizing only; dynamic modes
// derive the true tile count from the device count).
cudaError_t launch_conv_tc(int mode, const ConvArgs &a, int max_tiles_m, int num_sms, cudaStream_t st) {
    if (a.K % kBK != 0) return cudaErrorInvalidValue;
    switch (mode) {
        case CONV1_DYN: return launch_mode<CONV1_DYN>(a, max_tiles_m, num_sms, st);
        case CONV2_DYN: return launch_mode<CONV2_DYN>(a, max_tiles_m, num_sms, st);
        case CONV2_GATHER: return launch_mode<CONV2_GATHER>(a, max_tiles_m, num_sms, st);
        case CONV3_DYN: return launch_mode<CONV3_DYN>(a, max_tiles_m, num_sms, st);
        case CONV1_DENSE: return launch_mode<CONV1_DENSE>(a, max_tiles_m, num_sms, st);
        case CONV1_DENSE_MASK: return launch_mode<CONV1_DENSE_MASK>(a, max_tiles_m, num_sms, st);
        case CONV2_DENSE: return launch_mode<CONV2_DENSE>(a, max_tiles_m, num_sms, st);
        case CONV3_DENSE: return launch_mode<CONV3_DENSE>(a, max_tiles_m, num_sms, st);
        case PROJ_SC: return launch_mode<PROJ_SC>(a, max_tiles_m, num_sms, st);
        case STEM: {  // BN = 128: the two output rows' 64-channel accumulators (four rows, BN 256: 0.32 -> 0.36 ms)
            auto kern = conv_tc_kernel<STEM, 128, false>;
            const int smem = Cfg<STEM, 128>::smem_bytes(64, a.K);
            static int configured = 0;
            if (smem > configured) {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
                configured = smem;
            }
            const int grid = max_tiles_m < num_sms ? (max_tiles_m > 0 ? max_tiles_m : 1) : num_sms;
            return launch_k(kern, dim3(grid), dim3(threads_of<STEM, 128>()), smem, st, a);
        }
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lasnet

#ifdef LASNET_TRACE
extern "C" int lasnet_trace_read(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, lasnet::g_trace, sizeof(unsigned long long) * (n < 512 ? n : 512));
}
extern "C" int lasnet_trace_clear(int mode) {
    static unsigned long long z[512];
    cudaMemcpyToSymbol(lasnet::g_trace_mode, &mode, sizeof(int));
    cudaMemcpyToSymbol(lasnet::g_ktrace, z, sizeof(z));
    return (int)cudaMemcpyToSymbol(lasnet::g_trace, z, sizeof(z));
}
extern "C" int lasnet_ktrace_read(unsigned long long *host) {
    return (int)cudaMemcpyFromSymbol(host, lasnet::g_ktrace, sizeof(unsigned long long) * 512);
}
#endif

/*
 * lasnet.h -- C ABI of the B200-native LASNet coarse-grained spatially-dynamic
 * residual block (arXiv 2210.06223, "Latency-aware Spatial-wise Dynamic
 * Networks").  Citations: P:n = PAPER.md line n.
 *
 * The block (sec. 3.1, sec. 3.2 / Fig. 2, sec. 3.4,
 * P:556-577 App. B) runs as five steps:
 *   1 masker      lasnet_mask      pooled 1x1 conv + hard threshold -> S x S patch mask
 *   2 compaction  lasnet_compact   ascending index list of activated patches + count
 *   (1+2 fused:   lasnet_mask_compact, one launch)
 *   3 gather+conv1                 \
 *   4 conv2 (3x3)                   > lasnet_dyn_block
 *   5 conv3+scatter-add            /
 * and lasnet_dense_block runs the same convolutions on every pixel (the static
 * counterpart) as the comparator.
 *
 * Conventions for every entry point
 *  - Pointers are DEVICE pointers unless stated otherwise.  The caller owns and
 *    frees every buffer, including the workspace; the library never allocates
 *    device memory and keeps no per-call state.
 *  - Every call only enqueues work on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Results are valid once the stream has synchronised.
 *    The active-patch count never leaves the device: kernels read it from
 *    device memory, so the sequence mask -> compact -> dyn_block needs no host
 *    synchronisation and is CUDA-graph capturable.
 *  - Arguments are validated on the host before anything is launched.  On any
 *    error status nothing is launched and no output is touched.  No C++
 *    exception crosses this ABI.  Launch failures are reported as
 *    LASNET_ERR_CUDA (from cudaGetLastError()).
 *  - Layouts: activations NHWC, channels innermost; a pixel row is c*elt bytes.
 *    bf16 tensors are IEEE bfloat16 bit patterns (uint16).  Device pointers must
 *    be 16-byte aligned.
 *  - The bf16 path (dtype LASNET_BF16) runs tcgen05 tensor-core kernels fed by
 *    TMA: c_in a multiple of 64, c_mid and c_out equal to 64 or multiples of 128
 *    (at most 2048), s <= 11, w <= 128.  The fp32 path (LASNET_F32) runs fp32
 *    CUDA-core kernels: all channels multiples of 64.  Other valid shapes return
 *    LASNET_ERR_UNSUPPORTED.  lasnet_mask alone only needs c_in % 8 (bf16) or
 *    % 4 (fp32).
 */
#ifndef LASNET_H
#define LASNET_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LASNET_ABI_VERSION 2

typedef enum {
    LASNET_OK = 0,
    LASNET_ERR_NULL = 1,        /* a required pointer is NULL                            */
    LASNET_ERR_SHAPE = 2,       /* non-positive or inconsistent sizes                    */
    LASNET_ERR_DOMAIN = 3,      /* S < 1, stride not in {1,2}, unknown dtype             */
    LASNET_ERR_UNSUPPORTED = 4, /* valid but not built: channel multiples, stride 2      */
    LASNET_ERR_ALIAS = 5,       /* y partially overlaps x (only y == x is allowed)       */
    LASNET_ERR_WORKSPACE = 6,   /* workspace NULL or smaller than the *_workspace_bytes  */
    LASNET_ERR_CUDA = 7         /* a CUDA launch or runtime call failed                  */
} lasnet_status;

typedef enum { LASNET_F32 = 0, LASNET_BF16 = 1 } lasnet_dtype;

/* cudaStream_t without pulling in the CUDA headers. */
typedef struct CUstream_st *lasnet_stream_t;

/* Shape of one bottleneck block.  h, w are the OUTPUT spatial dims; the mask
 * lives on the output grid ("the corresponding location of the output
 * feature").  The coarse grid is gh = ceil(h/s) x gw = ceil(w/s); edge patches
 * are clipped when s does not divide h or w (reading R7). */
typedef struct {
    int32_t n, h, w;              /* batch, output height, output width              */
    int32_t c_in, c_mid, c_out;   /* bottleneck widths; identity block: c_in == c_out */
    int32_t stride;               /* 1, or 2 for a stage's first (projection) block   */
    int32_t s;                    /* spatial granularity S >= 1               */
    int32_t dtype;                /* lasnet_dtype of x, y and w1..w3                  */
} lasnet_block_desc;

/* BN-folded weights.  Biases are fp32; w1..w3 have the block dtype.
 *   w1 [c_mid][c_in]            conv1 1x1, K-major
 *   w2 [c_mid][3][3][c_mid]     conv2 3x3, OHWI (K = 9*c_mid, tap-major)
 *   w3 [c_out][c_mid]           conv3 1x1
 *   wd [c_out][c_in], bd [c_out] the 1x1 (stride-s) projection shortcut of lasnet_proj_block;
 *                               must be NULL for the identity-block calls */
typedef struct {
    const void *w1; const float *b1;
    const void *w2; const float *b2;
    const void *w3; const float *b3;
    const void *wd; const float *bd;
} lasnet_block_weights;

/* Step 1 -- masker ("a pooling layer followed by a 1x1 convolution";
 * App. B: the 2-channel argmax reduces to x*(W_0 - W_1) > 0).
 *   x      [n][h][w][c_in] (block dtype)
 *   wm     [c_in] fp32, the reduced weight W_0 - W_1
 *   bm     reduced bias b_0 - b_1 (host scalar)
 *   mask   [n][gh][gw] uint8 out: 1 iff logit > 0 (ties inactive, R3)
 *   logits [n][gh][gw] fp64 out, nullable: logit = sum_c wm_c * avgpool_c(x) + bm,
 *          average over the in-image pixels of the cell (R1, R7).
 * The decision is the one exact arithmetic takes (reading R20): fp32
 * accumulation with a rigorous rounding bound, and an fp64 re-sum of any cell
 * whose logit the bound does not separate from 0; logits (if requested) are
 * accumulated in fp64. */
lasnet_status lasnet_mask(const lasnet_block_desc *desc, const void *x, const float *wm,
                          float bm, uint8_t *mask, double *logits, lasnet_stream_t stream);

/* Steps 1+2 fused in one launch (App. B: "the masker generates the
 * indices of activated patches"): the same logits and decisions as lasnet_mask,
 * and the same idx/count as lasnet_compact on that mask.
 *   mask, logits  nullable outputs as in lasnet_mask
 *   idx [n*gh*gw], count   as in lasnet_compact
 *   ws     lasnet_mask_compact_workspace_bytes(desc) bytes that must be ALL ZERO
 *          before the first call; every call leaves them all zero again.
 *          Concurrent calls must not share a workspace. */
lasnet_status lasnet_mask_compact(const lasnet_block_desc *desc, const void *x, const float *wm, float bm,
                                  uint8_t *mask, double *logits, int32_t *idx, int32_t *count, void *ws,
                                  size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_mask_compact_workspace_bytes(const lasnet_block_desc *desc);

/* Step 2 -- compaction (App. B P:568-569 "the masker generates the indices of
 * activated patches instead of sparse mask").
 *   mask   [ncells] uint8 (ncells = n*gh*gw), nonzero = active
 *   idx    [ncells] int32 out: ascending linear cell ids n*gh*gw + gy*gw + gx of
 *          the active cells in idx[0 .. count-1]; the rest is untouched
 *   count  int32 device scalar out
 *   ws     device workspace of lasnet_compact_workspace_bytes(ncells) bytes
 * ncells == 0 is valid (count = 0). */
lasnet_status lasnet_compact(const uint8_t *mask, int32_t ncells, int32_t *idx,
                             int32_t *count, void *ws, size_t ws_bytes,
                             lasnet_stream_t stream);
size_t lasnet_compact_workspace_bytes(int32_t ncells);

/* Steps 3-5 -- the dynamic bottleneck on the activated patches
 * (P:89 gather -> compute -> scatter; P:162-166 gather fused into the dynamic
 * conv; P:168-170, P:574-577 scatter fused with the residual add).
 * For every active cell idx[t], t < *count:
 *   h1 = ReLU(conv1(x) + b1) on the (s+2)x(s+2) halo window, 0 outside the image (R6)
 *   h2 = ReLU(conv3x3_valid(h1, w2) + b2)                  -> s x s
 *   y  = ReLU(x + conv1x1(h2, w3) + b3) on the in-image pixels of the patch (R5, R7)
 * Pixels of inactive cells keep y = x (input fill, R4).
 *   x, y   [n][h][w][c_in]; y == x runs in place (inactive pixels cost nothing);
 *          y != x copies x to y first; any partial overlap -> LASNET_ERR_ALIAS
 *   idx, count  output of lasnet_compact (device); cap = capacity of idx (>= *count)
 *   ws     device workspace of lasnet_dyn_workspace_bytes(desc, cap) bytes
 * Intermediates h1/h2 are stored in the block dtype (bf16 RNE or fp32). */
lasnet_status lasnet_dyn_block(const lasnet_block_desc *desc, const lasnet_block_weights *wts,
                               const void *x, void *y, const int32_t *idx,
                               const int32_t *count, int32_t cap, void *ws,
                               size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_dyn_workspace_bytes(const lasnet_block_desc *desc, int32_t cap);

/* The same convolutions on every pixel (static block): y = ReLU(x +
 * conv3(ReLU(conv3x3(ReLU(conv1(x)))))), zero padding 1 for the 3x3.
 *   x, y   [n][h][w][c_in]; y == x allowed (in place); partial overlap -> ERR_ALIAS
 *   ws     lasnet_dense_workspace_bytes(desc) bytes */
lasnet_status lasnet_dense_block(const lasnet_block_desc *desc, const lasnet_block_weights *wts,
                                 const void *x, void *y, void *ws, size_t ws_bytes,
                                 lasnet_stream_t stream);
size_t lasnet_dense_workspace_bytes(const lasnet_block_desc *desc);

/* The projection (first) block of a ResNet stage, static (SURVEY 8(f) NEXT-f1:
 * the first blocks run dense until their dynamic form is built; the paper's
 * LASNet keeps the downsampling shortcut dense):
 *   h1 = ReLU(conv1x1(x) + b1)                  at the input resolution
 *   h2 = ReLU(conv3x3(h1, stride, pad 1) + b2)  at the output resolution
 *   y  = ReLU(conv1x1(h2, w3) + b3 + (wd * x_s + bd)),  x_s = x[:, ::stride, ::stride, :]
 *   desc    h, w are the OUTPUT dims, stride in {1, 2}; s is ignored; bf16 only;
 *           c_in % 64, c_mid 64 or % 128, c_out % 128, w * stride <= 128
 *   x       [n][h*stride][w*stride][c_in];  y [n][h][w][c_out] (must not overlap x)
 *   wts     w1..w3 as above and wd/bd (required)
 *   ws      lasnet_proj_workspace_bytes(desc) bytes, no contract on contents.
 * Stride 2 reads h1 through four parity views (every second pixel and row); conv3
 * and the shortcut run as one GEMM over [h2 | x_s] and [W3 | Wd] (the shortcut
 * output is never stored or rounded). */
lasnet_status lasnet_proj_block(const lasnet_block_desc *desc, const lasnet_block_weights *wts, const void *x,
                                void *y, void *ws, size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_proj_workspace_bytes(const lasnet_block_desc *desc);

/* The rest of a LAS-ResNet around the blocks, bf16 NHWC:
 *
 * lasnet_stem: 7x7 stride-2 convolution, 64 output channels, + bias, ReLU (the
 *   ResNet stem with BN folded) on tensor cores.
 *   x_pad  [n][2h][2w + 8][8]: the image with its 3 channels zero-padded to 8 and
 *          4 zero pixels on the left and right of every row (top/bottom padding
 *          is implicit); h, w are the OUTPUT dims, w % 4 == 0
 *   w      [64][7][7][8] OHWI (channels 3..7 zero), b [64] fp32
 *   y      [n][h][w][64]
 *   ws     lasnet_stem_workspace_bytes() bytes (packed weights), no contract
 * lasnet_maxpool: 3x3 stride-2 max pool, padding 1: x [n][2h][2w][c] -> y [n][h][w][c], c % 8 == 0.
 * lasnet_head: global average pool + fully connected classifier:
 *   x [n][hw][c] (c % 8 == 0), w [classes][c] (bf16), b [classes] fp32 -> logits [n][classes] fp32,
 *   ws lasnet_head_workspace_bytes(n, c) bytes. */
lasnet_status lasnet_stem(int32_t n, int32_t h, int32_t w, const void *x_pad, const void *wt, const float *b, void *y,
                          void *ws, size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_stem_workspace_bytes(void);
lasnet_status lasnet_maxpool(int32_t n, int32_t h, int32_t w, int32_t c, const void *x, void *y,
                             lasnet_stream_t stream);
lasnet_status lasnet_head(int32_t n, int32_t hw, int32_t c, int32_t classes, const void *x, const void *w,
                          const float *b, float *logits, void *ws, size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_head_workspace_bytes(int32_t n, int32_t c);

/* The whole block, steps 1-5, in one call, under one of two schedules.
 *
 * LASNET_SCHED_MASKER_SEPARATE -- the north-star branch: masker + compaction in
 *   one launch (lasnet_mask_compact), then lasnet_dyn_block (gather + conv1 on
 *   the (s+2)^2 halo of each active patch, conv2, conv3 + scatter-add).  The
 *   masker reads all of x once and conv1 reads the halos again.
 * LASNET_SCHED_MASKER_FUSED -- the paper's best schedule (Table 1 last row,
 *   P:336-342; sec. 3.4; App. B): the masker is fused into a
 *   STATIC conv1 that reads x once and computes h1 on every pixel together with
 *   the masker's per-pixel partial logits; one launch then decides every cell,
 *   a second compacts the indices; conv2 reads the (s+2)^2 h1 halo of every
 *   active patch straight out of the dense h1 (the "gather fused into the 3x3
 *   conv" of Table 1: one TMA box per patch and K-block, zero-filled outside the
 *   image) when c_mid <= 128 and s >= 4, else from a gathered copy; conv2 +
 *   conv3 + scatter-add as in lasnet_dyn_block.  bf16 only.
 * Both produce bit-identical mask / idx / count (the decision rule is the one
 * of lasnet_mask: certified fp32 with an exact fp64 re-sum when the bound does
 * not separate the logit from 0) and the same y up to fp32 accumulation order.
 *   x, y     [n][h][w][c_in]; y == x in place, else x is copied to y first;
 *            partial overlap -> LASNET_ERR_ALIAS
 *   wm, bm   masker as in lasnet_mask
 *   schedule lasnet_schedule value, else LASNET_ERR_DOMAIN
 *   mask     [n][gh][gw] uint8 out, nullable
 *   idx      [n*gh*gw] int32 out (capacity = all cells), count int32 device out
 *   ws       lasnet_block_forward_workspace_bytes(desc, schedule) bytes, ALL ZERO
 *            before the first call (its leading control words are left zero by
 *            every call, except one grid-barrier generation word whose value is
 *            arbitrary; the rest is scratch).  Concurrent calls must not share it.
 *
 * A stage's FIRST block (the dynamic projection block, SURVEY 8(f) NEXT-f1;
 * DESIGN.md reading R22) is selected by non-NULL wts->wd / wts->bd: x is
 * [n][h*stride][w*stride][c_in] (stride 1 or 2, desc h, w the OUTPUT dims),
 * y [n][h][w][c_out] must not overlap x, and
 *   R = Wd x_s + bd            dense 1x1 stride-s shortcut, stored bf16
 *   mask on the output grid    the masker pools each cell's (stride*s)^2 input
 *                              window (== lasnet_mask on x at granularity stride*s)
 *   y  = ReLU(R)               on inactive cells
 *   y  = ReLU(R + conv3(h2) + b3) on active cells, h2 the stride-s 3x3 over the
 *                              input window of side stride*(s-1)+3 at origin
 *                              (stride*s*gy - 1, stride*s*gx - 1), conv1 on it
 * Only LASNET_SCHED_MASKER_SEPARATE (else ERR_UNSUPPORTED); bf16; c_in % 64,
 * c_mid 64 or % 128, c_out % 128 (<= 2048); mask may be NULL (kept in ws). */
typedef enum { LASNET_SCHED_MASKER_SEPARATE = 0, LASNET_SCHED_MASKER_FUSED = 1 } lasnet_schedule;
lasnet_status lasnet_block_forward(const lasnet_block_desc *desc, const lasnet_block_weights *wts,
                                   const void *x, void *y, const float *wm, float bm, int32_t schedule,
                                   uint8_t *mask, int32_t *idx, int32_t *count, void *ws, size_t ws_bytes,
                                   lasnet_stream_t stream);
size_t lasnet_block_forward_workspace_bytes(const lasnet_block_desc *desc, int32_t schedule);
/* Host-side schedule choice for an expected activation rate r (the paper's
 * threshold r_th): the lasnet_schedule the B200 latency predictor
 * (lasnet_predict_latency, built-in calibration) predicts faster; a stage's
 * first block (stride 2 or c_in != c_out) always gets MASKER_SEPARATE.  Pure,
 * launches nothing. */
int32_t lasnet_choose_schedule(const lasnet_block_desc *desc, double r);

/* LAS-RegNetY Y-block ("bottleneck structure with
 * different channel numbers and convolution groups ... Squeeze-and-Excitation"),
 * BN folded, bf16, all widths multiples of 64 (RegNet widths zero-padded):
 *   h1  = ReLU(x Wa^T + ba)                         1x1, c_in -> c_mid
 *   h2  = ReLU(gconv3x3(h1, Wb, stride) + bb)       grouped 3x3, group width 16
 *   s   = sigmoid(W2 ReLU(W1 mean(h2) + b1) + b2)   SE; the mean over the computed
 *                                                   pixels (dynamic: the image's
 *                                                   ACTIVE pixels, R23)
 *   y   = ReLU(R + (h2 * s) Wc^T + bc)              R = x, or Wd x_s + bd (projection)
 * Dynamic (wm != NULL; identity only: stride 1, c_in == c_out, no wd): the five
 * steps -- masker + compaction, gather + conv1 on the (s+2)^2 halos, the grouped
 * 3x3 on the gathered windows, SE over the active pixels, conv3 + scatter-add in
 * place; y == x runs in place, else x is copied to y first; inactive pixels keep
 * x; mask nullable.  schedule (dynamic only): LASNET_SCHED_MASKER_SEPARATE
 * (masker + compaction, conv1 on the halos) or LASNET_SCHED_MASKER_FUSED (the
 * paper's Table-1 schedule: conv1 dense with the masker partials, one launch
 * deciding + gathering the h1 windows), as lasnet_block_forward.  Static (wm == NULL): every pixel, stride 1 or 2, y
 * must not overlap x.  h1, h2, h2*s and y are stored bf16 (RNE).
 *   w      weights; se_* fp32 [w_se][c_mid], [w_se], [c_mid][w_se], [c_mid]
 *   ws     lasnet_regnet_workspace_bytes(desc, dynamic) bytes, ALL ZERO before the
 *          first dynamic call (masker control words, left zero by every call). */
typedef struct {
    const void *wa; const float *ba;          /* [c_mid][c_in]                           */
    const void *wb; const float *bb;          /* [c_mid][3][3][16] grouped (OHWI in-group) */
    const float *se_w1; const float *se_b1;   /* [w_se][c_mid], [w_se]                   */
    const float *se_w2; const float *se_b2;   /* [c_mid][w_se], [c_mid]                  */
    int32_t w_se;
    const void *wc; const float *bc;          /* [c_out][c_mid]                          */
    const void *wd; const float *bd;          /* projection [c_out][c_in], or NULL       */
} lasnet_regnet_weights;
lasnet_status lasnet_regnet_block(const lasnet_block_desc *desc, const lasnet_regnet_weights *wts, const void *x,
                                  void *y, const float *wm, float bm, int32_t schedule, uint8_t *mask, int32_t *idx,
                                  int32_t *count, void *ws, size_t ws_bytes, lasnet_stream_t stream);
size_t lasnet_regnet_workspace_bytes(const lasnet_block_desc *desc, int32_t dynamic);
/* RegNet stem: 3x3 stride-2 conv, c_real (<= 64, even) output channels + bias +
 * ReLU, channels c_real..63 written 0: x_pad [n][2h][2w + 8][8] (as lasnet_stem),
 * wt [64][3][3][8] OHWI, b [64] fp32 -> y [n][h][w][64].  CUDA-core kernel. */
lasnet_status lasnet_regnet_stem(int32_t n, int32_t h, int32_t w, int32_t c_real, const void *x_pad, const void *wt,
                                 const float *b, void *y, lasnet_stream_t stream);

/* Latency predictor G(H, P, S, r) (sec. 3.3 "Latency prediction
 * model", App. A) re-targeted to B200.  Host-
 * side, pure: launches nothing.
 *   H  lasnet_hw: the device as `sms` processing engines behind off-chip (HBM),
 *      on-chip (L2 -> shared memory) and in-PE (tensor core) levels, a per-launch
 *      overhead, and per kernel type the achieved fraction of its bound
 *      (lasnet_hw_b200 fills the built-in B200 calibration)
 *   P  desc (layer parameters; stride 2 / c_in != c_out = a stage's first block)
 *   S  desc->s;  r  the activation rate (expected geometry of r*cells uniformly
 *      active cells, border clipping included)
 *   schedule  LASNET_SCHED_MASKER_SEPARATE, LASNET_SCHED_MASKER_FUSED, or
 *      LASNET_SCHED_DENSE (predictor only: the static block, lasnet_dense_block /
 *      lasnet_proj_block) for the latency ratio r_l = l_dyn / l_stat
 * The operators are exactly the launches the library makes for that schedule;
 * each is split into its 128-row GEMM tiles run by a persistent grid of one CTA
 * per SM: t = launch + t0 + ceil(tiles/sms) * max(HBM, L2, tensor time per tile) / eff.
 * Returns the predicted latency in microseconds (-1 on invalid arguments or an
 * unsupported schedule); kinds / kernel_us (nullable, max_kernels entries)
 * receive the per-launch kernel types and predicted times, n_kernels the count. */
typedef enum {
    LASNET_K_MASK_COMPACT = 0, LASNET_K_CONV1_DYN, LASNET_K_CONV1_MASK, LASNET_K_DECIDE, LASNET_K_DECIDE_GATHER,
    LASNET_K_CONV23, LASNET_K_CONV23_DIRECT, LASNET_K_CONV2_DYN, LASNET_K_CONV3_DYN, LASNET_K_CONV1_DENSE,
    LASNET_K_CONV2_DENSE, LASNET_K_CONV3_DENSE, LASNET_K_CONV23_DENSE, LASNET_K_SUBSAMPLE, LASNET_K_SHORTCUT,
    LASNET_K_MASK, LASNET_K_COMPACT, LASNET_K_CONV2_GATHER, LASNET_K_COUNT
} lasnet_kernel_type;
#define LASNET_SCHED_DENSE 2
typedef struct {
    int32_t sms;       /* processing engines (SMs)                                  */
    double hbm_gbs;    /* off-chip memory bandwidth, GB/s                           */
    double l2_gbs;     /* on-chip (L2 -> shared memory) bandwidth, GB/s, all SMs    */
    double tc_tflops;  /* dense bf16 tensor throughput, TFLOP/s                     */
    double launch_us;  /* per-kernel launch / fill / drain, us                      */
    double eff[LASNET_K_COUNT]; /* achieved fraction of the bound per kernel type   */
    double t0_us[LASNET_K_COUNT]; /* fixed per-launch cost per kernel type (pipeline
                                     fill, tails, dependent latency chains), us    */
} lasnet_hw;
void lasnet_hw_b200(lasnet_hw *hw);
const char *lasnet_kernel_type_name(int32_t kind);  /* "conv1_mask", ... (the event names) */
double lasnet_predict_latency(const lasnet_block_desc *desc, int32_t schedule, double r, const lasnet_hw *hw,
                              int32_t *kinds, double *kernel_us, int32_t max_kernels, int32_t *n_kernels);

/* Benchmark instrumentation.  The next n_pairs kernels this host thread
 * launches through the ABI are bracketed by cudaEventRecord(events[2i]) and
 * cudaEventRecord(events[2i+1]) on their launch stream (i counts launches from
 * this call).  events are cudaEvent_t handles owned by the caller and must stay
 * valid until recorded; n_pairs = 0 disables.  Host-side, launches nothing. */
lasnet_status lasnet_set_kernel_events(void *const *events, int32_t n_pairs);
/* Kernel name of the i-th event pair recorded since the last
 * lasnet_set_kernel_events call on this host thread (e.g. "conv1_mask",
 * "conv23_direct", "decide+ids" for a group of two launches), or NULL when i is
 * out of range.  Static strings; host-side, pure. */
const char *lasnet_kernel_event_name(int32_t i);
/* Number of event pairs recorded since the last lasnet_set_kernel_events call on
 * this host thread (0 when disarmed).  Host-side, pure. */
int32_t lasnet_kernel_event_count(void);

/* Host-side, pure helpers. */
const char *lasnet_status_str(lasnet_status st);
int32_t lasnet_abi_version(void);
/* Number of kernels the last successful call on this host thread enqueued
 * (bench bookkeeping for "gpu_launches"; memsets/copies are not counted). */
int32_t lasnet_last_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LASNET_H */

/*
 * lasnet_oracle.c -- plain, slow, obviously-correct CPU oracle for the LASNet
 * coarse-grained spatially-dynamic residual (bottleneck) block.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or execute this
 * file.  The product path (paper_2210_06223_b200/) never links or calls it,
 * and it shares no code, header, table or helper with the CUDA path.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (LaTeX source of
 * arXiv 2210.06223), "S:n" = SPEC.md line n.  Readings of silent or ambiguous
 * points are numbered R1..R19 as in DESIGN.md section "Readings".
 *
 * Arithmetic: every value is a C double.  Inputs are passed as doubles holding
 * the exact values of the bf16 / fp32 tensors the GPU sees.  Accumulation is
 * fp64 in the natural loop order written below.  The only rounding besides fp64
 * accumulation is the explicit `store_round` at the storage points of h1, h2
 * and y (R13): bf16 round-to-nearest-even or fp32 round-to-nearest.
 *
 * Layouts (R-layout in DESIGN.md): x, y are NHWC [n][h][w][c]; W1 [c_mid][c_in];
 * W2 [c_mid][3][3][c_mid] (OHWI); W3 [c_out][c_mid]; masker weights [c_in].
 * Cells: Gh = ceil(h/s), Gw = ceil(w/s); cell id = n*Gh*Gw + gy*Gw + gx (R15).
 *
 * Every function is a direct transcription; there is no blocking, fusion or
 * reordering beyond what the cited passage states.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_ROUND_NONE 0
#define ORACLE_ROUND_F32 1
#define ORACLE_ROUND_BF16 2

/* ------------------------------------------------------------------------ */
/* Storage rounding (R13).                                                   */
/* ------------------------------------------------------------------------ */

/* bf16 = 1 sign bit, 8 exponent bits (bias 127), 7 stored significand bits.
 * Round-to-nearest, ties-to-even, written from that definition: the quantum
 * (spacing of representable values) around v is 2^(e-8) for normal values
 * with v = m*2^e, 0.5 <= |m| < 1, and 2^-133 in the subnormal range.  rint()
 * in the default rounding mode rounds halfway cases to even. */
double oracle_round_bf16(double v)
{
    if (v == 0.0 || isnan(v) || isinf(v)) return v;
    int e;
    frexp(v, &e);                 /* v = m * 2^e, 0.5 <= |m| < 1 */
    int q = e - 8;                /* 8 significant bits incl. the implicit one */
    if (q < -133) q = -133;       /* bf16 subnormal quantum 2^-133 */
    double r = ldexp(rint(ldexp(v, -q)), q);
    /* largest finite bf16 = (2 - 2^-7) * 2^127; anything rounding above it is inf */
    const double maxbf = ldexp(255.0, 120);
    if (fabs(r) > maxbf) return v > 0 ? INFINITY : -INFINITY;
    return r;
}

double oracle_round_f32(double v) { return (double)(float)v; }

static double store_round(double v, int mode)
{
    if (mode == ORACLE_ROUND_BF16) return oracle_round_bf16(v);
    if (mode == ORACLE_ROUND_F32) return oracle_round_f32(v);
    return v;
}

static double relu(double v) { return v > 0.0 ? v : 0.0; }

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

/* ------------------------------------------------------------------------ */
/* Step 1: masker ("a pooling layer followed by a 1x1 convolution";    */
/* P:100 Fig. 2: M_coarse in {0,1}^{H/S x W/S}; App. B).           */
/* ------------------------------------------------------------------------ */

/* Average pooling over the S x S window of cell (gy,gx), clipped to the image
 * (R7: |Omega| = number of in-image pixels), R1: pooling is average. */
static void pool_cell(const double *x, int h, int w, int c, int s, int n,
                      int gy, int gx, double *pooled)
{
    int y0 = gy * s, x0 = gx * s;
    int y1 = y0 + s < h ? y0 + s : h;
    int x1 = x0 + s < w ? x0 + s : w;
    int omega = (y1 - y0) * (x1 - x0);
    for (int ci = 0; ci < c; ++ci) pooled[ci] = 0.0;
    for (int yy = y0; yy < y1; ++yy)
        for (int xx = x0; xx < x1; ++xx) {
            const double *px = x + (((size_t)n * h + yy) * w + xx) * c;
            for (int ci = 0; ci < c; ++ci) pooled[ci] += px[ci];
        }
    for (int ci = 0; ci < c; ++ci) pooled[ci] /= (double)omega;
}

/* Paper form: M_tilde = conv1x1(avgpool(x)) with 2 output channels
 * (Wm [2][c], bm [2]); decision = argmax, channel 0 = "compute" (P:562:
 * [x*W]_0 > [x*W]_1).  Ties resolve to inactive (R3, strict >). */
void oracle_masker_2ch(const double *x, int n_img, int h, int w, int c, int s,
                       const double *Wm, const double *bm,
                       uint8_t *mask, double *z0, double *z1)
{
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    double *pooled = (double *)malloc(sizeof(double) * (size_t)c);
    for (int n = 0; n < n_img; ++n)
        for (int gy = 0; gy < gh; ++gy)
            for (int gx = 0; gx < gw; ++gx) {
                pool_cell(x, h, w, c, s, n, gy, gx, pooled);
                double a = bm[0], b = bm[1];
                for (int ci = 0; ci < c; ++ci) {
                    a += Wm[ci] * pooled[ci];
                    b += Wm[c + ci] * pooled[ci];
                }
                size_t id = ((size_t)n * gh + gy) * gw + gx;
                mask[id] = (uint8_t)(a > b);
                if (z0) z0[id] = a;
                if (z1) z1[id] = b;
            }
    free(pooled);
}

/* Reduced form (App. B): x*(W_0 - W_1) > 0, here with the scalar bias
 * b = b_0 - b_1 (R2).  logit = sum_c w_c * avgpool_c + b; mask = logit > 0. */
void oracle_masker(const double *x, int n_img, int h, int w, int c, int s,
                   const double *wm, double bm, uint8_t *mask, double *logit)
{
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    double *pooled = (double *)malloc(sizeof(double) * (size_t)c);
    for (int n = 0; n < n_img; ++n)
        for (int gy = 0; gy < gh; ++gy)
            for (int gx = 0; gx < gw; ++gx) {
                pool_cell(x, h, w, c, s, n, gy, gx, pooled);
                double l = bm;
                for (int ci = 0; ci < c; ++ci) l += wm[ci] * pooled[ci];
                size_t id = ((size_t)n * gh + gy) * gw + gx;
                mask[id] = (uint8_t)(l > 0.0);
                if (logit) logit[id] = l;
            }
    free(pooled);
}

/* Nearest upsampling of the coarse mask to the output grid (Fig. 2
 * caption "upsampled to obtain the mask M with the same size as the output
 * feature"; R8 output grid). */
void oracle_upsample(const uint8_t *mc, int n_img, int h, int w, int s, uint8_t *m)
{
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    for (int n = 0; n < n_img; ++n)
        for (int yy = 0; yy < h; ++yy)
            for (int xx = 0; xx < w; ++xx)
                m[((size_t)n * h + yy) * w + xx] =
                    mc[((size_t)n * gh + yy / s) * gw + xx / s];
}

/* ------------------------------------------------------------------------ */
/* Step 2: index list of activated patches (App. B P:568-569 "the masker     */
/* generates the indices of activated patches instead of sparse mask").      */
/* Ascending linear cell id (R15).                                     */
/* ------------------------------------------------------------------------ */
int oracle_compact(const uint8_t *mask, int ncells, int32_t *idx)
{
    int count = 0;
    for (int i = 0; i < ncells; ++i)
        if (mask[i]) idx[count++] = i;
    return count;
}

/* ------------------------------------------------------------------------ */
/* Convolutions of the bottleneck ("the commonly used bottleneck       */
/* structure in [he2016resnet]"), BN folded into (W, b) (R10).         */
/* ------------------------------------------------------------------------ */

/* conv1 (1x1) at one pixel: out[c] = round(ReLU(sum_ci W1[c][ci] x[ci] + b1[c])) */
static void conv1_pixel(const double *xp, int c_in, int c_mid, const double *W1,
                        const double *b1, int rmode, double *out)
{
    for (int c = 0; c < c_mid; ++c) {
        double a = b1[c];
        const double *wr = W1 + (size_t)c * c_in;
        for (int ci = 0; ci < c_in; ++ci) a += wr[ci] * xp[ci];
        out[c] = store_round(relu(a), rmode);
    }
}

/* conv3 (1x1) + residual add + ReLU at one pixel ("scatter ... add";
 * R5: y = ReLU(x + F(x)) on computed pixels). */
static void conv3_residual_pixel(const double *h2p, const double *xp, int c_mid,
                                 int c_out, const double *W3, const double *b3,
                                 int rmode, double *yp)
{
    for (int co = 0; co < c_out; ++co) {
        double a = b3[co];
        const double *wr = W3 + (size_t)co * c_mid;
        for (int c = 0; c < c_mid; ++c) a += wr[c] * h2p[c];
        yp[co] = store_round(relu(xp[co] + a), rmode);
    }
}

/* Static bottleneck everywhere (definition of the result when every pixel
 * is computed; S:534 all-ones mask; P:245 static counterpart).
 * h1 = round(ReLU(conv1x1(x))); h2 = round(ReLU(conv3x3(h1, pad 1 zeros)));
 * y = round(ReLU(x + conv1x1(h2))).  Identity block: c_out == c_in. */
void oracle_static_block(const double *x, int n_img, int h, int w, int c_in,
                         int c_mid, int c_out, const double *W1, const double *b1,
                         const double *W2, const double *b2, const double *W3,
                         const double *b3, int rmode, double *y,
                         double *h1_out, double *h2_out)
{
    size_t npx = (size_t)n_img * h * w;
    double *h1 = h1_out ? h1_out : (double *)malloc(sizeof(double) * npx * c_mid);
    double *h2 = h2_out ? h2_out : (double *)malloc(sizeof(double) * npx * c_mid);
    for (size_t p = 0; p < npx; ++p)
        conv1_pixel(x + p * c_in, c_in, c_mid, W1, b1, rmode, h1 + p * c_mid);
    for (int n = 0; n < n_img; ++n)
        for (int yy = 0; yy < h; ++yy)
            for (int xx = 0; xx < w; ++xx) {
                double *o = h2 + (((size_t)n * h + yy) * w + xx) * c_mid;
                for (int c = 0; c < c_mid; ++c) {
                    double a = b2[c];
                    for (int dy = 0; dy < 3; ++dy)
                        for (int dx = 0; dx < 3; ++dx) {
                            int sy = yy + dy - 1, sx = xx + dx - 1;
                            if (sy < 0 || sy >= h || sx < 0 || sx >= w) continue; /* zero pad */
                            const double *hp = h1 + (((size_t)n * h + sy) * w + sx) * c_mid;
                            const double *wr = W2 + (((size_t)c * 3 + dy) * 3 + dx) * c_mid;
                            for (int ci = 0; ci < c_mid; ++ci) a += wr[ci] * hp[ci];
                        }
                    o[c] = store_round(relu(a), rmode);
                }
            }
    for (size_t p = 0; p < npx; ++p)
        conv3_residual_pixel(h2 + p * c_mid, x + p * c_in, c_mid, c_out, W3, b3,
                             rmode, y + p * c_out);
    if (!h1_out) free(h1);
    if (!h2_out) free(h2);
}

/* Definition mode (each element of M decides whether the output location
 * is computed; unselected regions are filled with the input, R4):
 * y = M ? ystat : x with M the nearest-upsampled coarse mask. */
void oracle_dyn_block_def(const double *x, int n_img, int h, int w, int c_in,
                          int c_mid, int c_out, const double *W1, const double *b1,
                          const double *W2, const double *b2, const double *W3,
                          const double *b3, const uint8_t *mask_cells, int s,
                          int rmode, double *y)
{
    size_t npx = (size_t)n_img * h * w;
    double *ystat = (double *)malloc(sizeof(double) * npx * c_out);
    uint8_t *m = (uint8_t *)malloc(npx);
    oracle_static_block(x, n_img, h, w, c_in, c_mid, c_out, W1, b1, W2, b2, W3, b3,
                        rmode, ystat, NULL, NULL);
    oracle_upsample(mask_cells, n_img, h, w, s, m);
    for (size_t p = 0; p < npx; ++p)
        for (int co = 0; co < c_out; ++co)
            y[p * c_out + co] = m[p] ? ystat[p * c_out + co] : x[p * c_in + co];
    free(ystat);
    free(m);
}

/* Literal mode: the paper's gather -> compute -> scatter procedure
 * (P:89 three steps; P:163-166 gather with the neighbours a 3x3 kernel needs;
 * P:168-170 / P:574-577 scatter fused with the residual add).
 * y := x; for each activated patch index, in list order:
 *   gather the (S+2)x(S+2) halo window of x at origin (gy*S-1, gx*S-1);
 *   conv1 on every window pixel; window pixels outside the image hold 0
 *   (conv2's zero padding applies to h1, R6);
 *   valid 3x3 conv2 on the window -> S x S;
 *   conv3, + residual x, ReLU, scatter to the in-image output pixels (R7).
 * Patches write disjoint output pixels, so the loop over patches may run in
 * parallel (used only to time the oracle on the host cores). */
void oracle_dyn_block_literal(const double *x, int n_img, int h, int w, int c_in,
                              int c_mid, int c_out, const double *W1, const double *b1,
                              const double *W2, const double *b2, const double *W3,
                              const double *b3, const int32_t *idx, int count, int s,
                              int rmode, double *y)
{
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    int hs = s + 2;
    size_t npx = (size_t)n_img * h * w;
    memcpy(y, x, sizeof(double) * npx * c_in); /* c_out == c_in: identity block */

#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int t = 0; t < count; ++t) {
        double *win = (double *)malloc(sizeof(double) * (size_t)hs * hs * c_mid);
        double *h2 = (double *)malloc(sizeof(double) * (size_t)s * s * c_mid);
        int id = idx[t];
        int n = id / (gh * gw), g = id % (gh * gw);
        int gy = g / gw, gx = g % gw;
        int oy = gy * s - 1, ox = gx * s - 1;
        /* gather + conv1 over the halo window */
        for (int wy = 0; wy < hs; ++wy)
            for (int wx = 0; wx < hs; ++wx) {
                int sy = oy + wy, sx = ox + wx;
                double *o = win + ((size_t)wy * hs + wx) * c_mid;
                if (sy < 0 || sy >= h || sx < 0 || sx >= w) {
                    for (int c = 0; c < c_mid; ++c) o[c] = 0.0;
                } else {
                    conv1_pixel(x + (((size_t)n * h + sy) * w + sx) * c_in, c_in,
                                c_mid, W1, b1, rmode, o);
                }
            }
        /* valid 3x3 conv2 over the window */
        for (int py = 0; py < s; ++py)
            for (int px = 0; px < s; ++px)
                for (int c = 0; c < c_mid; ++c) {
                    double a = b2[c];
                    for (int dy = 0; dy < 3; ++dy)
                        for (int dx = 0; dx < 3; ++dx) {
                            const double *hp = win + ((size_t)(py + dy) * hs + (px + dx)) * c_mid;
                            const double *wr = W2 + (((size_t)c * 3 + dy) * 3 + dx) * c_mid;
                            for (int ci = 0; ci < c_mid; ++ci) a += wr[ci] * hp[ci];
                        }
                    h2[((size_t)py * s + px) * c_mid + c] = store_round(relu(a), rmode);
                }
        /* conv3 + residual add, scatter (edge patches clipped, R7) */
        for (int py = 0; py < s; ++py)
            for (int px = 0; px < s; ++px) {
                int yy = gy * s + py, xx = gx * s + px;
                if (yy >= h || xx >= w) continue;
                size_t p = ((size_t)n * h + yy) * w + xx;
                conv3_residual_pixel(h2 + ((size_t)py * s + px) * c_mid, x + p * c_in,
                                     c_mid, c_out, W3, b3, rmode, y + p * c_out);
            }
        free(win);
        free(h2);
    }
}

/* One output pixel of the block, computed on its own (used to check sampled
 * outputs at full size, where running the whole oracle would take too long).
 * Returns 1 if the pixel is computed (active), 0 if it is passed through. */
int oracle_block_pixel(const double *x, int h, int w, int c_in, int c_mid, int c_out,
                       const double *W1, const double *b1, const double *W2,
                       const double *b2, const double *W3, const double *b3,
                       const uint8_t *mask_cells, int s, int rmode,
                       int n, int yy, int xx, double *yout)
{
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    const double *xp = x + (((size_t)n * h + yy) * w + xx) * c_in;
    if (!mask_cells[((size_t)n * gh + yy / s) * gw + xx / s]) {
        for (int co = 0; co < c_out; ++co) yout[co] = xp[co];
        return 0;
    }
    double *win = (double *)malloc(sizeof(double) * 9 * (size_t)c_mid);
    double *h2 = (double *)malloc(sizeof(double) * (size_t)c_mid);
    for (int dy = 0; dy < 3; ++dy)
        for (int dx = 0; dx < 3; ++dx) {
            int sy = yy + dy - 1, sx = xx + dx - 1;
            double *o = win + ((size_t)dy * 3 + dx) * c_mid;
            if (sy < 0 || sy >= h || sx < 0 || sx >= w) {
                for (int c = 0; c < c_mid; ++c) o[c] = 0.0;
            } else {
                conv1_pixel(x + (((size_t)n * h + sy) * w + sx) * c_in, c_in, c_mid,
                            W1, b1, rmode, o);
            }
        }
    for (int c = 0; c < c_mid; ++c) {
        double a = b2[c];
        for (int dy = 0; dy < 3; ++dy)
            for (int dx = 0; dx < 3; ++dx) {
                const double *hp = win + ((size_t)dy * 3 + dx) * c_mid;
                const double *wr = W2 + (((size_t)c * 3 + dy) * 3 + dx) * c_mid;
                for (int ci = 0; ci < c_mid; ++ci) a += wr[ci] * hp[ci];
            }
        h2[c] = store_round(relu(a), rmode);
    }
    conv3_residual_pixel(h2, xp, c_mid, c_out, W3, b3, rmode, yout);
    free(win);
    free(h2);
    return 1;
}

/* ------------------------------------------------------------------------ */
/* Dynamic projection (first) block of a stage, literal mode (SURVEY 8(f)    */
/* NEXT-f1; 8(c) reading 9; reading R22).  The stage's first block  */
/* changes resolution (stride 1 or 2) and channels (c_in -> c_out), so its    */
/* residual is the 1x1 stride-s projection R = Wd x_s + bd, computed densely  */
/* (the paper keeps the downsampling shortcut dense) and stored like   */
/* any feature map (rounded).  The block output is y = ReLU(R + M F(x)) with   */
/* the mask M on the OUTPUT grid ("the corresponding location of the     */
/* output feature"): y = rnd(ReLU(R + conv3(h2) + b3)) on active pixels and   */
/* ReLU(R) on the others -- for an identity block (R = x >= 0) this is the    */
/* input fill of P:86.                                                         */
/* The residual function F follows the gather -> compute -> scatter steps     */
/* (P:89): an output patch of S x S pixels at stride s reads the   */
/* input window of side s(S-1)+3 at origin (s S gy - 1, s S gx - 1); conv1 runs */
/* on every in-image window pixel (0 outside the image, R6), conv2 is the     */
/* valid 3x3 conv at stride s over the window, conv3 + R, ReLU, scatter.      */
/*   x [n][hi][wi][c_in] (hi, wi multiples of s); y [n][hi/s][wi/s][c_out]     */
/*   Wd [c_out][c_in], bd [c_out]; idx/count: active cells of the output grid   */
/* ------------------------------------------------------------------------ */
void oracle_proj_dyn_literal(const double *x, int n_img, int hi, int wi, int c_in,
                             int c_mid, int c_out, const double *W1, const double *b1,
                             const double *W2, const double *b2, const double *W3,
                             const double *b3, const double *Wd, const double *bd,
                             const int32_t *idx, int count, int s, int stride,
                             int rmode, double *y)
{
    int h = hi / stride, w = wi / stride;
    int gh = ceil_div(h, s), gw = ceil_div(w, s);
    int side = stride * (s - 1) + 3;
    size_t npx = (size_t)n_img * h * w;
    double *R = (double *)malloc(sizeof(double) * npx * c_out);
    /* the dense projection shortcut, stored rounded; y := ReLU(R) everywhere */
    for (int n = 0; n < n_img; ++n)
        for (int oy = 0; oy < h; ++oy)
            for (int ox = 0; ox < w; ++ox) {
                size_t p = ((size_t)n * h + oy) * w + ox;
                const double *xs = x + (((size_t)n * hi + (size_t)oy * stride) * wi + (size_t)ox * stride) * c_in;
                for (int co = 0; co < c_out; ++co) {
                    double a = bd[co];
                    const double *wr = Wd + (size_t)co * c_in;
                    for (int ci = 0; ci < c_in; ++ci) a += wr[ci] * xs[ci];
                    R[p * c_out + co] = store_round(a, rmode);
                    y[p * c_out + co] = relu(R[p * c_out + co]);
                }
            }
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int t = 0; t < count; ++t) {
        double *win = (double *)malloc(sizeof(double) * (size_t)side * side * c_mid);
        double *h2 = (double *)malloc(sizeof(double) * (size_t)s * s * c_mid);
        int id = idx[t];
        int n = id / (gh * gw), g = id % (gh * gw);
        int gy = g / gw, gx = g % gw;
        int oy0 = gy * s * stride - 1, ox0 = gx * s * stride - 1;
        /* gather + conv1 over the input window */
        for (int wy = 0; wy < side; ++wy)
            for (int wx = 0; wx < side; ++wx) {
                int sy = oy0 + wy, sx = ox0 + wx;
                double *o = win + ((size_t)wy * side + wx) * c_mid;
                if (sy < 0 || sy >= hi || sx < 0 || sx >= wi) {
                    for (int c = 0; c < c_mid; ++c) o[c] = 0.0;
                } else {
                    conv1_pixel(x + (((size_t)n * hi + sy) * wi + sx) * c_in, c_in, c_mid, W1, b1, rmode, o);
                }
            }
        /* valid 3x3 conv2 at stride s over the window -> S x S */
        for (int py = 0; py < s; ++py)
            for (int px = 0; px < s; ++px)
                for (int c = 0; c < c_mid; ++c) {
                    double a = b2[c];
                    for (int dy = 0; dy < 3; ++dy)
                        for (int dx = 0; dx < 3; ++dx) {
                            const double *hp = win + ((size_t)(stride * py + dy) * side + (stride * px + dx)) * c_mid;
                            const double *wr = W2 + (((size_t)c * 3 + dy) * 3 + dx) * c_mid;
                            for (int ci = 0; ci < c_mid; ++ci) a += wr[ci] * hp[ci];
                        }
                    h2[((size_t)py * s + px) * c_mid + c] = store_round(relu(a), rmode);
                }
        /* conv3 + the stored shortcut R, ReLU, scatter (edge patches clipped, R7) */
        for (int py = 0; py < s; ++py)
            for (int px = 0; px < s; ++px) {
                int yy = gy * s + py, xx = gx * s + px;
                if (yy >= h || xx >= w) continue;
                size_t p = ((size_t)n * h + yy) * w + xx;
                conv3_residual_pixel(h2 + ((size_t)py * s + px) * c_mid, R + p * c_out, c_mid, c_out, W3, b3,
                                     rmode, y + p * c_out);
            }
        free(win);
        free(h2);
    }
    free(R);
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

// rowmap.cuh -- how GEMM rows of the three convolutions map onto pixels.
//
// The dynamic block is run as three implicit GEMMs:
//   conv1  rows = (active patch t, halo pixel j), j < (S+2)^2   K = c_in
//   conv2  rows = (active patch t, output pixel j), j < S^2     K = 9*c_mid (3x3 taps on h1)
//   conv3  rows = (active patch t, output pixel j)              K = c_mid, scatter-add epilogue
// and the dense comparator uses rows = pixels for all three.
#pragma once
#include <cstdint>
#include <cuda.h>

namespace lasnet {

// Division by a runtime constant via multiply-high (valid for 0 <= n < 2^31):
// p = 31 + ceil(log2 d), mul = ceil(2^p / d), q = umulhi(n, mul) >> (p - 32).
struct FastDiv {
    uint32_t d, mul, shr;
    __host__ __device__ FastDiv() : d(1), mul(0), shr(0) {}
    __host__ FastDiv(uint32_t div) : d(div), mul(0), shr(0) {
        if (d > 1) {
            int l = 0;
            while ((1u << l) < d) ++l;  // ceil(log2 d)
            const int p = 31 + l;
            mul = (uint32_t)(((1ull << p) + d - 1) / d);
            shr = (uint32_t)(p - 32);
        }
    }
    __device__ __forceinline__ int div(int n) const {
        return d == 1 ? n : (int)(__umulhi((uint32_t)n, mul) >> shr);
    }
};

enum ConvMode : int {
    CONV1_DYN = 0,    // A = gathered halo rows of x, out = h1 [P][(S+2)^2][c_mid]
    CONV2_DYN = 1,    // A = im2col of h1 patch windows, out = h2 [P][S^2][c_mid]
    CONV3_DYN = 2,    // A = h2 rows, out = y pixels (residual add, ReLU, scatter)
    CONV1_DENSE = 3,  // A = x pixel rows, out = h1 [n*h*w][c_mid]
    CONV2_DENSE = 4,  // A = im2col of h1 with zero padding, out = h2 [n*h*w][c_mid]
    CONV3_DENSE = 5,  // A = h2 rows, out = y (residual add, ReLU)
    CONV1_DENSE_MASK = 6,  // CONV1_DENSE + per-pixel masker partials (the paper's masker-conv1 fusion)
    STEM = 7,              // ResNet stem 7x7 stride 2 on 8-channel (3 + zero) input: tile = one output row
    CONV2_GATHER = 8,      // CONV2_DYN whose A rows are gathered by cp.async straight from the DENSE h1
                           // [c_mid/64][m_dense][64] (masker-fused schedule: no gathered window copy)
    PROJ_SC = 9,           // CONV3_DENSE without a residual (the projection blocks' dense 1x1 shortcut / the
                           // static block's [W3 | Wd] conv): 256-column tiles, whole tiles stored by TMA
};

struct ConvArgs {
    // TMA descriptors (tcgen05 path only; see conv_tc.cu for the box shapes)
    CUtensorMap tmap_a;     // activation operand A (x, h1 or h2)
    CUtensorMap tmap_b;     // weight matrix [N][K]
    CUtensorMap tmap_out;   // output (h1, h2 or y)
    CUtensorMap tmap_res;   // residual x (conv3)
    CUtensorMap tmap_b3;    // conv3 weights [c_out][c_mid] (fused conv2+conv3 kernel)
    CUtensorMap tmap_s[8];  // stem: A window views (residue k of the output column mod 4) [0..3], output views [4..7]
    const void *w3;         // fused kernel: conv3 weights
    const float *bias3;     // fused kernel: conv3 bias [c_out]
    int32_t n3;             // fused kernel: c_out
    const void *a_src;      // x (conv1), h1 (conv2), h2 (conv3)
    const void *w;          // [N][K] row-major (K-major)
    const float *bias;      // [N]
    void *out;              // h1, h2 or y
    const void *resid;      // x (conv3 epilogue)
    const int32_t *idx;     // active cell ids (dynamic modes)
    const int32_t *count;   // device count (dynamic modes)
    int32_t m_dense;        // rows for dense modes
    int32_t K, N;           // GEMM sizes
    int32_t a_ld;           // elements per A source row (c_in for conv1, c_mid otherwise)
    int32_t out_ld;         // elements per output row
    int32_t n_img, H, W, S, Gh, Gw;
    // conv1 windows (gather modes): cell pitch at the block INPUT resolution (S_in = stride * S)
    // and window side (hs = stride * (S - 1) + 3: S + 2 for stride 1, 2S + 1 for stride 2);
    // H, W are the input dims for conv1 and the output dims for conv2 / conv3
    int32_t S_in, hs;
    FastDiv fd_G, fd_Gw, fd_hs, fd_hs2, fd_S, fd_SS;  // G = Gh*Gw, hs (window side), SS = S*S
    FastDiv fd_HW, fd_W;                             // dense rows -> (image, y, x) (relu_mask)
    // dense epilogue: ReLU only on pixels of INACTIVE cells of this mask [n][Gh][Gw] (the dynamic
    // projection block's shortcut R: inactive pixels store ReLU(R), active ones R for the scatter-add)
    const uint8_t *relu_mask;
    int32_t tma_y;            // dense conv3: the epilogue TMA-stores whole 128-row tiles of y (tmap_out = y [px][c_out])
    int32_t view4;            // dense conv3 (strided projection shortcut): A = a 4-D strided view of x, dense tiles
                              // (dense_tiling), y stored through a 4-D view (tmap_out)
    // tcgen05 tile geometry (host-computed)
    int32_t units_per_tile;   // dynamic: TMA boxes (conv1) / patches (conv2, conv3) per 128-row tile
    int32_t units_per_patch;  // conv1: 1 (whole halo box) or S+2 (one box per halo row)
    int32_t unit_rows;        // conv1: GEMM rows per box
    int32_t unit_halo_rows;   // conv1: halo rows per box
    int32_t box_rows;         // rows one A box delivers (conv2 dyn/dense, conv3 dyn)
    int32_t rows_h, imgs_box; // conv2 dense: image rows / images per box
    int32_t cols_w, tiles_x;  // conv2 dense: image columns per box, column blocks per row band (W > 128)
    int32_t dense_tiles;      // conv2 dense: M tiles
    int32_t conv_stride;      // dense 3x3: 2 = stride 2 through the four parity views tmap_s[(row odd) * 2 + (col odd)]
    int32_t a2_kb;            // dense conv3: K-blocks >= a2_kb of A come from tmap_s[0] (K-concatenated sources)
    int32_t no_relu;          // 1: the epilogue stores acc + bias (+ residual) without ReLU (projection shortcut)
    int32_t pair_tc;          // conv_tc: 2-SM UMMAs over CTA pairs (conv_tc_plan; weight box of bn / 2 rows)
    int32_t balance;          // dynamic fused conv23: spread the active cells evenly over whole rounds of tiles
    int32_t direct;           // dynamic conv2 (fused conv23): A patches read straight from the dense h1
                              // [c_mid/64][N][H][W][64] by one {64, S, S} TMA box per active cell (no gather)
    // masker fused into the dense conv1 (CONV1_DENSE_MASK): per pixel p the fp32
    // partial logits sum_c wm_c x[p,c] and magnitudes sum_c |wm_c x[p,c]| over the
    // lower and the upper 32 channels of every 64-channel K-block
    const float *wm;          // [c_in] reduced masker weight W_0 - W_1
    float4 *mpart;            // [n*h*w] (partial, magnitude) of the lower and of the upper channel halves
};

// Total GEMM rows; dynamic modes read the device-resident active count.
__device__ __forceinline__ int gemm_rows(int mode, const ConvArgs &a) {
    if (mode <= CONV3_DYN || mode == CONV2_GATHER) return (*a.count) * (mode == CONV1_DYN ? a.hs * a.hs : a.S * a.S);
    return a.m_dense;
}

// Dense 3x3 tile mt -> (first image, first row, first column) of its box: a box
// covers imgs_box whole images (h*w <= 128), or rows_h rows x cols_w columns of one
// image (tiles_x column blocks per row band when w > 128).
__device__ __forceinline__ void dense_tile_origin(const ConvArgs &a, int mt, int &n0, int &y0, int &x0) {
    if (a.rows_h < a.H || a.tiles_x > 1) {
        const int bands = (a.H + a.rows_h - 1) / a.rows_h;
        const int tpi = bands * a.tiles_x;
        n0 = mt / tpi;
        const int rem = mt - n0 * tpi;
        const int band = rem / a.tiles_x;
        y0 = band * a.rows_h;
        x0 = (rem - band * a.tiles_x) * a.cols_w;
    } else {
        n0 = mt * a.imgs_box;
        y0 = 0;
        x0 = 0;
    }
}

// Active cell t -> (image n, cell row gy, cell col gx).
__device__ __forceinline__ void cell_decode(const ConvArgs &a, int cell, int &n, int &gy, int &gx) {
    n = a.fd_G.div(cell);
    const int g = cell - n * (int)a.fd_G.d;
    gy = a.fd_Gw.div(g);
    gx = g - gy * a.Gw;
}
__device__ __forceinline__ void cell_coords(const ConvArgs &a, int t, int &n, int &gy, int &gx) {
    cell_decode(a, a.idx[t], n, gy, gx);
}

// conv1 (dynamic): GEMM row -> source pixel of x, or -1 for a halo pixel outside
// the image / a row past the end (zero row; the epilogue also writes 0, R6).
__device__ __forceinline__ int halo_pixel(const ConvArgs &a, int r, int M) {
    if (r >= M) return -1;
    const int hs = a.hs, hs2 = hs * hs;
    const int t = a.fd_hs2.div(r), j = r - t * hs2;
    int n, gy, gx;
    cell_coords(a, t, n, gy, gx);
    const int jy = a.fd_hs.div(j);
    const int hy = gy * a.S_in - 1 + jy, hx = gx * a.S_in - 1 + (j - jy * hs);
    if (hy < 0 || hy >= a.H || hx < 0 || hx >= a.W) return -1;
    return (n * a.H + hy) * a.W + hx;
}

// conv2 (dynamic): GEMM row -> h1 row of the window centre of output pixel j of patch t.
__device__ __forceinline__ int conv2_center_row(const ConvArgs &a, int r, int M) {
    if (r >= M) return -1;
    const int ss = a.S * a.S, hs = a.hs;
    const int t = a.fd_SS.div(r), j = r - t * ss;
    const int py = a.fd_S.div(j), px = j - py * a.S;
    return t * hs * hs + (py + 1) * hs + (px + 1);
}

// conv3 (dynamic): GEMM row -> output pixel, or -1 when the patch is clipped at
// the image border (R7) or the row is past the end.
__device__ __forceinline__ int out_pixel(const ConvArgs &a, int r, int M) {
    if (r >= M) return -1;
    const int ss = a.S * a.S;
    const int t = a.fd_SS.div(r), j = r - t * ss;
    int n, gy, gx;
    cell_coords(a, t, n, gy, gx);
    const int py = a.fd_S.div(j);
    const int yy = gy * a.S + py, xx = gx * a.S + (j - py * a.S);
    if (yy >= a.H || xx >= a.W) return -1;
    return (n * a.H + yy) * a.W + xx;
}

}  // namespace lasnet

// regnet.cuh -- launch arguments of the LAS-RegNetY kernels (regnet.cu), shared
// with the C ABI (lasnet_capi.cu).
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace lasnet {

struct GconvArgs {
    const __nv_bfloat16 *h1;  // chunk-major [C/64][h1_rows][64]
    const __nv_bfloat16 *wb;  // [C][3][3][16]
    const float *bias;        // [C]
    __nv_bfloat16 *h2;        // [rows][C]
    const int32_t *count;     // dynamic: active patches (device); dense: nullptr
    int64_t h1_rows;          // rows of one h1 chunk (cap * hs^2, or n * H * W)
    int C;                    // channels (multiple of 64)
    int rows;                 // dense: output rows (n * Ho * Wo)
    int S, hs;                // dynamic: patch side, window side (S + 2)
    int H, W, Ho, Wo, stride; // dense: input / output dims
    int n_img;                // dense: images
    int upt, trows;           // tile geometry (host-computed): patches / output rows per tile
    // dynamic, direct: the windows are read straight from the DENSE h1 [C/64][h1_rows = n H W][64] at the
    // active cells' positions (ids in idx; G cells per image, Gw per grid row; H, W the map), 0 outside
    int direct;
    const int32_t *idx;
    int G, Gw;
};

struct SeArgs {
    const __nv_bfloat16 *h2;  // [rows][C]
    const float *w1, *b1;     // [w_se][C], [w_se]
    const float *w2, *b2;     // [C][w_se], [C]
    float *scale;             // [n][C] out
    float *pooled;            // [n][C] scratch: mean of h2 over the image's computed pixels
    float *z;                 // [n][w_se] scratch: the squeeze
    const int32_t *idx;       // dynamic: ascending active cell ids
    const int32_t *count;     // dynamic: device count; dense: nullptr
    int C, w_se, n_img;
    int S, H, W, G, Gw;       // dynamic: patch side, output dims, cells per image, grid width
    int HW;                   // dense: output pixels per image
};

cudaError_t launch_gconv(bool dyn, const GconvArgs &a, int max_rows, int num_sms, cudaStream_t st);
cudaError_t launch_se(const SeArgs &a, cudaStream_t st);
cudaError_t launch_se_apply(__nv_bfloat16 *h2, const float *scale, const int32_t *idx, const int32_t *count,
                            int max_rows, int C, int S, int G, int HW, int num_sms, cudaStream_t st);
cudaError_t launch_regnet_stem(const void *x, const void *w, const float *b, void *y, int n_img, int h, int wo,
                               int co_real, int num_sms, cudaStream_t st);

}  // namespace lasnet

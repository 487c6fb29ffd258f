// small_block.cuh -- arguments of the single-launch fp32 small-batch block (small_block.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lasnet {

struct SmallArgs {
    const float *x;
    float *y;
    const float *w1, *b1, *w2, *b2, *w3, *b3;
    const float *wm;  // nullptr: dense comparator
    float bm;
    int n, H, W, ci, cm, co, S, Gh, Gw, ncells, px;
    uint8_t *mask;    // [ncells] (dynamic)
    int32_t *idx, *count;
    float *h1;        // [px][cm]
    float *h2;        // [rows][cm]: rows = active cells x S^2 (dense: px)
    unsigned *bar;    // [0] arrivals (zero on entry, left zero), [1] generation (any value)
};

cudaError_t launch_small_block(const SmallArgs &a, int num_sms, cudaStream_t st);

}  // namespace lasnet

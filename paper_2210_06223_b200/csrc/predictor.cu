// predictor.cu -- the latency predictor G(H, P, S, r) of LASNet (P:113-121
// sec. 3.3, App. A) re-targeted to B200.
// Host-only code: no kernels.
//
// The paper models a device as processing engines (PEs) behind a three-level
// memory system (off-chip memory, on-chip global memory, memory in the PE,
// P:117-118) and predicts a dynamic block's latency from the data movement and
// the computation of its operators under their tiling.
// Here:
//   PEs          the SMs (148), one persistent CTA each
//   off-chip     HBM3e: the compulsory bytes of every kernel
//   on-chip      L2: every operand tile staged into shared memory (the A tile
//                and the weight tile of each 128-row GEMM tile -- weights are
//                re-streamed per tile, the im2col taps re-read per tile)
//   in-PE        tcgen05 tensor throughput per SM
// and the operators are the library's actual launches for the block's schedule
// (the same plan lasnet_block_forward / lasnet_dense_block execute: fused or
// unfused steps 4-5, direct or gathered conv2 operands, projection blocks).
// Each kernel's work is split into its 128-row tiles; a persistent grid of one
// CTA per SM runs ceil(tiles / SMs) rounds of the slowest per-tile resource:
//   t_k = launch + t0_k + rounds_k * max(hbm_k, l2_k, tc_k per tile) / eff_k
// with eff_k the achieved fraction of the bound and t0_k a fixed cost (pipeline
// fill and drain, dependent latency chains) per kernel type, both calibrated on
// B200 measurements (tools/calibrate_predictor.py -> profiles/predictor_r2.json).
// The expected geometry at activation rate r assumes r of the cells active,
// uniformly (P, halo pixels and output pixels are r times their all-cells sums,
// border clipping included).
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/lasnet.h"

namespace lasnet {
bool plan_fused23(const lasnet_block_desc *d);
bool plan_direct(const lasnet_block_desc *d);
bool plan_gather2(const lasnet_block_desc *d);
bool plan_proj_mask_fused();
}  // namespace lasnet

namespace {

const char *const kNames[LASNET_K_COUNT] = {
    "mask_compact", "conv1_dyn", "conv1_mask", "decide", "decide+gather", "conv23", "conv23_direct", "conv2_dyn",
    "conv3_dyn", "conv1_dense", "conv2_dense", "conv3_dense", "conv23_dense", "subsample", "shortcut", "mask",
    "compact", "conv2_gather"};

struct Work {
    int type;
    double hbm;    // compulsory HBM bytes
    double l2;     // bytes staged from L2 into shared memory
    double flops;  // 2 * MAC
    double tiles;  // persistent work units (0: a streaming kernel spread over every SM)
};

struct Plan {
    Work k[8];
    int n = 0;
    void add(int type, double hbm, double l2, double flops, double tiles) { k[n++] = {type, hbm, l2, flops, tiles}; }
};

double ceil_div(double a, double b) { return std::ceil(a / b); }

// sum over all cells of the in-image pixels of a window of side `side` at origin
// pitch*g - 1 (1-D; the 2-D sum is the product of the row and column sums)
double window_sum_1d(int n_out_cells, int pitch, int side, int extent) {
    double s = 0;
    for (int g = 0; g < n_out_cells; ++g) {
        const int a = g * pitch - 1, b = a + side;
        s += (b < extent ? b : extent) - (a > 0 ? a : 0);
    }
    return s;
}

// steps 4-5 on gathered / direct h1 (fused conv23 or conv2 + conv3)
void plan_steps45(Plan &p, const lasnet_block_desc *d, double P, double out_px, double halo_h1, bool direct) {
    const double e = 2, S = d->s, ss = S * S, C = d->c_mid, CO = d->c_out;
    const double W2 = 9 * C * C * e, W3 = CO * C * e;
    const int hs = d->stride * (d->s - 1) + 3;
    const double win = P * hs * hs * C * e;  // gathered windows
    if (lasnet::plan_fused23(d)) {
        const double upt = std::floor(128.0 / ss);
        const double tiles = ceil_div(P, upt);
        const double hbm = (direct ? halo_h1 : win) + 2 * out_px * CO * e + W2 + W3;
        const double l2 = tiles * (128 * 9 * C * e + W2 + W3);
        p.add(direct ? LASNET_K_CONV23_DIRECT : LASNET_K_CONV23, hbm, l2,
              2 * out_px * (9 * C * C + C * CO), tiles);
        return;
    }
    const double rows = P * ss;
    const double t2 = ceil_div(P, std::floor(128.0 / ss)) * (C / 128 > 1 ? C / 128 : 1);
    p.add(LASNET_K_CONV2_DYN, win + rows * C * e + W2, t2 * (128 * 9 * C * e + 9 * C * (C < 128 ? C : 128) * e),
          2 * out_px * 9 * C * C, t2);
    const double t3 = ceil_div(rows, 128) * (CO / 128);
    p.add(LASNET_K_CONV3_DYN, rows * C * e + 2 * out_px * CO * e + W3, t3 * (128 * C * e + 128 * C * e),
          2 * out_px * C * CO, t3);
}

bool build_plan(Plan &p, const lasnet_block_desc *d, int schedule, double r) {
    const double e = 2;
    const int st = d->stride, S = d->s;
    const int Hi = d->h * st, Wi = d->w * st;
    const int gh = (d->h + S - 1) / S, gw = (d->w + S - 1) / S;
    const double n = d->n, px = n * d->h * d->w, pxi = n * Hi * Wi;
    const double G = n * gh * gw, P = r * G;
    const double C = d->c_mid, CI = d->c_in, CO = d->c_out;
    const double W1 = C * CI * e;
    const bool proj = st != 1 || d->c_in != d->c_out;
    const int hs = st * (S - 1) + 3;
    // expected in-image window pixels (input resolution) and output pixels of the active cells
    const double halo = r * n * window_sum_1d(gh, S * st, hs, Hi) * window_sum_1d(gw, S * st, hs, Wi);
    const double out_px = r * px;
    const double bn1 = (int)C % 256 == 0 ? 256 : (C == 64 ? 64 : 128);
    if (schedule == LASNET_SCHED_DENSE) {
        const double t1 = ceil_div(pxi, 128) * (C / bn1);
        p.add(LASNET_K_CONV1_DENSE, pxi * (CI + C) * e + W1, t1 * (128 + bn1) * CI * e, 2 * pxi * CI * C, t1);
        if (!proj && lasnet::plan_fused23(d)) {
            const double tiles = ceil_div(px, 128);
            p.add(LASNET_K_CONV23_DENSE, px * C * e + 2 * px * CO * e + 9 * C * C * e + CO * C * e,
                  tiles * (128 * 9 * C * e + 9 * C * C * e + CO * C * e), 2 * px * (9 * C * C + C * CO), tiles);
            return true;
        }
        const double t2 = ceil_div(px, 128) * (C / 128 > 1 ? C / 128 : 1);
        p.add(LASNET_K_CONV2_DENSE, pxi * C * e + px * C * e + 9 * C * C * e, t2 * (128 + (C < 128 ? C : 128)) * 9 * C * e,
              2 * px * 9 * C * C, t2);
        if (proj && st > 1) p.add(LASNET_K_SUBSAMPLE, 2 * px * CI * e, 0, 0, 0);
        const double K3 = proj ? C + CI : C;
        const double t3 = ceil_div(px, 128) * (CO / 128);
        p.add(LASNET_K_CONV3_DENSE, px * K3 * e + (proj ? 1 : 2) * px * CO * e + CO * K3 * e, t3 * 256 * K3 * e,
              2 * px * K3 * CO, t3);
        return true;
    }
    if (proj) {  // the dynamic first block (reading R22): separate schedule only
        if (schedule != LASNET_SCHED_MASKER_SEPARATE) return false;
        if (lasnet::plan_proj_mask_fused()) {
            p.add(LASNET_K_MASK_COMPACT, pxi * CI * e + G + 4 * P, 0, 2 * pxi * CI, 0);
        } else {
            p.add(LASNET_K_MASK, pxi * CI * e + G, 0, 2 * pxi * CI, 0);
            p.add(LASNET_K_COMPACT, G + 4 * P, 0, 0, 0);
        }
        // the shortcut reads x_s through a strided view of x (no subsample launch)
        const double ts = ceil_div(px, 128) * (CO / 128);
        p.add(LASNET_K_SHORTCUT, px * CI * e + px * CO * e + CO * CI * e + G, ts * 256 * CI * e, 2 * px * CI * CO, ts);
        const double rows = P * hs * hs;
        const double t1 = ceil_div(rows, 128) * (C / bn1);
        p.add(LASNET_K_CONV1_DYN, halo * CI * e + rows * C * e + W1, t1 * (128 + bn1) * CI * e, 2 * halo * CI * C, t1);
        plan_steps45(p, d, P, out_px, 0, false);
        return true;
    }
    if (schedule == LASNET_SCHED_MASKER_SEPARATE) {
        p.add(LASNET_K_MASK_COMPACT, px * CI * e + G + 4 * P, 0, 2 * px * CI, 0);
        const double rows = P * hs * hs;
        const double t1 = ceil_div(rows, 128) * (C / bn1);
        p.add(LASNET_K_CONV1_DYN, halo * CI * e + rows * C * e + W1, t1 * (128 + bn1) * CI * e, 2 * halo * CI * C, t1);
        plan_steps45(p, d, P, out_px, 0, false);
        return true;
    }
    if (schedule == LASNET_SCHED_MASKER_FUSED) {
        const double t1 = ceil_div(px, 128) * (C / bn1);
        p.add(LASNET_K_CONV1_MASK, px * (CI + C) * e + 16 * px + W1, t1 * (128 + bn1) * CI * e, 2 * px * CI * (C + 1),
              t1);
        const bool direct = lasnet::plan_direct(d);
        const double h1_halo = halo * C * e;
        if (lasnet::plan_gather2(d)) {
            // conv2 gathers the im2col rows from the dense h1 (L2): the windows' bytes once from
            // HBM, 9 taps re-read per tile from L2; then conv3 + scatter-add
            p.add(LASNET_K_DECIDE, 16 * px + G + 4 * P, 0, 0, 0);
            const double S2 = (double)d->s * d->s, rows = P * S2;
            const double t2 = ceil_div(P, std::floor(128.0 / S2)) * (C / 256 >= 1 ? C / 256 : 1);
            const double bn2 = (int)C % 256 == 0 ? 256 : 128;
            p.add(LASNET_K_CONV2_GATHER, h1_halo + rows * C * e + 9 * C * C * e,
                  t2 * (128 * 9 * C * e + 9 * C * bn2 * e), 2 * out_px * 9 * C * C, t2);
            const double t3 = ceil_div(rows, 128) * (CO / 128);
            p.add(LASNET_K_CONV3_DYN, rows * C * e + 2 * out_px * CO * e + CO * C * e, t3 * (128 * C * e + 128 * C * e),
                  2 * out_px * C * CO, t3);
            return true;
        }
        if (direct) {
            p.add(LASNET_K_DECIDE, 16 * px + G + 4 * P, 0, 0, 0);
        } else {
            p.add(LASNET_K_DECIDE_GATHER, 16 * px + G + 4 * P + h1_halo + P * hs * hs * C * e, 0, 0, 0);
        }
        plan_steps45(p, d, P, out_px, h1_halo, direct);
        return true;
    }
    return false;
}

}  // namespace

extern "C" {

const char *lasnet_kernel_type_name(int32_t k) { return k >= 0 && k < LASNET_K_COUNT ? kNames[k] : nullptr; }

void lasnet_hw_b200(lasnet_hw *hw) {
    if (!hw) return;
    std::memset(hw, 0, sizeof(*hw));
    // B200: 148 SMs; HBM copy bandwidth and dense bf16 tensor throughput as measured on
    // this pool (MEASURED_PEAKS.json); L2 -> SM staging bandwidth from the round-1 probes
    // (tools/bw_probe.cu, profiles/microbench_r1.md: ~75 GB/s per SM for TMA streams);
    // a graph-replayed launch costs ~2 us of fill/drain.
    hw->sms = 148;
    hw->hbm_gbs = 6553.6;
    hw->tc_tflops = 1652.2;
    hw->l2_gbs = 11100.0;
    hw->launch_us = 2.0;
    // achieved fraction of the bound per kernel type, calibrated on B200 launches
    // (tools/calibrate_predictor.py; profiles/predictor_r2.json)
#include "predictor_b200.inc"
}

double lasnet_predict_latency(const lasnet_block_desc *d, int32_t schedule, double r, const lasnet_hw *hw,
                              int32_t *kinds, double *kernel_us, int32_t max_kernels, int32_t *n_kernels) {
    if (n_kernels) *n_kernels = 0;
    if (!d || d->n <= 0 || d->h <= 0 || d->w <= 0 || d->s < 1 || d->c_in <= 0 || d->c_mid <= 0 || d->c_out <= 0)
        return -1.0;
    if (d->stride != 1 && d->stride != 2) return -1.0;
    if (!(r >= 0.0 && r <= 1.0)) return -1.0;
    lasnet_hw def;
    if (!hw) {
        lasnet_hw_b200(&def);
        hw = &def;
    }
    Plan p;
    if (!build_plan(p, d, schedule, r)) return -1.0;
    const double sms = hw->sms > 0 ? hw->sms : 148;
    const double hbm_sm = hw->hbm_gbs * 1e3 / sms, l2_sm = hw->l2_gbs * 1e3 / sms;  // bytes per us per SM
    const double tc_sm = hw->tc_tflops * 1e6 / sms;                                  // flop per us per SM
    double total = 0;
    for (int i = 0; i < p.n; ++i) {
        const Work &w = p.k[i];
        const double eff = hw->eff[w.type] > 0 ? hw->eff[w.type] : 1.0;
        double t;
        if (w.tiles <= 0) {  // streaming: every SM busy
            t = std::fmax(w.hbm / (hbm_sm * sms), w.flops / (tc_sm * sms)) / eff;
        } else {
            const double rounds = std::ceil(w.tiles / sms);
            const double per_tile =
                std::fmax(std::fmax(w.hbm / w.tiles / hbm_sm, w.l2 / w.tiles / l2_sm), w.flops / w.tiles / tc_sm);
            // HBM is shared by all SMs: a partial last round does not speed up the HBM part
            t = std::fmax(rounds * per_tile, std::fmax(w.hbm / (hbm_sm * sms), w.flops / (tc_sm * sms))) / eff;
        }
        t += hw->launch_us + hw->t0_us[w.type];
        if (i < max_kernels) {
            if (kinds) kinds[i] = w.type;
            if (kernel_us) kernel_us[i] = t;
        }
        total += t;
    }
    if (n_kernels) *n_kernels = p.n;
    return total;
}

}  // extern "C"

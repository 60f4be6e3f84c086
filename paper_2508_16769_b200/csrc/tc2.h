// tc2.h — host interface of the warp-specialised tcgen05 GEMMs (internal).
//
// Every dense contraction of a HeteroConv layer is one of two shapes:
//   row GEMM  : Y[n x N] = sum_g-segments A_seg[n x K_seg] B_seg[K_seg x N]   (+ epilogue)
//               the forward projections (Eq. 4 W^psi) with the max-merge
//               epilogue (Eq. 8 / Eq. 14), and the backward dZ' = c (mask(dY) Wn^T)
//               (Eq. 10-13) with the Sage root term (mask(dY) Wr^T) sampled at the
//               CBSR indices fused as extra output columns;
//   reduce GEMM: dW[K_seg x N] = A_seg^T mask(dY) over all n rows, db = colsum(mask(dY)).
// Precision (north_star 1e-4): each fp32 operand is split x = hi + lo with hi, lo
// bf16 (hi = rn(x), lo = rn(x - hi); |x - hi - lo| <= 2^-17 |x|), and every
// product is hi*hi + hi*lo + lo*hi: 3 kind::f16 MMAs, fp32 accumulation in TMEM.
#pragma once
#include "dr_internal.h"

namespace dr {

enum { kMask2None = 0, kMask2M = 1, kMask2NotM = 2 };   // = kMaskNone/kMaskM/kMaskNotM
enum { kEpi2Fwd = 0, kEpi2Dz = 1 };

struct Tc2Seg {
    const float *A = nullptr;          // dense n x K row-major, or nullptr => CBSR
    bool split = false;                // A holds [hi | lo] bf16 rows (4 K bytes, K % 64 == 0)
    const float *hval = nullptr;       // CBSR n x k (values), idx n x k (uint8)
    const uint8_t *hidx = nullptr;
    int k = 0;
    int K = 0;                         // width of the segment (dense K, or CBSR dim)
    int mask_mode = kMask2None;        // dense only: route dY_cell by the merge mask
};

struct Tc2RowsDesc {
    int64_t n = 0;
    int N = 0;                         // output columns of one accumulator group
    int G = 1;                         // accumulator groups (2: near | pinned for the merge)
    int nseg[2] = {0, 0};
    Tc2Seg seg[2][2];
    const uint8_t *bimg[2] = {nullptr, nullptr};   // packed B per group (tc2_bimg_bytes)
    const uint32_t *mask_in = nullptr;             // n x ceil(mask_width/32) merge-mask words
    int mask_width = 0;
    int epi = kEpi2Fwd;
    // forward epilogue
    const float *bias[2] = {nullptr, nullptr};
    int merge = DR_MERGE_MAX;
    float *y = nullptr;
    uint32_t *mask_out = nullptr;
    float *tap_a = nullptr, *tap_b = nullptr;
    // dz epilogue: columns [0, n_dz) -> dz (n x n_dz) scaled by crow; columns
    // [n_dz, N) -> the root row, sampled at root_idx (n x root_k) -> root (n x root_k)
    int n_dz = 0;
    const float *crow = nullptr;
    float *dz = nullptr;
    // dz_split: write dz rows as [hi | lo] bf16 halves (x = hi + lo, |x - hi - lo| <=
    // 2^-17 |x|, 4 n_dz bytes per row as fp32 would take): the operand format the
    // tensor-core tiled SSpMM (tspmm.cu) gathers without converting
    bool dz_split = false;
    const uint8_t *root_idx = nullptr;
    int root_k = 0;
    float *root = nullptr;
    // forward epilogue, fused next-layer D-ReLU (row a5; Eq. 2-3 on this GEMM's
    // output y, after the merge): next_k > 0 also writes next_val / next_idx
    // (n x next_k CBSR, ascending columns, exactly next_k per row, ties -> lowest
    // column, values verbatim), bit-identical to launch_drelu on the written y.
    // y may be null then (the dense output is not stored).
    int next_k = 0;
    float *next_val = nullptr;
    uint8_t *next_idx = nullptr;
    // forward epilogue, fused linear head + MSE on Y (the last layer's Y_cell, G =
    // 2; reading Q14): with head_w set, writes head_dy = dL/dY (n x N) and, per CTA
    // c < grid (launch_tc2_rows' return value), head_part[c][0..N+2) = the partial
    // sums of y dp over rows, of dp and of r^2 (dp = 2 (pred - label) / n), which
    // launch_head_reduce finishes; y may be null.
    const float *head_w = nullptr, *head_b = nullptr, *labels = nullptr;
    float *head_dy = nullptr, *head_part = nullptr;
};
// shapes the fused next-layer D-ReLU covers (else: dense y + launch_drelu)
bool tc2_next_drelu_supported(int epi, int N, int k);

// Packed B image: per 64-wide K chunk, hi then lo, each Ntot rows x 128 B
// (bf16, K-major, 128-B swizzle).
size_t tc2_bimg_bytes(int K, int Ntot);
// rows [n0, n0 + NB) of the image of a K x Ntot operand:
// B_op[n0 + n][kk] = transpose ? W[kk*ldw + n] : W[n*ldw + kk].
void launch_tc2_pack_b(const float *W, int ldw, int K, int NB, int n0, int Ntot, bool transpose,
                       uint8_t *img, cudaStream_t s);
// one packing job (launch_tc2_pack_b's arguments); several in one launch
struct Tc2PackJob {
    const float *W = nullptr;
    int ldw = 0, K = 0, NB = 0, n0 = 0, Ntot = 0, transpose = 0;
    uint8_t *img = nullptr;
};
constexpr int kMaxPackJobs = 8;
void launch_tc2_pack_b_multi(const Tc2PackJob *jobs, int n, cudaStream_t s);
bool tc2_rows_supported(const Tc2RowsDesc &d);
int launch_tc2_rows(const Tc2RowsDesc &d, cudaStream_t s);   // returns the grid

struct Tc2RedSeg {
    const float *Z = nullptr;          // dense n x w, or nullptr => CBSR (hval/hidx/k, width w)
    bool split = false;                // Z holds [hi | lo] bf16 rows (4 w bytes)
    const float *hval = nullptr;
    const uint8_t *hidx = nullptr;
    int k = 0, w = 0;
    float *grad = nullptr;             // w x N row-major
};
struct Tc2ReduceDesc {
    int64_t n = 0;
    int N = 0, G = 1;                  // G accumulator groups of 128 feature rows
    int nseg[2] = {0, 0};              // segments stacked inside a group (widths sum <= 128)
    Tc2RedSeg seg[2][2];
    const float *dy = nullptr;
    const uint32_t *mask = nullptr;
    int mask_mode = kMask2None;
    float *db = nullptr;
    // dual B (the near + pinned weight gradients of a max-merge layer in one launch,
    // Eq. 12-13): mask_mode1 >= 0 gives group 1 its own B = mask_mode1(dY) and bias
    // gradient db1 (both B operands converted from one read of dY and the mask)
    int mask_mode1 = -1;
    float *db1 = nullptr;
};
bool tc2_reduce_supported(const Tc2ReduceDesc &d);
size_t tc2_reduce_work_floats(int G, int N);
// The reduce GEMM leaves per-CTA partials in `work`; a second, fixed-order pass
// sums them into the gradient tensors (deterministic, no atomics). With `defer`
// that pass is queued instead of launched, so a whole layer / step sums all its
// weight gradients in ONE launch (launch_tc2_reduce_parts, on a stream ordered
// after every queued reduce).
struct Tc2PartsJob {
    const float *part = nullptr;
    int nparts = 0, G = 0, N = 0, nout = 0;
    int g[4] = {0, 0, 0, 0}, m0[4] = {0, 0, 0, 0}, w[4] = {0, 0, 0, 0};
    float *dst[4] = {nullptr, nullptr, nullptr, nullptr};
    float *db = nullptr;
    float *db1 = nullptr;              // dual B: group 1's bias gradient
    int ndb = 1;                       // bias-gradient vectors after the G x 128 x N block
};
struct Tc2Deferred {
    static constexpr int kMax = 8;
    int n = 0;
    Tc2PartsJob job[kMax];
};
void launch_tc2_reduce(const Tc2ReduceDesc &d, float *work, cudaStream_t s,
                       Tc2Deferred *defer = nullptr);
void launch_tc2_reduce_parts(Tc2Deferred &defer, cudaStream_t s);   // flushes (n = 0 after)

}  // namespace dr

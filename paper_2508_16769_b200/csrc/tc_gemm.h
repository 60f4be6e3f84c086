// tc_gemm.h — host interface of the tcgen05 row-tile GEMMs (internal).
#pragma once
#include "dr_internal.h"

namespace dr {

enum { kEpiFwd = 0, kEpiDz = 1 };

struct TcSegDesc {
    const float *A = nullptr;           // dense n x K (row-major), or nullptr for CBSR
    const float *hval = nullptr;
    const uint8_t *hidx = nullptr;
    int k = 0;
    int K = 0;
    int mask_mode = 0;                  // dense segments: kMaskNone / kMaskM / kMaskNotM
};

struct TcRowsDesc {
    int64_t n = 0;
    int N = 0;
    int G = 1;
    int nseg[2] = {0, 0};
    TcSegDesc seg[2][2];
    const uint8_t *bimg[2] = {nullptr, nullptr};
    const uint32_t *mask_in = nullptr;
    int mask_in_width = 0;
    int epi = kEpiFwd;
    const float *bias[2] = {nullptr, nullptr};
    int merge = DR_MERGE_MAX;
    float *y = nullptr;
    uint32_t *mask_out = nullptr;
    float *tap_a = nullptr, *tap_b = nullptr;
    const float *crow = nullptr;
    float *dz = nullptr;
};

// Bytes of a packed B image for a K x NB operand (chunks of 32 K, hi + lo).
size_t tc_bimg_bytes(int K, int NB);
// Pack W into the image: B_op[n][kk] = transpose ? W[kk*ldw+n] : W[n*ldw+kk].
void launch_pack_b(const float *W, int ldw, int K, int NB, bool transpose, uint8_t *img,
                   cudaStream_t s);
bool tc_supported(int N);

// dW = Z^T mask(dY) over all rows, up to 2 accumulator groups of M=128 feature
// rows, each stacking up to 2 segments (dense Z or densified CBSR). grad of a
// segment is a w x N row-major matrix; db (N) = colsum(mask(dY)) if non-null.
struct TcRedSegDesc {
    const float *Z = nullptr;
    const float *hval = nullptr;
    const uint8_t *hidx = nullptr;
    int k = 0, w = 0;
    float *grad = nullptr;
};
struct TcReduceDesc {
    int64_t n = 0;
    int N = 0, G = 1;
    int nseg[2] = {0, 0};
    TcRedSegDesc seg[2][2];
    const float *dy = nullptr;
    const uint32_t *mask = nullptr;
    int mask_mode = 0;
    float *db = nullptr;
};
size_t tc_reduce_work_floats(int64_t n, int G, int N);
void launch_tc_reduce(const TcReduceDesc &d, float *work, cudaStream_t s);
void launch_tc_rows(const TcRowsDesc &d, cudaStream_t s);

}  // namespace dr

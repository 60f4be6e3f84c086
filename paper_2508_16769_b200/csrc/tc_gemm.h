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
void launch_tc_rows(const TcRowsDesc &d, cudaStream_t s);

}  // namespace dr

// proj.h — argument blocks of the dense-part kernels (internal).
#pragma once
#include "dr_internal.h"

namespace dr {

enum { kMaskNone = 0, kMaskM = 1, kMaskNotM = 2 };   // Eq. 12-13 routing of dY_cell

// Raise a kernel's dynamic shared-memory limit once.
void ensure_smem(const void *fn, size_t bytes);

struct ProjFwdArgs {
    int64_t n = 0;
    int Ka = 0, Kb = 0, N = 0;             // input widths of term a / b, output width
    const float *Za = nullptr, *Wa = nullptr, *ba = nullptr;
    const float *hval = nullptr;           // root term: densify(H) Wr (Wr == nullptr: none)
    const uint8_t *hidx = nullptr;
    int k = 0;
    const float *Wr = nullptr;
    const float *Zb = nullptr, *Wb = nullptr, *bb = nullptr;   // second relation (cell)
    int merge = DR_MERGE_MAX;
    float *y = nullptr;
    uint32_t *mask = nullptr;
    float *tap_a = nullptr, *tap_b = nullptr;
};
void launch_proj_fwd(const ProjFwdArgs &a, cudaStream_t s);

struct ProjBwdArgs {
    int64_t n = 0;
    int N = 0, K = 0;                      // dY width (d_out), output width (d_in)
    const float *dy = nullptr;
    const uint32_t *mask = nullptr;
    int mask_mode = kMaskNone;
    const float *W = nullptr;              // K x N
    const float *c = nullptr;              // row scale (dst normaliser) or nullptr
    float *dz = nullptr;                   // n x K
};
void launch_proj_bwd_dz(const ProjBwdArgs &a, cudaStream_t s);

struct RootArgs {
    int64_t n = 0;
    int N = 0, k = 0;
    const float *dy = nullptr;
    const uint32_t *mask = nullptr;
    int mask_mode = kMaskNone;
    const float *Wr = nullptr;             // d_in x N
    const uint8_t *hidx = nullptr;
    float *out = nullptr;                  // n x k
};
void launch_root_dots(const RootArgs &a, cudaStream_t s);

struct DwArgs {
    int64_t n = 0;
    int K = 0, N = 0;
    const float *Z = nullptr;              // n x K dense, or nullptr => densify(hval, hidx)
    const float *hval = nullptr;
    const uint8_t *hidx = nullptr;
    int k = 0;
    const float *dy = nullptr;
    const uint32_t *mask = nullptr;
    int mask_mode = kMaskNone;
    int rows_per_chunk = 0;
    float *part = nullptr, *part_b = nullptr;
};
int dw_num_chunks(int64_t n);
size_t dw_part_floats(int64_t n, int K, int N);
void launch_dw(DwArgs a, float *grad_w, float *grad_b, float *work, cudaStream_t s);

// Head + MSE (reading Q14): pred = y w_h + b_h over n cells; writes dy = dpred w_h^T,
// and (via fixed-order partials) grad_w (N), grad_b (1), loss (1).
struct HeadArgs {
    int64_t n = 0;
    int N = 0;
    const float *y = nullptr, *w = nullptr, *b = nullptr, *labels = nullptr;
    float *dy = nullptr, *grad_w = nullptr, *grad_b = nullptr, *loss = nullptr;
    float *work = nullptr;                 // head_work_floats(N)
};
size_t head_work_floats(int N);
void launch_head_mse(const HeadArgs &a, cudaStream_t s);
// Only the final fixed-order sum of `nparts` per-CTA head partials in a.work
// (the head fused into the last projection's epilogue, tc2.h head_w).
void launch_head_reduce(const HeadArgs &a, int nparts, cudaStream_t s);

// Adam with coupled L2 weight decay (reading Q15); grad is scaled by inv_world first.
void launch_adam(float *theta, const float *grad, float *m, float *v, int64_t n, float lr,
                 float wd, float b1, float b2, float eps, int64_t *step_dev, float inv_world,
                 cudaStream_t s);
void launch_scale(float *x, int64_t n, float a, cudaStream_t s);

}  // namespace dr

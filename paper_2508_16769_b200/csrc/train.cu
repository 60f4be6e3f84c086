// train.cu — linear head + MSE loss (reading Q14) and Adam (reading Q15, lr/wd
// of P:466) for the training step. Reductions over rows use a fixed number of
// per-CTA partials summed in a fixed order (deterministic, no atomics).
#include "proj.h"

namespace dr {
namespace {

constexpr int kHeadBlocks = 148 * 8;      // one wave at 8 x 256 threads per SM
constexpr int kHeadThreads = 256;
constexpr int kHeadU = 8;          // rows in flight per warp

// S = ceil(N / 32) column slots per lane (compile time: registers for kHeadU rows)
template <int S>
__global__ void __launch_bounds__(kHeadThreads) head_kernel(HeadArgs a, float inv_n) {
    __shared__ float wpart[kHeadThreads / 32][256 + 2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int N = a.N;
    float w[S], accw[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int o = lane + 32 * s;
        w[s] = o < N ? __ldg(a.w + o) : 0.f;
        accw[s] = 0.f;
    }
    const float b = __ldg(a.b);
    float accb = 0.f, accl = 0.f;
    const int64_t nw = (int64_t)gridDim.x * (kHeadThreads / 32);
    // kHeadU rows per warp iteration, all loads issued before the reductions
    // (the row loop is latency-bound otherwise: one dependent shuffle chain per row)
    for (int64_t j0 = ((int64_t)blockIdx.x * (kHeadThreads / 32) + wid) * kHeadU; j0 < a.n;
         j0 += nw * kHeadU) {
        float y[kHeadU][S], p[kHeadU], lab[kHeadU];
#pragma unroll
        for (int u = 0; u < kHeadU; ++u) {
            const int64_t j = j0 + u;
            const bool ok = j < a.n;
            lab[u] = ok ? __ldg(a.labels + j) : 0.f;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int o = lane + 32 * s;
                y[u][s] = (ok && o < N) ? __ldg(a.y + j * N + o) : 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < kHeadU; ++u) {
            p[u] = 0.f;
#pragma unroll
            for (int s = 0; s < S; ++s) p[u] += y[u][s] * w[s];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < kHeadU; ++u) p[u] += __shfl_xor_sync(0xffffffffu, p[u], o);
#pragma unroll
        for (int u = 0; u < kHeadU; ++u) {
            const int64_t j = j0 + u;
            if (j >= a.n) break;
            const float r = p[u] + b - lab[u];
            const float dp = 2.0f * r * inv_n;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int o = lane + 32 * s;
                if (o < N) a.dy[j * N + o] = dp * w[s];
                accw[s] += y[u][s] * dp;
            }
            accb += dp;
            accl += r * r;
        }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int o = lane + 32 * s;
        if (o < N) wpart[wid][o] = accw[s];
    }
    if (lane == 0) {
        wpart[wid][N] = accb;
        wpart[wid][N + 1] = accl;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < N + 2; e += blockDim.x) {
        float s = 0.f;
        for (int q = 0; q < kHeadThreads / 32; ++q) s += wpart[q][e];
        a.work[(int64_t)blockIdx.x * (N + 2) + e] = s;
    }
}

// One warp per output element: lanes take every 32nd block partial, then a
// fixed butterfly (deterministic; a single-thread loop over 296 dependent loads
// was latency-bound).
__global__ void head_reduce_kernel(HeadArgs a, float inv_n, int nparts) {
    const int N = a.N, lane = threadIdx.x & 31;
    const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (e >= N + 2) return;
    float s = 0.f;
    for (int q = lane; q < nparts; q += 32) s += a.work[(int64_t)q * (N + 2) + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane) return;
    if (e < N) a.grad_w[e] = s;
    else if (e == N) a.grad_b[0] = s;
    else a.loss[0] = s * inv_n;
}

// Adam step counter lives on the device (so a captured CUDA graph of the whole
// training step replays correctly): bump it, then every thread derives the bias
// corrections 1 - beta^t in double, exactly as the host formula did.
__global__ void step_bump_kernel(int64_t *step) { *step += 1; }

__global__ void adam_kernel(float *__restrict__ th, const float *__restrict__ g,
                            float *__restrict__ m, float *__restrict__ v, int64_t n, float lr,
                            float wd, float b1, float b2, float eps, const int64_t *step_dev,
                            float inv_world) {
    const double st = (double)*step_dev;
    const float bc1 = (float)(1.0 - pow((double)b1, st));
    const float bc2 = (float)(1.0 - pow((double)b2, st));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float t = th[i];
        const float gi = g[i] * inv_world + wd * t;        // coupled L2 (torch.optim.Adam)
        const float mi = b1 * m[i] + (1.f - b1) * gi;
        const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const float denom = sqrtf(vi / bc2) + eps;
        th[i] = t - lr * (mi / bc1) / denom;
    }
}

__global__ void scale_kernel(float *x, int64_t n, float a) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= a;
}

}  // namespace

size_t head_work_floats(int N) { return (size_t)kHeadBlocks * (N + 2); }

void launch_head_mse(const HeadArgs &a, cudaStream_t s) {
    const float inv_n = a.n > 0 ? 1.0f / (float)a.n : 0.f;
    ProfScope ps("head_mse", s);
    if (a.N <= 32) head_kernel<1><<<kHeadBlocks, kHeadThreads, 0, s>>>(a, inv_n);
    else if (a.N <= 64) head_kernel<2><<<kHeadBlocks, kHeadThreads, 0, s>>>(a, inv_n);
    else if (a.N <= 128) head_kernel<4><<<kHeadBlocks, kHeadThreads, 0, s>>>(a, inv_n);
    else head_kernel<8><<<kHeadBlocks, kHeadThreads, 0, s>>>(a, inv_n);
    note_launch("head_mse");
    head_reduce_kernel<<<(unsigned)((a.N + 2 + 7) / 8), 256, 0, s>>>(a, inv_n, kHeadBlocks);
    note_launch("head_reduce");
}

void launch_head_reduce(const HeadArgs &a, int nparts, cudaStream_t s) {
    const float inv_n = a.n > 0 ? 1.0f / (float)a.n : 0.f;
    ProfScope ps("head_mse", s);
    head_reduce_kernel<<<(unsigned)((a.N + 2 + 7) / 8), 256, 0, s>>>(a, inv_n, nparts);
    note_launch("head_reduce");
}

void launch_adam(float *theta, const float *grad, float *m, float *v, int64_t n, float lr,
                 float wd, float b1, float b2, float eps, int64_t *step_dev, float inv_world,
                 cudaStream_t s) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    step_bump_kernel<<<1, 1, 0, s>>>(step_dev);
    note_launch("step_bump");
    ProfScope ps("adam", s);
    adam_kernel<<<(unsigned)blocks, 256, 0, s>>>(theta, grad, m, v, n, lr, wd, b1, b2, eps,
                                                  step_dev, inv_world);
    note_launch("adam");
}

void launch_scale(float *x, int64_t n, float a, cudaStream_t s) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    scale_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, n, a);
    note_launch("scale");
}

}  // namespace dr

// drelu.cu — D-ReLU row-wise top-k → CBSR (Eq. 2-3; CBSR P:229).
//
// One warp per row. Lane l holds V consecutive columns [l*V, l*V+V), so column
// order is (lane, slot). Each value maps to an order-preserving uint32 key
// (x + 0.0f first, so -0.0 and +0.0 share a key and tie, reading Q5). The k-th
// largest key is found by the paper's "row-wise binary search": an
// MSB-first bitwise search whose probe counts are warp reductions
// (__reduce_add_sync). The search stops early once a probe selects exactly k
// keys. Survivors: key > T, plus the first (k - #{key > T}) keys == T in
// column order (exactly-k, ties to the lowest column). A warp exclusive scan
// gives each survivor its slot; outputs are idx-ascending (val, idx) pairs.
#include "dr_internal.h"

namespace dr {
namespace {

__device__ __forceinline__ uint32_t order_key(float x) {
    uint32_t u = __float_as_uint(x + 0.0f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int warp_excl_scan(int v, int lane) {
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    return inc - v;
}

template <int V>
__global__ void __launch_bounds__(256) drelu_kernel(const float *__restrict__ x, int64_t n,
                                                    int dim, int64_t ldx, int k, bool vec,
                                                    float *__restrict__ val,
                                                    uint8_t *__restrict__ idx) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = warp; r < n; r += nwarps) {
        const float *xr = x + r * ldx;
        float v[V];
        uint32_t key[V];
        if (vec) {  // dim == 32*V, 4V-byte aligned rows: one vector load per lane
            if constexpr (V == 1) {
                v[0] = __ldg(xr + lane);
            } else if constexpr (V == 2) {
                float2 q = __ldg(reinterpret_cast<const float2 *>(xr) + lane);
                v[0] = q.x; v[1] = q.y;
            } else if constexpr (V == 4) {
                float4 q = __ldg(reinterpret_cast<const float4 *>(xr) + lane);
                v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
            } else {
                float4 q0 = __ldg(reinterpret_cast<const float4 *>(xr) + 2 * lane);
                float4 q1 = __ldg(reinterpret_cast<const float4 *>(xr) + 2 * lane + 1);
                v[0] = q0.x; v[1] = q0.y; v[2] = q0.z; v[3] = q0.w;
                v[4] = q1.x; v[5] = q1.y; v[6] = q1.z; v[7] = q1.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < V; ++j) {
                int c = lane * V + j;
                v[j] = c < dim ? __ldg(xr + c) : 0.0f;
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j) key[j] = (lane * V + j < dim) ? order_key(v[j]) : 0u;

        // largest T with #{key >= T} >= k  (k-th largest key), early exit at == k
        uint32_t T = 0;
        bool exact = false;
        for (int b = 31; b >= 0; --b) {
            uint32_t cand = T | (1u << b);
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < V; ++j) cnt += key[j] >= cand;
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (cnt >= k) {
                T = cand;
                if (cnt == k) { exact = true; break; }
            }
        }
        bool sel[V];
        if (exact) {
#pragma unroll
            for (int j = 0; j < V; ++j) sel[j] = key[j] >= T;
        } else {
            int gt = 0, eq = 0;
#pragma unroll
            for (int j = 0; j < V; ++j) { gt += key[j] > T; eq += key[j] == T; }
            int need = k - __reduce_add_sync(0xffffffffu, gt);
            int rank = warp_excl_scan(eq, lane);
#pragma unroll
            for (int j = 0; j < V; ++j) {
                bool tie = key[j] == T;
                sel[j] = key[j] > T || (tie && rank < need);
                rank += tie;
            }
        }
        int ns = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) ns += sel[j];
        int pos = warp_excl_scan(ns, lane);
        float *vo = val + r * k;
        uint8_t *io = idx + r * k;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            if (sel[j]) {
                vo[pos] = v[j];
                io[pos] = (uint8_t)(lane * V + j);
                ++pos;
            }
        }
    }
}

}  // namespace

void launch_drelu(const float *x, int64_t n, int dim, int64_t ldx, int k, float *val,
                  uint8_t *idx, cudaStream_t s) {
    if (n <= 0) return;
    ProfScope ps("drelu", s);
    const int threads = 256, rows_per_cta = threads / 32;
    int64_t blocks = (n + rows_per_cta - 1) / rows_per_cta;
    if (blocks > 148 * 16) blocks = 148 * 16;
    const int V = dim <= 32 ? 1 : dim <= 64 ? 2 : dim <= 128 ? 4 : 8;
    const bool vec = dim == 32 * V && (ldx % V) == 0 &&
                     (reinterpret_cast<uintptr_t>(x) % (4 * V)) == 0;
    if (V == 1)
        drelu_kernel<1><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else if (V == 2)
        drelu_kernel<2><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else if (V == 4)
        drelu_kernel<4><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else
        drelu_kernel<8><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    note_launch("drelu");
}

}  // namespace dr

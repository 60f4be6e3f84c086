// proj.cu — the small dense parts of a HeteroConv layer (reported separately
// from the SpMM, north_star): per-module projections (Eq. 4 W^psi, P:236-238;
// SageConv fc_neigh + fc_self + bias, GraphConv weight + bias, reading Q2),
// the max-merge with its mask (Eq. 8, Eq. 14), and the
// backward dense parts (Eq. 12-13 mask routing, dW = Z^T dY, db, dZ = dY W^T,
// sampled root-term dots).
//
// Round-1 implementation: SIMT FFMA row tiles in fp32 (4 rows x 4 columns per
// thread, K staged through shared memory in chunks of 32). dW reductions over
// rows use per-CTA partials over contiguous row chunks followed by a
// fixed-order chunk sum, so every result is deterministic.
#include "dr_internal.h"
#include "proj.h"

namespace dr {
namespace {

constexpr int kThreads = 256;
constexpr int kKC = 32;          // K chunk staged in shared memory

__device__ __forceinline__ bool mask_keep(const uint32_t *mask, int mw, int64_t row, int col,
                                          int mode) {
    if (mode == kMaskNone) return true;
    const uint32_t m = (__ldg(mask + row * mw + (col >> 5)) >> (col & 31)) & 1u;
    return mode == kMaskM ? m != 0u : m == 0u;
}

// ------------------------------------------------------------------ forward projection
template <bool TWO>
__global__ void __launch_bounds__(kThreads) proj_fwd_kernel(ProjFwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int N = a.N, NQ = N >> 2, RG = kThreads / NQ, TM = 4 * RG;
    float *As = sm;                                   // [TM][kKC+1]
    float *Bs = sm + TM * (kKC + 1);                  // [kKC][N]
    const int tid = threadIdx.x, q = tid % NQ, rg = tid / NQ;
    const bool active = rg < RG;
    const int64_t r0 = (int64_t)blockIdx.x * TM;

    float acc[2][4][4];
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[g][i][c] = 0.f;

#pragma unroll
    for (int g = 0; g < (TWO ? 2 : 1); ++g) {
        const float *Z = g == 0 ? a.Za : a.Zb;
        const float *W = g == 0 ? a.Wa : a.Wb;
        const int K = g == 0 ? a.Ka : a.Kb;
        for (int kc = 0; kc < K; kc += kKC) {
            for (int e = tid; e < TM * kKC; e += kThreads) {
                const int rr = e / kKC, cc = e % kKC;
                const int64_t row = r0 + rr;
                As[rr * (kKC + 1) + cc] =
                    (row < a.n && kc + cc < K) ? __ldg(Z + row * K + kc + cc) : 0.f;
            }
            for (int e = tid; e < kKC * N; e += kThreads) {
                const int rr = e / N, cc = e % N;
                Bs[e] = (kc + rr < K) ? __ldg(W + (int64_t)(kc + rr) * N + cc) : 0.f;
            }
            __syncthreads();
            if (active) {
#pragma unroll 8
                for (int kk = 0; kk < kKC; ++kk) {
                    const float4 b = reinterpret_cast<const float4 *>(Bs + kk * N)[q];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float av = As[(rg * 4 + i) * (kKC + 1) + kk];
                        acc[g][i][0] += av * b.x;
                        acc[g][i][1] += av * b.y;
                        acc[g][i][2] += av * b.z;
                        acc[g][i][3] += av * b.w;
                    }
                }
            }
            __syncthreads();
        }
    }
    // epilogue
    const int lane = tid & 31;
    const int G = NQ < 8 ? NQ : 8;                    // quads per mask word
    const int mw = (N + 31) >> 5;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + rg * 4 + i;
        const bool ok = active && row < a.n;
        uint32_t nib = 0;
        if (ok) {
            float ya[4], yb[4];
            const float4 ba = reinterpret_cast<const float4 *>(a.ba)[q];
            ya[0] = acc[0][i][0] + ba.x; ya[1] = acc[0][i][1] + ba.y;
            ya[2] = acc[0][i][2] + ba.z; ya[3] = acc[0][i][3] + ba.w;
            if (a.Wr) {                               // sparse root term densify(H) Wr
                const float *hv = a.hval + row * a.k;
                const uint8_t *hi = a.hidx + row * a.k;
                for (int t = 0; t < a.k; ++t) {
                    const float v = __ldg(hv + t);
                    const float4 w = __ldg(reinterpret_cast<const float4 *>(
                                               a.Wr + (int64_t)__ldg(hi + t) * N) + q);
                    ya[0] += v * w.x; ya[1] += v * w.y; ya[2] += v * w.z; ya[3] += v * w.w;
                }
            }
            float y[4];
            if (TWO) {
                const float4 bb = reinterpret_cast<const float4 *>(a.bb)[q];
                yb[0] = acc[1][i][0] + bb.x; yb[1] = acc[1][i][1] + bb.y;
                yb[2] = acc[1][i][2] + bb.z; yb[3] = acc[1][i][3] + bb.w;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (a.merge == DR_MERGE_MAX) {
                        const bool m = ya[c] >= yb[c];          // Eq. 14: ties -> near
                        y[c] = m ? ya[c] : yb[c];
                        nib |= (uint32_t)m << c;
                    } else {
                        y[c] = ya[c] + yb[c];
                    }
                }
                if (a.tap_a)
                    reinterpret_cast<float4 *>(a.tap_a + row * N)[q] =
                        make_float4(ya[0], ya[1], ya[2], ya[3]);
                if (a.tap_b)
                    reinterpret_cast<float4 *>(a.tap_b + row * N)[q] =
                        make_float4(yb[0], yb[1], yb[2], yb[3]);
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c) y[c] = ya[c];
            }
            if (a.y)
                reinterpret_cast<float4 *>(a.y + row * N)[q] = make_float4(y[0], y[1], y[2], y[3]);
        }
        if (TWO && a.mask) {
            // assemble 32-bit mask words from G consecutive quads (lanes)
            uint32_t w = nib << (4 * (q % G));
            for (int o = 1; o < G; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
            if (ok && (q % G) == 0) a.mask[row * mw + (q * 4) / 32] = w;
        }
    }
    (void)lane;
}

// ------------------------------------------------------------------ dZ = c * (mask(dY) W^T)
__global__ void __launch_bounds__(kThreads) proj_bwd_dz_kernel(ProjBwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int K = a.K, N = a.N, NQ = K >> 2, RG = kThreads / NQ, TM = 4 * RG;
    const int mw = (N + 31) >> 5;
    float *As = sm;                                   // [TM][kKC+1]   masked dY chunk
    float *Bs = sm + TM * (kKC + 1);                  // [kKC][K]      W^T chunk
    const int tid = threadIdx.x, q = tid % NQ, rg = tid / NQ;
    const bool active = rg < RG;
    const int64_t r0 = (int64_t)blockIdx.x * TM;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][c] = 0.f;
    for (int oc = 0; oc < N; oc += kKC) {
        for (int e = tid; e < TM * kKC; e += kThreads) {
            const int rr = e / kKC, cc = e % kKC;
            const int64_t row = r0 + rr;
            const int o = oc + cc;
            float v = 0.f;
            if (row < a.n && o < N && mask_keep(a.mask, mw, row, o, a.mask_mode))
                v = __ldg(a.dy + row * N + o);
            As[rr * (kKC + 1) + cc] = v;
        }
        for (int e = tid; e < kKC * K; e += kThreads) {
            const int kk = e / kKC, cc = e % kKC;     // W[kk, oc+cc] -> Bs[cc][kk]
            Bs[cc * K + kk] = (oc + cc < N) ? __ldg(a.W + (int64_t)kk * N + oc + cc) : 0.f;
        }
        __syncthreads();
        if (active) {
#pragma unroll 8
            for (int cc = 0; cc < kKC; ++cc) {
                const float4 b = reinterpret_cast<const float4 *>(Bs + cc * K)[q];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float av = As[(rg * 4 + i) * (kKC + 1) + cc];
                    acc[i][0] += av * b.x;
                    acc[i][1] += av * b.y;
                    acc[i][2] += av * b.z;
                    acc[i][3] += av * b.w;
                }
            }
        }
        __syncthreads();
    }
    if (!active) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t row = r0 + rg * 4 + i;
        if (row >= a.n) continue;
        const float cr = a.c ? __ldg(a.c + row) : 1.0f;
        reinterpret_cast<float4 *>(a.dz + row * K)[q] =
            make_float4(cr * acc[i][0], cr * acc[i][1], cr * acc[i][2], cr * acc[i][3]);
    }
}

// ------------------------------------------------------------------ root[j,t] = mask(dY)[j,:] . Wr[idx[j,t],:]
__global__ void __launch_bounds__(kThreads) root_dots_kernel(RootArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
    const int N = a.N, mw = (N + 31) >> 5;
    for (int64_t j = warp; j < a.n; j += nw) {
        float dy[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            const int o = lane + 32 * s;
            dy[s] = (o < N && mask_keep(a.mask, mw, j, o, a.mask_mode)) ? __ldg(a.dy + j * N + o)
                                                                       : 0.f;
        }
        for (int t = 0; t < a.k; ++t) {
            const float *w = a.Wr + (int64_t)__ldg(a.hidx + j * a.k + t) * N;
            float p = 0.f;
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const int o = lane + 32 * s;
                if (o < N) p += dy[s] * __ldg(w + o);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (lane == 0) a.out[j * a.k + t] = p;
        }
    }
}

// ------------------------------------------------------------------ dW partials: Z^T mask(dY), colsum
// One CTA per contiguous row chunk; the K x N accumulator is split into 4x4
// blocks owned by threads (<= 4 blocks each, grid.y slices beyond). Rows are
// staged 32 at a time with 128-bit loads; the merge mask is applied per
// 4-column group from one 32-bit word. Partials go to part[chunk][K*N (+N)].
__global__ void __launch_bounds__(kThreads) dw_partial_kernel(DwArgs a) {
    extern __shared__ __align__(16) float sm[];
    constexpr int RS = 32;
    const int K = a.K, N = a.N, mw = (N + 31) >> 5, K4 = K >> 2, N4 = N >> 2;
    float *Zs = sm;                                   // [RS][K]
    float *Ys = sm + RS * K;                          // [RS][N]
    const int tid = threadIdx.x;
    const int NB = K4 * N4;
    const int blk0 = blockIdx.y * (4 * kThreads);     // this CTA's slice of 4x4 blocks
    const int64_t len = (int64_t)K * N + (a.part_b ? N : 0);
    float acc[4][4][4];
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[b][i][c] = 0.f;
    float bsum = 0.f;
    const int64_t rbeg = (int64_t)blockIdx.x * a.rows_per_chunk;
    const int64_t rend = min((int64_t)a.n, rbeg + a.rows_per_chunk);
    for (int64_t rb = rbeg; rb < rend; rb += RS) {
        if (a.Z) {
            for (int e = tid; e < RS * K4; e += kThreads) {
                const int rr = e / K4, c4 = e % K4;
                const int64_t row = rb + rr;
                reinterpret_cast<float4 *>(Zs)[e] =
                    row < rend ? __ldg(reinterpret_cast<const float4 *>(a.Z + row * K) + c4)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        } else {                                      // densify the CBSR rows
            for (int e = tid; e < RS * K4; e += kThreads)
                reinterpret_cast<float4 *>(Zs)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncthreads();
            for (int e = tid; e < RS * a.k; e += kThreads) {
                const int rr = e / a.k, t = e % a.k;
                const int64_t row = rb + rr;
                if (row < rend)
                    Zs[rr * K + __ldg(a.hidx + row * a.k + t)] = __ldg(a.hval + row * a.k + t);
            }
        }
        for (int e = tid; e < RS * N4; e += kThreads) {
            const int rr = e / N4, c4 = e % N4;
            const int64_t row = rb + rr;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (row < rend) {
                v = __ldg(reinterpret_cast<const float4 *>(a.dy + row * N) + c4);
                if (a.mask_mode != kMaskNone) {
                    uint32_t bits = (__ldg(a.mask + row * mw + (c4 >> 3)) >> (4 * (c4 & 7))) & 0xfu;
                    if (a.mask_mode == kMaskNotM) bits = ~bits;
                    if (!(bits & 1u)) v.x = 0.f;
                    if (!(bits & 2u)) v.y = 0.f;
                    if (!(bits & 4u)) v.z = 0.f;
                    if (!(bits & 8u)) v.w = 0.f;
                }
            }
            reinterpret_cast<float4 *>(Ys)[e] = v;
        }
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int blk = blk0 + tid + b * kThreads;
            if (blk >= NB) break;
            const int bk = blk / N4, bo = blk % N4;
#pragma unroll 4
            for (int rr = 0; rr < RS; ++rr) {
                const float4 z = reinterpret_cast<const float4 *>(Zs + rr * K)[bk];
                const float4 y = reinterpret_cast<const float4 *>(Ys + rr * N)[bo];
                const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    acc[b][i][0] += zz[i] * y.x;
                    acc[b][i][1] += zz[i] * y.y;
                    acc[b][i][2] += zz[i] * y.z;
                    acc[b][i][3] += zz[i] * y.w;
                }
            }
        }
        if (a.part_b && blockIdx.y == 0 && tid < N)
            for (int rr = 0; rr < RS; ++rr) bsum += Ys[rr * N + tid];
        __syncthreads();
    }
    float *out = a.part + (int64_t)blockIdx.x * len;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const int blk = blk0 + tid + b * kThreads;
        if (blk >= NB) break;
        const int bk = blk / N4, bo = blk % N4;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            reinterpret_cast<float4 *>(out + (int64_t)(bk * 4 + i) * N)[bo] =
                make_float4(acc[b][i][0], acc[b][i][1], acc[b][i][2], acc[b][i][3]);
    }
    if (a.part_b && blockIdx.y == 0 && tid < N) out[(int64_t)K * N + tid] = bsum;
}

// out[e] = sum_{c < n_parts} part[c*len + e] in a fixed order: block (32 x 8),
// thread (e, s) sums chunks c = s, s+8, ..., then the 8 slices are added in order.
__global__ void reduce_parts_kernel(const float *__restrict__ part, int n_parts, int64_t len,
                                    int64_t len_w, float *__restrict__ out_w,
                                    float *__restrict__ out_b) {
    __shared__ float red[8][33];
    const int64_t e = (int64_t)blockIdx.x * 32 + threadIdx.x;
    float acc = 0.f;
    if (e < len)
        for (int c = threadIdx.y; c < n_parts; c += 8) acc += __ldg(part + (int64_t)c * len + e);
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && e < len) {
        float s = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x];
        if (e < len_w) out_w[e] = s;
        else if (out_b) out_b[e - len_w] = s;
    }
}

}  // namespace

// ------------------------------------------------------------------ launchers
static size_t proj_tile_rows(int N) { return 4 * (kThreads / (N >> 2)); }

void launch_proj_fwd(const ProjFwdArgs &a, cudaStream_t s) {
    if (a.n <= 0) return;
    const int TM = (int)proj_tile_rows(a.N);
    const size_t smem = ((size_t)TM * (kKC + 1) + (size_t)kKC * a.N) * 4;
    const unsigned grid = (unsigned)((a.n + TM - 1) / TM);
    ProfScope ps("proj_fwd", s);
    if (a.Zb) {
        ensure_smem((const void *)proj_fwd_kernel<true>, smem);
        proj_fwd_kernel<true><<<grid, kThreads, smem, s>>>(a);
    } else {
        ensure_smem((const void *)proj_fwd_kernel<false>, smem);
        proj_fwd_kernel<false><<<grid, kThreads, smem, s>>>(a);
    }
    note_launch("proj_fwd");
}

void launch_proj_bwd_dz(const ProjBwdArgs &a, cudaStream_t s) {
    if (a.n <= 0) return;
    const int TM = (int)proj_tile_rows(a.K);
    const size_t smem = ((size_t)TM * (kKC + 1) + (size_t)kKC * a.K) * 4;
    const unsigned grid = (unsigned)((a.n + TM - 1) / TM);
    ensure_smem((const void *)proj_bwd_dz_kernel, smem);
    ProfScope ps("proj_bwd_dz", s);
    proj_bwd_dz_kernel<<<grid, kThreads, smem, s>>>(a);
    note_launch("proj_bwd_dz");
}

void launch_root_dots(const RootArgs &a, cudaStream_t s) {
    if (a.n <= 0) return;
    int64_t blocks = (a.n + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    ProfScope ps("root_dots", s);
    root_dots_kernel<<<(unsigned)blocks, kThreads, 0, s>>>(a);
    note_launch("root_dots");
}

int dw_num_chunks(int64_t n) {
    int64_t c = (n + 511) / 512;
    if (c > 148) c = 148;
    if (c < 1) c = 1;
    return (int)c;
}

size_t dw_part_floats(int64_t n, int K, int N) {
    return (size_t)dw_num_chunks(n) * ((size_t)K * N + N);
}

// grad_w (K x N) = Z^T mask(dY); grad_b (N) = colsum(mask(dY)) if non-null.
void launch_dw(DwArgs a, float *grad_w, float *grad_b, float *work, cudaStream_t s) {
    ProfScope ps("dw", s);
    const int chunks = a.n > 0 ? dw_num_chunks(a.n) : 0;
    a.rows_per_chunk = chunks ? (int)((a.n + chunks - 1) / chunks) : 0;
    a.part = work;
    a.part_b = grad_b ? work : nullptr;             // flag only: bias lives after K*N per chunk
    const int64_t len_w = (int64_t)a.K * a.N, len = len_w + (grad_b ? a.N : 0);
    if (chunks) {
        const size_t smem = (size_t)32 * (a.K + a.N) * 4;
        const int NB = (a.K / 4) * (a.N / 4);
        dim3 grid((unsigned)chunks, (unsigned)((NB + 4 * kThreads - 1) / (4 * kThreads)));
        ensure_smem((const void *)dw_partial_kernel, smem);
        dw_partial_kernel<<<grid, kThreads, smem, s>>>(a);
        note_launch("dw_partial");
    }
    reduce_parts_kernel<<<(unsigned)((len + 31) / 32), dim3(32, 8), 0, s>>>(work, chunks, len, len_w,
                                                                             grad_w, grad_b);
    note_launch("reduce_parts");
}

}  // namespace dr

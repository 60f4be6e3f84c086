// spmm.cu — DR-SpMM forward (Alg. 1, Eq. 5-7) and SSpMM backward (Alg. 2,
// Eq. 10-11) over CBSR operands, for sm_100a.
//
// Lane mapping (Alg. 1 stage 2, "partition into ceil(32/K) parts"):
// a warp is split into R = 32/L sub-warps of L = k/P lanes; each lane owns P of
// a CBSR row's k pairs (P = 4: one 128-bit value load + one 32-bit index load
// per neighbour). Rows are processed in the graph's degree-descending order and
// split into the three degree classes of stage 2:
//   sub rows  (deg <= 32):         R rows per warp, one sub-warp per row;
//   warp rows (32 < deg <= 256):   one row per warp, the R sub-warps take every
//                                  R-th neighbour, private partial rows are summed
//                                  in a fixed order at the end;
//   hub rows  (deg > 256, "evil rows" §2.3): one CTA per row, its
//                                  sub-warps take contiguous neighbour chunks,
//                                  partials summed in a fixed order.
// Every output element has one owner and a fixed summation order: no atomics
// anywhere (reading Q23), bit-reproducible results.
//
// Forward: sub-warps accumulate densify(H_j) into D-float shared-memory rows.
// The k indices of one CBSR row are distinct, so a sub-warp's lanes never
// collide; each neighbour's P read-modify-writes are issued loads-first.
// Backward: each lane keeps P of the source row's k CBSR indices in registers
// and pulls dz[i, idx] over the CSC list (sampled gather) into registers;
// warp rows reduce across sub-warps with a shuffle butterfly. The D-ReLU mask
// gradient is the scatter of those k values into a zero row.
#include <cstdlib>

#include "dr_internal.h"

namespace dr {
namespace {

// x = hi + lo in bf16 (round to nearest), two values packed per word (a low half)
__device__ __forceinline__ void tc_split_bf16x2(float a, float b, uint32_t &hi, uint32_t &lo) {
    uint32_t h, l;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(b), "f"(a));
    const float ha = __uint_as_float(h << 16), hb = __uint_as_float(h & 0xffff0000u);
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(b - hb), "f"(a - ha));
    hi = h;
    lo = l;
}

constexpr int kU = 4;           // neighbours in flight per lane (memory-level parallelism)
constexpr int kHubCtas = 296;   // 2 per SM

template <int P>
struct Pairs {
    float v[P];
    uint32_t id[P];
};

template <int P>
__device__ __forceinline__ void load_pairs(const float *__restrict__ hval,
                                           const uint8_t *__restrict__ hidx, int64_t off,
                                           Pairs<P> &o) {
    if constexpr (P == 4) {
        float4 q = __ldg(reinterpret_cast<const float4 *>(hval + off));
        uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(hidx + off));
        o.v[0] = q.x; o.v[1] = q.y; o.v[2] = q.z; o.v[3] = q.w;
        o.id[0] = w & 0xff; o.id[1] = (w >> 8) & 0xff; o.id[2] = (w >> 16) & 0xff; o.id[3] = w >> 24;
    } else if constexpr (P == 2) {
        float2 q = __ldg(reinterpret_cast<const float2 *>(hval + off));
        uint32_t w = __ldg(reinterpret_cast<const uint16_t *>(hidx + off));
        o.v[0] = q.x; o.v[1] = q.y;
        o.id[0] = w & 0xff; o.id[1] = w >> 8;
    } else {
        o.v[0] = __ldg(hval + off);
        o.id[0] = __ldg(hidx + off);
    }
}

// Accumulate neighbours e0, e0+stride, ... < e1 of one row into `acc` (shared,
// D floats). Column ids and weights are prefetched one iteration ahead.
template <int P, bool PEER = false>
__device__ __forceinline__ void fwd_accumulate(int e0, int e1, int stride,
                                               const int32_t *__restrict__ col,
                                               const float *__restrict__ ew,
                                               const float *__restrict__ hval,
                                               const uint8_t *__restrict__ hidx, int k, int ll,
                                               float *acc, int kr, unsigned smask,
                                               const PeerSrc *ps = nullptr) {
    int jn[kU];
    float wn[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const int ee = e0 + u * stride;
        const bool ok = ee < e1;
        jn[u] = ok ? __ldg(col + ee) : -1;
        wn[u] = (ok && ew) ? __ldg(ew + ee) : 1.0f;
    }
    for (int e = e0; e < e1; e += kU * stride) {
        int j[kU];
        float w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) { j[u] = jn[u]; w[u] = wn[u]; }
        Pairs<P> pr[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (j[u] >= 0 && ll * P < kr) {                    // lanes beyond the K prefix idle
                if constexpr (PEER) {   // row j of owner q = j / m, read in place (peer memory)
                    const int q = j[u] / ps->m, loc = j[u] - q * ps->m;
                    load_pairs<P>(ps->pv[q], ps->pi[q], (int64_t)loc * k + ll * P, pr[u]);
                } else {
                    load_pairs<P>(hval, hidx, (int64_t)j[u] * k + ll * P, pr[u]);
                }
#pragma unroll
                for (int p = 0; p < P; ++p)
                    if (ll * P + p >= kr) pr[u].v[p] = 0.f;     // beyond this row's K prefix
            }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int ee = e + (kU + u) * stride;
            const bool ok = ee < e1;
            jn[u] = ok ? __ldg(col + ee) : -1;
            wn[u] = (ok && ew) ? __ldg(ew + ee) : 1.0f;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (j[u] >= 0 && ll * P < kr) {
                float old[P];
#pragma unroll
                for (int p = 0; p < P; ++p) old[p] = acc[pr[u].id[p]];
#pragma unroll
                for (int p = 0; p < P; ++p) acc[pr[u].id[p]] = old[p] + w[u] * pr[u].v[p];
            }
            // lanes of the sub-warp may hit the same column for the next neighbour:
            // order this read-modify-write before theirs (independent thread scheduling)
            __syncwarp(smask);
        }
    }
}

struct FwdArgs {
    PeerSrc peer;                    // f4 fused exchange (PEER kernels only)
    const int32_t *order;
    int32_t n_hub, n_warp, n_rows;   // [0,n_hub) hubs, [n_hub,n_hub+n_warp) warp rows, rest sub
    int32_t hub_ctas, warp_ctas;     // block ranges: hubs, warp rows, then sub rows
    const int32_t *rowptr, *col;
    const float *ew, *c;
    const float *hval;
    const uint8_t *hidx;
    int k, D, L;
    float *z;
    int z_split;                     // z rows as [hi | lo] bf16 halves (4 D bytes per row)
    NgSched ng;                      // per-neighbour-group K (value-sorted CBSR prefix)
};

__device__ __forceinline__ int ng_k(const NgSched &ng, int deg, int k) {
    if (!ng.on) return k;
    return deg <= ng.thr0 ? ng.kb0 : deg <= ng.thr1 ? ng.kb1 : ng.kb2;
}

// Z output: fp32, or split bf16 halves (x = hi + lo, the tensor-core operand
// format of the projection / dW kernels, tc2.h)
__device__ __forceinline__ void store_z4(const FwdArgs &a, int row, int c4, float4 v) {
    if (!a.z_split) {
        __stcs(reinterpret_cast<float4 *>(a.z + (int64_t)row * a.D) + c4, v);
        return;
    }
    uint2 h, l;
    tc_split_bf16x2(v.x, v.y, h.x, l.x);
    tc_split_bf16x2(v.z, v.w, h.y, l.y);
    uint8_t *rowp = reinterpret_cast<uint8_t *>(a.z) + (int64_t)row * a.D * 4;
    __stcs(reinterpret_cast<uint2 *>(rowp + 8 * c4), h);
    __stcs(reinterpret_cast<uint2 *>(rowp + 2 * a.D + 8 * c4), l);
}
__device__ __forceinline__ void store_z1(const FwdArgs &a, int row, int c, float v) {
    if (!a.z_split) {
        a.z[(int64_t)row * a.D + c] = v;
        return;
    }
    uint32_t h, l;
    tc_split_bf16x2(v, 0.f, h, l);
    uint16_t *rowp = reinterpret_cast<uint16_t *>(a.z) + (int64_t)row * a.D * 2;
    rowp[c] = (uint16_t)(h & 0xffffu);
    rowp[a.D + c] = (uint16_t)(l & 0xffffu);
}

template <int P, bool PEER = false>
__global__ void __launch_bounds__(256, 4) spmm_fwd_kernel(const __grid_constant__ FwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int L = a.L, R = 32 / L, sub = lane / L, ll = lane % L, D = a.D, D4 = D >> 2;
    float *acc = sm + (size_t)(wid * R + sub) * D;
    float4 *acc4 = reinterpret_cast<float4 *>(acc);
    const unsigned smask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (sub * L));
    const int b = blockIdx.x;

    if (b < a.hub_ctas) {
        // ---- hub rows: CTA per row, contiguous chunks per sub-warp, fixed-order sum
        const int S = wpc * R, sidx = wid * R + sub;
        for (int h = b; h < a.n_hub; h += a.hub_ctas) {
            const int row = __ldg(a.order + h);
            const int e0 = __ldg(a.rowptr + row), e1 = __ldg(a.rowptr + row + 1);
            for (int c4 = ll; c4 < D4; c4 += L) acc4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            const int chunk = (e1 - e0 + S - 1) / S;
            const int b0 = min(e1, e0 + sidx * chunk), b1 = min(e1, b0 + chunk);
            fwd_accumulate<P, PEER>(b0, b1, 1, a.col, a.ew, a.hval, a.hidx, a.k, ll, acc,
                                    ng_k(a.ng, e1 - e0, a.k), smask, &a.peer);
            __syncthreads();
            const float cr = __ldg(a.c + row);
            for (int cc = threadIdx.x; cc < D; cc += blockDim.x) {
                float s = 0.f;
                for (int q = 0; q < S; ++q) s += sm[(size_t)q * D + cc];
                store_z1(a, row, cc, cr * s);
            }
            __syncthreads();
        }
        return;
    }
    if (b < a.hub_ctas + a.warp_ctas) {
        // ---- warp rows: R sub-warps interleave the neighbour list
        const int pos = a.n_hub + (b - a.hub_ctas) * wpc + wid;
        const bool valid = pos < a.n_hub + a.n_warp;
        const int row = valid ? __ldg(a.order + pos) : 0;
        for (int c4 = ll; c4 < D4; c4 += L) acc4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        if (valid) {
            const int e0 = __ldg(a.rowptr + row), e1 = __ldg(a.rowptr + row + 1);
            fwd_accumulate<P, PEER>(e0 + sub, e1, R, a.col, a.ew, a.hval, a.hidx, a.k, ll, acc,
                                    ng_k(a.ng, e1 - e0, a.k), smask, &a.peer);
        }
        __syncwarp();
        if (valid) {
            const float cr = __ldg(a.c + row);
            const float4 *w4 = reinterpret_cast<const float4 *>(sm + (size_t)wid * R * D);
            for (int c4 = lane; c4 < D4; c4 += 32) {
                float4 s = w4[c4];
                for (int q = 1; q < R; ++q) {
                    const float4 t = w4[(size_t)q * D4 + c4];
                    s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
                }
                store_z4(a, row, c4, make_float4(cr * s.x, cr * s.y, cr * s.z, cr * s.w));
            }
        }
        return;
    }
    // ---- sub rows: R rows per warp
    const int64_t gw = (int64_t)(b - a.hub_ctas - a.warp_ctas) * wpc + wid;
    const int64_t pos = (int64_t)a.n_hub + a.n_warp + gw * R + sub;
    const bool valid = pos < a.n_rows;
    const int row = valid ? __ldg(a.order + pos) : 0;
    for (int c4 = ll; c4 < D4; c4 += L) acc4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    if (valid) {
        const int e0 = __ldg(a.rowptr + row), e1 = __ldg(a.rowptr + row + 1);
        fwd_accumulate<P, PEER>(e0, e1, 1, a.col, a.ew, a.hval, a.hidx, a.k, ll, acc,
                                ng_k(a.ng, e1 - e0, a.k), smask, &a.peer);
    }
    __syncwarp();
    // the warp's R accumulator rows are contiguous in shared memory: store them
    // together, D/4 consecutive lanes per row (coalesced rows, also for split Z)
    const float4 *w4 = reinterpret_cast<const float4 *>(sm + (size_t)wid * R * D);
    const int64_t pos0 = (int64_t)a.n_hub + a.n_warp + gw * R;
    const int rpi = (D4 < 32 && 32 % D4 == 0) ? 32 / D4 : 1;      // rows per warp pass
    const int lr = rpi > 1 ? lane / D4 : 0, lc = rpi > 1 ? lane - lr * D4 : lane;
    const int cstep = rpi > 1 ? D4 : 32;
    // row ids and scales of the warp's R rows, fetched at once (lane r holds row r)
    const bool lok = lane < R && pos0 + lane < a.n_rows;
    const int rw_l = lok ? __ldg(a.order + pos0 + lane) : 0;
    const float cr_l = lok ? __ldg(a.c + rw_l) : 0.f;
    for (int r0 = 0; r0 < R; r0 += rpi) {
        const int r = r0 + lr;
        const int rw = __shfl_sync(0xffffffffu, rw_l, r & 31);
        const float cr = __shfl_sync(0xffffffffu, cr_l, r & 31);
        if (r >= R || pos0 + r >= a.n_rows) continue;
        for (int c4 = lc; c4 < D4; c4 += cstep) {
            const float4 v = w4[r * D4 + c4];
            store_z4(a, rw, c4, make_float4(cr * v.x, cr * v.y, cr * v.z, cr * v.w));
        }
    }
}

// ------------------------------------------------------------------ backward
struct TermDev {
    const int32_t *colptr, *row;
    const float *ewT, *s, *c;    // c != nullptr: apply c_i per edge (standalone ABI)
    const float *dz;
};

struct BwdArgs {
    PeerSrc peer;                    // f4 fused exchange (PEER kernels only)
    const int32_t *order;
    int32_t n_hub, n_warp, n_rows, hub_ctas, warp_ctas;
    TermDev t[2];
    int n_terms;
    const float *root;
    const uint8_t *hidx;
    int k, D, L;
    float *g_kept, *dx;
    int accumulate;
    NgSched ng;
};

// Pull dz[i, id[p]] over CSC entries e0, e0+stride, ... < e1 into a[p].
// NEXT-2 (ng.on): destination i used only the first K(deg_i) = ng.kT[e] entries of
// this source row, so positions pos0 + p >= K(deg_i) neither load nor add.
template <int P>
__device__ __forceinline__ void bwd_term(const TermDev &t, int e0, int e1, int stride,
                                         const uint32_t *id, int D, float *a, const NgSched &ng,
                                         int pos0, int k) {
    int in[kU], kn[kU];
    float wn[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        const int ee = e0 + u * stride;
        const bool ok = ee < e1;
        in[u] = ok ? __ldg(t.row + ee) : -1;
        wn[u] = (ok && t.ewT) ? __ldg(t.ewT + ee) : 1.0f;
        kn[u] = (ok && ng.on) ? (int)__ldg(ng.kT + ee) : k;
    }
    for (int e = e0; e < e1; e += kU * stride) {
        int i[kU], ki[kU];
        float w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) { i[u] = in[u]; w[u] = wn[u]; ki[u] = kn[u]; }
        float v[kU][P];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
#pragma unroll
            for (int p = 0; p < P; ++p) v[u][p] = 0.f;
            if (i[u] >= 0 && pos0 < ki[u]) {
                const float *dzr = t.dz + (int64_t)i[u] * D;
#pragma unroll
                for (int p = 0; p < P; ++p)
                    if (pos0 + p < ki[u]) v[u][p] = __ldg(dzr + id[p]);
                if (t.c) w[u] *= __ldg(t.c + i[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int ee = e + (kU + u) * stride;
            const bool ok = ee < e1;
            in[u] = ok ? __ldg(t.row + ee) : -1;
            wn[u] = (ok && t.ewT) ? __ldg(t.ewT + ee) : 1.0f;
            kn[u] = (ok && ng.on) ? (int)__ldg(ng.kT + ee) : k;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (i[u] >= 0) {
#pragma unroll
                for (int p = 0; p < P; ++p) a[p] += w[u] * v[u][p];
            }
    }
}

template <int P>
__device__ __forceinline__ void load_idx(const uint8_t *__restrict__ hidx, int64_t off,
                                         uint32_t *id) {
    if constexpr (P == 4) {
        uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(hidx + off));
        id[0] = w & 0xff; id[1] = (w >> 8) & 0xff; id[2] = (w >> 16) & 0xff; id[3] = w >> 24;
    } else if constexpr (P == 2) {
        uint32_t w = __ldg(reinterpret_cast<const uint16_t *>(hidx + off));
        id[0] = w & 0xff; id[1] = w >> 8;
    } else {
        id[0] = __ldg(hidx + off);
    }
}

// source row j's CBSR indices and its g row (PEER: the owner's buffers / inbox slot)
template <bool PEER>
__device__ __forceinline__ const uint8_t *idx_row(const BwdArgs &a, int j) {
    if constexpr (PEER) {
        const int q = j / a.peer.m;
        return a.peer.pi[q] + (int64_t)(j - q * a.peer.m) * a.k;
    }
    return a.hidx + (int64_t)j * a.k;
}
template <bool PEER>
__device__ __forceinline__ float *g_row(const BwdArgs &a, int j) {
    if constexpr (PEER) {
        const int q = j / a.peer.m;
        return a.peer.pg[q] + ((int64_t)a.peer.rank * a.peer.m + (j - q * a.peer.m)) * a.k;
    }
    return a.g_kept + (int64_t)j * a.k;
}

// Write lane ll's P values of source row j: g_kept and/or the dense dX row
// (zeros + k values, staged in the sub-warp's shared row). Whole warp calls it.
template <int P, bool PEER = false>
__device__ __forceinline__ void bwd_store(const BwdArgs &a, bool valid, int j, int ll,
                                          const uint32_t *id, const float *g, float *srow) {
    const int D = a.D, D4 = D >> 2, L = a.L;
    if (valid && (PEER || a.g_kept)) {
        float *gk = g_row<PEER>(a, j) + ll * P;
#pragma unroll
        for (int p = 0; p < P; ++p) gk[p] = a.accumulate ? gk[p] + g[p] : g[p];
    }
    if (!a.dx) return;
    if (a.accumulate) {
        if (valid) {
            float *dr = a.dx + (int64_t)j * D;
#pragma unroll
            for (int p = 0; p < P; ++p) dr[id[p]] += g[p];
        }
        return;
    }
    float4 *s4 = reinterpret_cast<float4 *>(srow);
    if (valid)
        for (int c4 = ll; c4 < D4; c4 += L) s4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    if (valid) {
#pragma unroll
        for (int p = 0; p < P; ++p) srow[id[p]] = g[p];
    }
    __syncwarp();
    if (valid) {
        float4 *d4 = reinterpret_cast<float4 *>(a.dx + (int64_t)j * D);
        for (int c4 = ll; c4 < D4; c4 += L) __stcs(d4 + c4, s4[c4]);
    }
    __syncwarp();
}

template <int P, bool PEER = false>
__global__ void __launch_bounds__(256, 4) spmm_bwd_kernel(const __grid_constant__ BwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int L = a.L, R = 32 / L, sub = lane / L, ll = lane % L;
    float *srow = sm + (size_t)(wid * R + sub) * a.D;
    const int b = blockIdx.x;

    if (b < a.hub_ctas) {
        // ---- hub source rows: partials over contiguous chunks, fixed-order sum
        const int S = wpc * R, sidx = wid * R + sub;
        float *part = sm;                            // [S][k] partials + final row
        for (int h = b; h < a.n_hub; h += a.hub_ctas) {
            const int j = __ldg(a.order + h);
            uint32_t id[P];
            load_idx<P>(idx_row<PEER>(a, j), ll * P, id);
            float g[P];
#pragma unroll
            for (int p = 0; p < P; ++p) g[p] = 0.f;
            for (int q = 0; q < a.n_terms; ++q) {
                const TermDev &t = a.t[q];
                const int e0 = __ldg(t.colptr + j), e1 = __ldg(t.colptr + j + 1);
                const int chunk = (e1 - e0 + S - 1) / S;
                const int b0 = min(e1, e0 + sidx * chunk), b1 = min(e1, b0 + chunk);
                float acc[P];
#pragma unroll
                for (int p = 0; p < P; ++p) acc[p] = 0.f;
                bwd_term<P>(t, b0, b1, 1, id, a.D, acc, a.ng, ll * P, a.k);
                const float sj = __ldg(t.s + j);
#pragma unroll
                for (int p = 0; p < P; ++p) g[p] += sj * acc[p];
            }
            __syncthreads();                         // previous iteration done with `part`
#pragma unroll
            for (int p = 0; p < P; ++p) part[(size_t)sidx * a.k + ll * P + p] = g[p];
            __syncthreads();
            if (threadIdx.x < a.k) {
                const int t = threadIdx.x;
                float s = 0.f;
                for (int q = 0; q < S; ++q) s += part[(size_t)q * a.k + t];
                if (a.root) s += __ldg(a.root + (int64_t)j * a.k + t);
                part[(size_t)S * a.k + t] = s;
            }
            __syncthreads();
            if (wid == 0 && sub == 0) {
                float gf[P];
#pragma unroll
                for (int p = 0; p < P; ++p) gf[p] = part[(size_t)S * a.k + ll * P + p];
                if (PEER || a.g_kept) {
                    float *gk = g_row<PEER>(a, j) + ll * P;
#pragma unroll
                    for (int p = 0; p < P; ++p) gk[p] = a.accumulate ? gk[p] + gf[p] : gf[p];
                }
                if (a.dx) {
                    float *dr = a.dx + (int64_t)j * a.D;
                    if (!a.accumulate)
                        for (int cc = ll; cc < a.D; cc += L) dr[cc] = 0.f;
                    __syncwarp(L == 32 ? 0xffffffffu : ((1u << L) - 1u));
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        if (a.accumulate) dr[id[p]] += gf[p];
                        else dr[id[p]] = gf[p];
                    }
                }
            }
        }
        return;
    }
    const bool warp_rows = b < a.hub_ctas + a.warp_ctas;
    int64_t pos;
    if (warp_rows) pos = (int64_t)a.n_hub + (int64_t)(b - a.hub_ctas) * wpc + wid;
    else pos = (int64_t)a.n_hub + a.n_warp + ((int64_t)(b - a.hub_ctas - a.warp_ctas) * wpc + wid) * R + sub;
    const int64_t end = warp_rows ? (int64_t)a.n_hub + a.n_warp : (int64_t)a.n_rows;
    const bool valid = pos < end;
    const int j = valid ? __ldg(a.order + pos) : 0;
    uint32_t id[P];
    float g[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { g[p] = 0.f; id[p] = 0; }
    if (valid) {
        load_idx<P>(idx_row<PEER>(a, j), ll * P, id);
        const int first = warp_rows ? sub : 0, stride = warp_rows ? R : 1;
        for (int q = 0; q < a.n_terms; ++q) {
            const TermDev &t = a.t[q];
            float acc[P];
#pragma unroll
            for (int p = 0; p < P; ++p) acc[p] = 0.f;
            bwd_term<P>(t, __ldg(t.colptr + j) + first, __ldg(t.colptr + j + 1), stride, id, a.D,
                        acc, a.ng, ll * P, a.k);
            const float sj = __ldg(t.s + j);
#pragma unroll
            for (int p = 0; p < P; ++p) g[p] += sj * acc[p];
        }
    }
    if (warp_rows) {
        // butterfly over the R sub-warps (lanes with equal ll hold the same positions);
        // every lane ends with the identical, order-fixed total
        for (int off = L; off < 32; off <<= 1) {
#pragma unroll
            for (int p = 0; p < P; ++p) g[p] += __shfl_xor_sync(0xffffffffu, g[p], off);
        }
    }
    if (valid && a.root) {
#pragma unroll
        for (int p = 0; p < P; ++p) g[p] += __ldg(a.root + (int64_t)j * a.k + ll * P + p);
    }
    bwd_store<P, PEER>(a, valid && (!warp_rows || sub == 0), j, ll, id, g,
                 warp_rows ? sm + (size_t)wid * R * a.D : srow);
}

// ------------------------------------------------------------------ host helpers
int choose_P(int k, int D) {
    const int cands[3] = {4, 2, 1};
    for (int P : cands)
        if (k % P == 0 && k / P <= 32 && (32 / (k / P)) * D <= 1024) return P;
    for (int P : cands)
        if (k % P == 0 && k / P <= 32) return P;
    return -1;
}

}  // namespace

void ensure_smem(const void *fn, size_t bytes);

void launch_spmm_fwd(const RelDev &r, const float *hval, const uint8_t *hidx, int k, int dim,
                     float *z, cudaStream_t s, bool z_split, NgSched ng, const PeerSrc *peer) {
    if (r.n_dst <= 0) return;
    if (!peer && !ng.on && !r.ew && tspmm_supported(r.tiles, dim, k)) {     // tensor-core tiled path
        launch_tspmm_fwd(r, hval, hidx, k, dim, z, s, z_split);
        return;
    }
    const int P = choose_P(k, dim);
    DR_CHECK(P > 0, DR_ERR_BAD_K, "spmm_fwd: unsupported k");
    FwdArgs a{};
    a.order = r.fwd.order;
    a.L = k / P;
    const int R = 32 / a.L;
    a.n_hub = r.fwd.n_hub;
    a.n_warp = r.fwd.n_warp;
    a.n_rows = r.n_dst;
    a.rowptr = r.rowptr;
    a.col = r.col;
    a.ew = r.ew;
    a.c = r.c;
    a.hval = hval;
    a.hidx = hidx;
    a.k = k;
    a.D = dim;
    a.z = z;
    a.z_split = z_split ? 1 : 0;
    a.ng = ng;
    if (peer) a.peer = *peer;
    int wpc = (int)knobs().spmm_wpc;
    while (wpc > 1 && (size_t)wpc * R * dim * 4 > 96 * 1024) wpc >>= 1;
    const size_t smem = (size_t)wpc * R * dim * 4;
    a.hub_ctas = a.n_hub > 0 ? (a.n_hub < kHubCtas ? a.n_hub : kHubCtas) : 0;
    a.warp_ctas = (a.n_warp + wpc - 1) / wpc;
    const int64_t n_sub = (int64_t)r.n_dst - a.n_hub - a.n_warp;
    const int64_t sub_ctas = (n_sub + (int64_t)wpc * R - 1) / ((int64_t)wpc * R);
    const unsigned grid = (unsigned)(a.hub_ctas + a.warp_ctas + sub_ctas);
    if (grid == 0) return;
    ProfScope ps("spmm_fwd", s);
    const void *fn = peer ? (P == 4 ? (const void *)spmm_fwd_kernel<4, true>
                             : P == 2 ? (const void *)spmm_fwd_kernel<2, true>
                                      : (const void *)spmm_fwd_kernel<1, true>)
                          : (P == 4 ? (const void *)spmm_fwd_kernel<4>
                             : P == 2 ? (const void *)spmm_fwd_kernel<2>
                                      : (const void *)spmm_fwd_kernel<1>);
    ensure_smem(fn, smem);
    void *args[] = {(void *)&a};
    DR_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(wpc * 32), args, smem, s));
    note_launch("spmm_fwd");
}

// Backward lane mapping: two CBSR positions per lane (P = 2, L = k/2 lanes per
// row): the sampled gathers of one warp instruction then touch fewer neighbour
// rows of dZ (fewer distinct cache lines per request) than with P = 4, while
// keeping two independent loads per lane; measured best at C2 (k=8) and C4
// (k=16) against P = 1 and 4 (profiles/r01/ab_bwdP.txt). Row sums stay in registers.
static int choose_P_bwd(int k) {
    const int p = (int)knobs().bwd_p;                // experiments only
    if (p > 0 && k % p == 0 && k / p <= 32) return p;
    if (k == 1) return 1;
    return k / 2 <= 32 ? 2 : k / 32;
}

void launch_spmm_bwd(const SrcSched &sched, int n_src, BwdTerm t0, BwdTerm t1, const float *root,
                     const uint8_t *hidx, int k, int dim, float *g_kept, float *dx,
                     bool accumulate, cudaStream_t s, NgSched ng, const PeerSrc *peer) {
    if (n_src <= 0) return;
    DR_CHECK(!peer || (!root && !dx && !accumulate && !ng.on), DR_ERR_INVALID_ARGUMENT,
             "spmm_bwd: the peer path writes g only");
    if (!peer && !ng.on && t0.rel && !t1.rel && !t0.rel->ewT && !accumulate && tspmm_supported(t0.rel->tilesT, dim, k) &&
        t0.rel->n_src == n_src) {                           // tensor-core tiled path
        launch_tspmm_bwd(*t0.rel, t0.dz, false, t0.apply_c, root, hidx, k, dim, g_kept, dx, s);
        return;
    }
    const int P = choose_P_bwd(k);
    DR_CHECK(P > 0, DR_ERR_BAD_K, "spmm_bwd: unsupported k");
    DR_CHECK(!ng.on || ((ng.kT || !t0.rel || t0.rel->nnz == 0) && !t1.rel), DR_ERR_INVALID_ARGUMENT,
             "spmm_bwd: NEXT-2 needs kT (relation with edges), one term");
    BwdArgs a{};
    a.order = sched.order;
    a.L = k / P;
    const int R = 32 / a.L;
    a.n_hub = sched.n_hub;
    a.n_warp = sched.n_warp;
    a.n_rows = n_src;
    BwdTerm terms[2] = {t0, t1};
    a.n_terms = 0;
    for (int q = 0; q < 2; ++q) {
        if (!terms[q].rel) continue;
        const RelDev &r = *terms[q].rel;
        TermDev &t = a.t[a.n_terms++];
        t.colptr = r.colptr;
        t.row = r.row;
        t.ewT = r.ewT;
        t.s = r.s;
        t.c = terms[q].apply_c ? r.c : nullptr;
        t.dz = terms[q].dz;
    }
    a.root = root;
    a.hidx = hidx;
    a.k = k;
    a.D = dim;
    a.g_kept = g_kept;
    a.dx = dx;
    a.accumulate = accumulate ? 1 : 0;
    a.ng = ng;
    if (peer) a.peer = *peer;
    int wpc = (int)knobs().spmm_wpc;
    while (wpc > 1 && (size_t)wpc * R * dim * 4 > 96 * 1024) wpc >>= 1;
    size_t smem = (size_t)wpc * R * dim * 4;
    const size_t hub_need = ((size_t)wpc * R + 1) * k * 4;    // partials + final row
    if (hub_need > smem) smem = hub_need;
    a.hub_ctas = a.n_hub > 0 ? (a.n_hub < kHubCtas ? a.n_hub : kHubCtas) : 0;
    a.warp_ctas = (a.n_warp + wpc - 1) / wpc;
    const int64_t n_sub = (int64_t)n_src - a.n_hub - a.n_warp;
    const int64_t sub_ctas = (n_sub + (int64_t)wpc * R - 1) / ((int64_t)wpc * R);
    const unsigned grid = (unsigned)(a.hub_ctas + a.warp_ctas + sub_ctas);
    if (grid == 0) return;
    ProfScope ps("spmm_bwd", s);
    const void *fn = peer ? (P == 4 ? (const void *)spmm_bwd_kernel<4, true>
                             : P == 2 ? (const void *)spmm_bwd_kernel<2, true>
                                      : (const void *)spmm_bwd_kernel<1, true>)
                          : (P == 4 ? (const void *)spmm_bwd_kernel<4>
                             : P == 2 ? (const void *)spmm_bwd_kernel<2>
                                      : (const void *)spmm_bwd_kernel<1>);
    ensure_smem(fn, smem);
    void *args[] = {(void *)&a};
    DR_CUDA(cudaLaunchKernel(fn, dim3(grid), dim3(wpc * 32), args, smem, s));
    note_launch("spmm_bwd");
}

// f4 inbox sum: out[e] = sum over p = 0 .. world-1 of inbox[p][e], fixed order
__global__ void inbox_sum_kernel(const float *__restrict__ inbox, int world, int64_t n,
                                 float *__restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        float acc = 0.f;
        for (int p = 0; p < world; ++p) acc += __ldg(inbox + (int64_t)p * n + e);
        out[e] = acc;
    }
}

// f4 sharded layer: g[e] = root[e] (optional) + sum over slots s of inbox[s][e], fixed order
__global__ void inbox_root_kernel(const float *__restrict__ inbox, int nslots, int64_t slot_stride,
                                  const float *root, int64_t n, float *out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        float acc = root ? root[e] : 0.f;          // (out may alias root: same element)
        for (int q = 0; q < nslots; ++q) acc += __ldg(inbox + (int64_t)q * slot_stride + e);
        out[e] = acc;
    }
}

// one warp per row: zero the row, then drop the k values at their columns
__global__ void cbsr_scatter_kernel(const float *__restrict__ g, const uint8_t *__restrict__ idx,
                                    int64_t n, int k, int dim, float *__restrict__ dx) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        float *row = dx + r * dim;
        for (int c = lane; c < dim; c += 32) row[c] = 0.f;
        __syncwarp();
        for (int t = lane; t < k; t += 32) row[__ldg(idx + r * k + t)] = __ldg(g + r * k + t);
        __syncwarp();
    }
}

void launch_inbox_sum(const float *inbox, int world, int64_t n, float *out, cudaStream_t s) {
    if (n <= 0) return;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    inbox_sum_kernel<<<(unsigned)blocks, 256, 0, s>>>(inbox, world, n, out);
    note_launch("inbox_sum");
}

void launch_inbox_root(const float *inbox, int nslots, int64_t slot_stride, const float *root,
                       int64_t n, float *out, cudaStream_t s) {
    if (n <= 0) return;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    inbox_root_kernel<<<(unsigned)blocks, 256, 0, s>>>(inbox, nslots, slot_stride, root, n, out);
    note_launch("inbox_root");
}

void launch_cbsr_scatter(const float *g, const uint8_t *idx, int64_t n, int k, int dim, float *dx,
                         cudaStream_t s) {
    if (n <= 0) return;
    ProfScope ps("cbsr_scatter", s);
    int64_t blocks = (n + 7) / 8;
    if (blocks > 148 * 8) blocks = 148 * 8;
    cbsr_scatter_kernel<<<(unsigned)blocks, 256, 0, s>>>(g, idx, n, k, dim, dx);
    note_launch("cbsr_scatter");
}

__global__ void ng_edge_k_kernel(const int32_t *__restrict__ row, const int32_t *__restrict__ rowptr,
                                 int64_t nnz, NgSched ng, uint8_t *__restrict__ kT) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nnz;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = __ldg(row + e);
        const int deg = __ldg(rowptr + i + 1) - __ldg(rowptr + i);
        kT[e] = (uint8_t)(deg <= ng.thr0 ? ng.kb0 : deg <= ng.thr1 ? ng.kb1 : ng.kb2);
    }
}

void launch_ng_edge_k(const RelDev &r, const NgSched &ng, uint8_t *kT, cudaStream_t s) {
    if (r.nnz <= 0) return;
    ProfScope ps("ng_edge_k", s);
    int64_t blocks = (r.nnz + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    ng_edge_k_kernel<<<(unsigned)blocks, 256, 0, s>>>(r.row, r.rowptr, r.nnz, ng, kT);
    note_launch("ng_edge_k");
}

}  // namespace dr

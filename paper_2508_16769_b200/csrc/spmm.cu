// spmm.cu — DR-SpMM forward (Alg. 1, Eq. 5-7) and SSpMM backward (Alg. 2,
// Eq. 10-11) over CBSR operands, for sm_100a.
//
// Mapping (Alg. 1 stage 2, "partition into ceil(32/K) parts"):
// a warp is split into R = 32/L sub-warps of L = k/P lanes; each sub-warp owns
// one row, each lane owns P of the row's k CBSR pairs (P = 4 -> one 128-bit
// value load + one 32-bit index load per neighbour). Rows are processed in the
// graph's degree-descending order so the R rows of a warp have similar work and
// the heaviest rows start first. Rows with more than kHubDeg neighbours
// ("evil rows", §2.3) are handled by one CTA each: its sub-warps
// split the neighbour list into contiguous chunks and their partials are
// summed in a fixed order. Every output element therefore has one owner and a
// fixed summation order: no atomics anywhere (reading Q23), results are
// bit-reproducible run to run.
//
// Forward: the sub-warp accumulates densify(H_j) for its row into a D-float
// shared-memory row (the k indices of one CBSR row are distinct, so the lanes
// of a sub-warp never collide), then writes c_i * acc with 128-bit stores.
// Backward: the sub-warp of source row j keeps its k CBSR indices in registers
// and pulls dz[i, idx_j,t] over j's CSC list (sampled gather), accumulating in
// registers; the D-ReLU mask gradient is the scatter of those k values.
#include "dr_internal.h"

namespace dr {
namespace {

constexpr int kU = 4;           // neighbours in flight per lane (memory-level parallelism)

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

// Accumulate the neighbours [e0, e1) of one row into `acc` (shared, D floats).
template <int P>
__device__ __forceinline__ void fwd_accumulate(int e0, int e1, const int32_t *__restrict__ col,
                                               const float *__restrict__ ew,
                                               const float *__restrict__ hval,
                                               const uint8_t *__restrict__ hidx, int k, int ll,
                                               float *acc) {
    for (int e = e0; e < e1; e += kU) {
        int j[kU];
        float w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const bool ok = e + u < e1;
            j[u] = ok ? __ldg(col + e + u) : -1;
            w[u] = (ok && ew) ? __ldg(ew + e + u) : 1.0f;
        }
        Pairs<P> pr[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (j[u] >= 0) load_pairs<P>(hval, hidx, (int64_t)j[u] * k + ll * P, pr[u]);
#pragma unroll
        for (int u = 0; u < kU; ++u)
            if (j[u] >= 0) {
#pragma unroll
                for (int p = 0; p < P; ++p) acc[pr[u].id[p]] += w[u] * pr[u].v[p];
            }
    }
}

struct FwdArgs {
    const int32_t *order;
    int32_t n_hub, n_rows;       // order[0..n_hub) hubs, order[n_hub..n_rows) warp rows
    int32_t hub_ctas;            // blocks [0, hub_ctas) serve hubs
    const int32_t *rowptr, *col;
    const float *ew, *c;
    const float *hval;
    const uint8_t *hidx;
    int k, D, L;
    float *z;
};

template <int P>
__global__ void __launch_bounds__(256) spmm_fwd_kernel(FwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int L = a.L, R = 32 / L, sub = lane / L, ll = lane % L, D = a.D, D4 = D >> 2;
    float *acc = sm + (size_t)(wid * R + sub) * D;
    float4 *acc4 = reinterpret_cast<float4 *>(acc);

    if ((int)blockIdx.x < a.hub_ctas) {
        // ---- CTA per hub row: S sub-warps split the neighbour list, fixed-order reduce
        const int S = wpc * R, sidx = wid * R + sub;
        for (int h = blockIdx.x; h < a.n_hub; h += a.hub_ctas) {
            const int row = __ldg(a.order + h);
            const int e0 = __ldg(a.rowptr + row), e1 = __ldg(a.rowptr + row + 1);
            for (int c4 = ll; c4 < D4; c4 += L) acc4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncwarp();
            const int chunk = (e1 - e0 + S - 1) / S;
            const int b0 = min(e1, e0 + sidx * chunk), b1 = min(e1, b0 + chunk);
            fwd_accumulate<P>(b0, b1, a.col, a.ew, a.hval, a.hidx, a.k, ll, acc);
            __syncthreads();
            const float cr = __ldg(a.c + row);
            for (int cc = threadIdx.x; cc < D; cc += blockDim.x) {
                float sacc = 0.f;
                for (int q = 0; q < S; ++q) sacc += sm[(size_t)q * D + cc];
                a.z[(int64_t)row * D + cc] = cr * sacc;
            }
            __syncthreads();
        }
        return;
    }
    // ---- sub-warp per row
    const int64_t gw = (int64_t)(blockIdx.x - a.hub_ctas) * wpc + wid;
    const int pos = a.n_hub + (int)(gw * R) + sub;
    const bool valid = pos < a.n_rows;
    const int row = valid ? __ldg(a.order + pos) : 0;
    for (int c4 = ll; c4 < D4; c4 += L) acc4[c4] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    if (valid)
        fwd_accumulate<P>(__ldg(a.rowptr + row), __ldg(a.rowptr + row + 1), a.col, a.ew, a.hval,
                          a.hidx, a.k, ll, acc);
    __syncwarp();
    if (valid) {
        const float cr = __ldg(a.c + row);
        float4 *zr = reinterpret_cast<float4 *>(a.z + (int64_t)row * D);
        for (int c4 = ll; c4 < D4; c4 += L) {
            float4 v = acc4[c4];
            __stcs(zr + c4, make_float4(cr * v.x, cr * v.y, cr * v.z, cr * v.w));
        }
    }
}

// ------------------------------------------------------------------ backward
struct TermDev {
    const int32_t *colptr, *row;
    const float *ewT, *s, *c;    // c != nullptr: apply c_i per edge
    const float *dz;
};

struct BwdArgs {
    const int32_t *order;
    int32_t n_hub, n_rows, hub_ctas;
    TermDev t[2];
    int n_terms;
    const float *root;
    const uint8_t *hidx;
    int k, D, L;
    float *g_kept, *dx;
    int accumulate;
};

template <int P>
__device__ __forceinline__ void bwd_term(const TermDev &t, int e0, int e1, const uint32_t *id,
                                         int D, float *a) {
    for (int e = e0; e < e1; e += kU) {
        int i[kU];
        float w[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const bool ok = e + u < e1;
            i[u] = ok ? __ldg(t.row + e + u) : -1;
            w[u] = (ok && t.ewT) ? __ldg(t.ewT + e + u) : 1.0f;
        }
        float v[kU][P];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (i[u] >= 0) {
                const float *dzr = t.dz + (int64_t)i[u] * D;
#pragma unroll
                for (int p = 0; p < P; ++p) v[u][p] = __ldg(dzr + id[p]);
                if (t.c) w[u] *= __ldg(t.c + i[u]);
            }
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

// Write the P values of lane ll for source row j (g_kept and/or dense dx via
// the sub-warp's shared staging row `srow`). Must be reached by the whole warp.
template <int P>
__device__ __forceinline__ void bwd_store(const BwdArgs &a, bool valid, int j, int ll,
                                          const uint32_t *id, const float *g, float *srow) {
    const int D = a.D, D4 = D >> 2, L = a.L;
    if (valid && a.g_kept) {
        float *gk = a.g_kept + (int64_t)j * a.k + ll * P;
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

template <int P>
__global__ void __launch_bounds__(256) spmm_bwd_kernel(BwdArgs a) {
    extern __shared__ __align__(16) float sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int L = a.L, R = 32 / L, sub = lane / L, ll = lane % L;
    float *srow = sm + (size_t)(wid * R + sub) * a.D;

    if ((int)blockIdx.x < a.hub_ctas) {
        // ---- CTA per hub source row: partials over contiguous chunks, fixed-order sum
        const int S = wpc * R, sidx = wid * R + sub;
        float *part = sm;                            // [S][k] partials (reuses staging area)
        for (int h = blockIdx.x; h < a.n_hub; h += a.hub_ctas) {
            const int j = __ldg(a.order + h);
            uint32_t id[P];
            load_idx<P>(a.hidx, (int64_t)j * a.k + ll * P, id);
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
                bwd_term<P>(t, b0, b1, id, a.D, acc);
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
                float sacc = 0.f;
                for (int q = 0; q < S; ++q) sacc += part[(size_t)q * a.k + t];
                if (a.root) sacc += __ldg(a.root + (int64_t)j * a.k + t);
                part[(size_t)S * a.k + t] = sacc;    // final values after the partials
            }
            __syncthreads();
            if (wid == 0 && sub == 0) {              // sub-warp 0 stores the row
                float gf[P];
#pragma unroll
                for (int p = 0; p < P; ++p) gf[p] = part[(size_t)S * a.k + ll * P + p];
                if (a.g_kept) {
                    float *gk = a.g_kept + (int64_t)j * a.k + ll * P;
#pragma unroll
                    for (int p = 0; p < P; ++p) gk[p] = a.accumulate ? gk[p] + gf[p] : gf[p];
                }
                if (a.dx) {
                    float *dr = a.dx + (int64_t)j * a.D;
                    if (!a.accumulate)
                        for (int cc = ll; cc < a.D; cc += L) dr[cc] = 0.f;
                    __syncwarp((1u << L) - 1u);
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
    // ---- sub-warp per source row
    const int64_t gw = (int64_t)(blockIdx.x - a.hub_ctas) * wpc + wid;
    const int pos = a.n_hub + (int)(gw * R) + sub;
    const bool valid = pos < a.n_rows;
    const int j = valid ? __ldg(a.order + pos) : 0;
    uint32_t id[P];
    float g[P];
#pragma unroll
    for (int p = 0; p < P; ++p) { g[p] = 0.f; id[p] = 0; }
    if (valid) {
        load_idx<P>(a.hidx, (int64_t)j * a.k + ll * P, id);
        for (int q = 0; q < a.n_terms; ++q) {
            const TermDev &t = a.t[q];
            float acc[P];
#pragma unroll
            for (int p = 0; p < P; ++p) acc[p] = 0.f;
            bwd_term<P>(t, __ldg(t.colptr + j), __ldg(t.colptr + j + 1), id, a.D, acc);
            const float sj = __ldg(t.s + j);
#pragma unroll
            for (int p = 0; p < P; ++p) g[p] += sj * acc[p];
        }
        if (a.root) {
#pragma unroll
            for (int p = 0; p < P; ++p) g[p] += __ldg(a.root + (int64_t)j * a.k + ll * P + p);
        }
    }
    bwd_store<P>(a, valid, j, ll, id, g, srow);
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

template <typename K>
void set_smem_attr(K kernel, size_t bytes) {
    static thread_local size_t done = 0;
    (void)done;
    if (bytes > 48 * 1024)
        DR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)bytes));
}

}  // namespace

void launch_spmm_fwd(const RelDev &r, const float *hval, const uint8_t *hidx, int k, int dim,
                     float *z, cudaStream_t s) {
    if (r.n_dst <= 0) return;
    const int P = choose_P(k, dim);
    DR_CHECK(P > 0, DR_ERR_BAD_K, "spmm_fwd: unsupported k");
    FwdArgs a{};
    a.order = r.order;
    a.n_hub = r.n_hub;
    a.n_rows = r.n_dst;
    a.rowptr = r.rowptr;
    a.col = r.col;
    a.ew = r.ew;
    a.c = r.c;
    a.hval = hval;
    a.hidx = hidx;
    a.k = k;
    a.D = dim;
    a.L = k / P;
    a.z = z;
    const int R = 32 / a.L;
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * R * dim * 4 > 96 * 1024) wpc >>= 1;
    const size_t smem = (size_t)wpc * R * dim * 4;
    a.hub_ctas = r.n_hub > 0 ? (r.n_hub < 296 ? r.n_hub : 296) : 0;
    const int64_t rows = (int64_t)r.n_dst - r.n_hub;
    const int64_t warp_ctas = (rows + (int64_t)wpc * R - 1) / ((int64_t)wpc * R);
    const unsigned grid = (unsigned)(a.hub_ctas + warp_ctas);
    if (grid == 0) return;
    ProfScope ps("spmm_fwd", s);
    if (P == 4) {
        set_smem_attr(spmm_fwd_kernel<4>, smem);
        spmm_fwd_kernel<4><<<grid, wpc * 32, smem, s>>>(a);
    } else if (P == 2) {
        set_smem_attr(spmm_fwd_kernel<2>, smem);
        spmm_fwd_kernel<2><<<grid, wpc * 32, smem, s>>>(a);
    } else {
        set_smem_attr(spmm_fwd_kernel<1>, smem);
        spmm_fwd_kernel<1><<<grid, wpc * 32, smem, s>>>(a);
    }
    note_launch("spmm_fwd");
}

void launch_spmm_bwd(const SrcSched &sched, int n_src, BwdTerm t0, BwdTerm t1, const float *root,
                     const uint8_t *hidx, int k, int dim, float *g_kept, float *dx,
                     bool accumulate, cudaStream_t s) {
    if (n_src <= 0) return;
    const int P = choose_P(k, dim);
    DR_CHECK(P > 0, DR_ERR_BAD_K, "spmm_bwd: unsupported k");
    BwdArgs a{};
    a.order = sched.order;
    a.n_hub = sched.n_hub;
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
    a.L = k / P;
    a.g_kept = g_kept;
    a.dx = dx;
    a.accumulate = accumulate ? 1 : 0;
    const int R = 32 / a.L;
    int wpc = 8;
    while (wpc > 1 && (size_t)wpc * R * dim * 4 > 96 * 1024) wpc >>= 1;
    size_t smem = (size_t)wpc * R * dim * 4;
    const size_t hub_need = ((size_t)wpc * R + 1) * k * 4;    // partials + final row
    if (hub_need > smem) smem = hub_need;
    a.hub_ctas = sched.n_hub > 0 ? (sched.n_hub < 296 ? sched.n_hub : 296) : 0;
    const int64_t rows = (int64_t)n_src - sched.n_hub;
    const int64_t warp_ctas = (rows + (int64_t)wpc * R - 1) / ((int64_t)wpc * R);
    const unsigned grid = (unsigned)(a.hub_ctas + warp_ctas);
    if (grid == 0) return;
    ProfScope ps("spmm_bwd", s);
    if (P == 4) {
        set_smem_attr(spmm_bwd_kernel<4>, smem);
        spmm_bwd_kernel<4><<<grid, wpc * 32, smem, s>>>(a);
    } else if (P == 2) {
        set_smem_attr(spmm_bwd_kernel<2>, smem);
        spmm_bwd_kernel<2><<<grid, wpc * 32, smem, s>>>(a);
    } else {
        set_smem_attr(spmm_bwd_kernel<1>, smem);
        spmm_bwd_kernel<1><<<grid, wpc * 32, smem, s>>>(a);
    }
    note_launch("spmm_bwd");
}

}  // namespace dr

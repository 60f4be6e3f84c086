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
#include "drelu_net.cuh"

namespace dr {
namespace {

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
__device__ __forceinline__ void load_row(const float *__restrict__ xr, int dim, bool vec, int lane,
                                         float (&v)[V]) {
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
}

// RW rows per warp, searched together (independent reductions interleave, so
// their latencies overlap); the next RW rows are loaded before the current ones
// are processed.
template <int V, int RW>
__global__ void __launch_bounds__(256) drelu_kernel(const float *__restrict__ x, int64_t n,
                                                    int dim, int64_t ldx, int k, bool vec,
                                                    float *__restrict__ val,
                                                    uint8_t *__restrict__ idx) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    float nv[RW][V];
    int64_t r0 = warp * RW;
#pragma unroll
    for (int i = 0; i < RW; ++i)
        if (r0 + i < n) load_row<V>(x + (r0 + i) * ldx, dim, vec, lane, nv[i]);
    for (; r0 < n; r0 += nwarps * RW) {
        float v[RW][V];
        uint32_t key[RW][V];
#pragma unroll
        for (int i = 0; i < RW; ++i)
#pragma unroll
            for (int j = 0; j < V; ++j) v[i][j] = nv[i][j];
        const int64_t rn = r0 + nwarps * RW;
#pragma unroll
        for (int i = 0; i < RW; ++i)
            if (rn + i < n) load_row<V>(x + (rn + i) * ldx, dim, vec, lane, nv[i]);
#pragma unroll
        for (int i = 0; i < RW; ++i)
#pragma unroll
            for (int j = 0; j < V; ++j)
                key[i][j] = (lane * V + j < dim && r0 + i < n) ? order_key(v[i][j]) : 0u;

        // per row: largest T with #{key >= T} >= k (the k-th largest key), MSB first,
        // a row stops once a probe selects exactly k
        uint32_t T[RW];
        bool exact[RW], done[RW];
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            T[i] = 0;
            exact[i] = false;
            done[i] = r0 + i >= n;
        }
        for (int b = 31; b >= 0; --b) {
            bool all = true;
#pragma unroll
            for (int i = 0; i < RW; ++i) all = all && done[i];
            if (all) break;
            int cnt[RW];
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const uint32_t cand = T[i] | (1u << b);
                int c = 0;
#pragma unroll
                for (int j = 0; j < V; ++j) c += key[i][j] >= cand;
                cnt[i] = __reduce_add_sync(0xffffffffu, c);
            }
#pragma unroll
            for (int i = 0; i < RW; ++i)
                if (!done[i] && cnt[i] >= k) {
                    T[i] |= 1u << b;
                    if (cnt[i] == k) exact[i] = done[i] = true;
                }
        }
#pragma unroll
        for (int i = 0; i < RW; ++i) {
            const int64_t r = r0 + i;
            if (r >= n) break;
            bool sel[V];
            if (exact[i]) {
#pragma unroll
                for (int j = 0; j < V; ++j) sel[j] = key[i][j] >= T[i];
            } else {
                int gt = 0, eq = 0;
#pragma unroll
                for (int j = 0; j < V; ++j) { gt += key[i][j] > T[i]; eq += key[i][j] == T[i]; }
                int need = k - __reduce_add_sync(0xffffffffu, gt);
                int rank = warp_excl_scan(eq, lane);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    bool tie = key[i][j] == T[i];
                    sel[j] = key[i][j] > T[i] || (tie && rank < need);
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
                    vo[pos] = v[i][j];
                    io[pos] = (uint8_t)(lane * V + j);
                    ++pos;
                }
            }
        }
    }
}

// Successive-max selection (k <= 32): each lane sorts its V keys descending
// (ties: lower column first) once; then k rounds pick the warp-wide largest
// head (redux.max), the lowest lane holding it takes it (ties -> lowest column,
// since lane l holds columns [lV, lV+V)) and pops its head. That is exactly the
// top-k under (value desc, column asc) of the binary search above. The rounds
// run on keys carrying (31 - lane) in their low 5 bits (one redux, no ballot,
// per round), with an exactness check and a full-key rerun for the rare rows it
// flags; the kernel is issue-bound, so instructions per round are what count.
template <int V>
__device__ __forceinline__ int pick_i(const int (&a)[V], int q) {
    int r = a[0];
#pragma unroll
    for (int i = 1; i < V; ++i) r = q == i ? a[i] : r;
    return r;
}
template <int V>
__device__ __forceinline__ float pick_f(const float (&a)[V], int q) {
    float r = a[0];
#pragma unroll
    for (int i = 1; i < V; ++i) r = q == i ? a[i] : r;
    return r;
}

// SORTED: rows stored in extraction order = value descending, ties lower column
// first (the value-sorted CBSR of NEXT-2, reading Q26): the winner of round t
// writes its element at position t; no column-order compaction. Rounds whose heads
// from different lanes tie on the truncated key are ordered by lane, not value, so
// SORTED also sends those rows to the full-key rerun.
template <int V, bool SORTED>
__global__ void __launch_bounds__(256) drelu_extract_kernel(const float *__restrict__ x, int64_t n,
                                                            int dim, int64_t ldx, int k, bool vec,
                                                            float *__restrict__ val,
                                                            uint8_t *__restrict__ idx) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t ltmask;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltmask));
    float nv[V];
    if (warp < n) load_row<V>(x + warp * ldx, dim, vec, lane, nv);
    for (int64_t r = warp; r < n; r += nwarps) {
        float v[V];
#pragma unroll
        for (int j = 0; j < V; ++j) v[j] = nv[j];
        if (r + nwarps < n) load_row<V>(x + (r + nwarps) * ldx, dim, vec, lane, nv);
        uint32_t sk[V];
        int sp[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            sk[j] = (lane * V + j < dim) ? order_key(v[j]) : 0u;
            sp[j] = j;
        }
        // odd-even transposition sort, descending by key; it only swaps on a strict
        // '<', so it is stable: equal keys keep ascending slot (column) order
#pragma unroll
        for (int round = 0; round < V; ++round) {
#pragma unroll
            for (int a = round & 1; a + 1 < V; a += 2) {
                const bool sw = sk[a] < sk[a + 1];
                const uint32_t k0 = sk[a], k1 = sk[a + 1];
                const int p0 = sp[a], p1 = sp[a + 1];
                sk[a] = sw ? k1 : k0;
                sk[a + 1] = sw ? k0 : k1;
                sp[a] = sw ? p1 : p0;
                sp[a + 1] = sw ? p0 : p1;
            }
        }
        // k rounds of successive-max on keys whose low 5 bits are replaced by
        // (31 - lane): one redux.max both finds the largest head and breaks ties to
        // the lowest lane, with no ballot. Truncation is monotone, so this is exact
        // unless an element left behind shares the truncated key of the last one
        // taken -- checked below; such (rare) rows rerun with full keys + ballot.
        // SORTED: the lane's q-th popped element went out in round t_q; the t_q are
        // packed 5 bits each into `pos` and the stores happen once, after the rounds.
        const uint32_t lanebits = 31u - (uint32_t)lane;
        uint32_t fk[V];
#pragma unroll
        for (int j = 0; j < V; ++j) fk[j] = sk[j] ? ((sk[j] & ~31u) | lanebits) : 0u;
        uint32_t m = 0, prev = 0;
        uint64_t tpos = 0;
        int popped = 0;
        bool amb = false;   // SORTED: two heads from different lanes shared a truncated key
        (void)prev;
        (void)tpos;
        (void)popped;
#pragma unroll 4
        for (int t = 0; t < k; ++t) {
            m = __reduce_max_sync(0xffffffffu, fk[0]);
            if constexpr (SORTED) {
                // the set is still exact, but their order was decided by lane, not value
                amb |= m != prev && ((m ^ prev) & ~31u) == 0u;
                prev = m;
            }
            if (fk[0] == m) {
                if constexpr (SORTED) {
                    tpos |= (uint64_t)t << (5 * popped);
                    ++popped;
                }
#pragma unroll
                for (int j = 0; j + 1 < V; ++j) fk[j] = fk[j + 1];
                fk[V - 1] = 0u;
            }
        }
        // pops = zeros shifted in = zeros now - zero (padding) keys the lane had
        int taken = 0;
#pragma unroll
        for (int j = 0; j < V; ++j) taken += (fk[j] == 0u ? 1 : 0) - (sk[j] == 0u ? 1 : 0);
        const bool unsafe =
            __any_sync(0xffffffffu, fk[0] != 0u && (fk[0] & ~31u) == (m & ~31u)) || amb;
        if (unsafe) {
            taken = 0;
            tpos = 0;
#pragma unroll 4
            for (int t = 0; t < k; ++t) {
                const uint32_t mm = __reduce_max_sync(0xffffffffu, sk[0]);
                const bool mine = sk[0] == mm;
                const uint32_t b = __ballot_sync(0xffffffffu, mine);
                if (mine && (b & ltmask) == 0u) {
                    if constexpr (SORTED) tpos |= (uint64_t)t << (5 * taken);
                    ++taken;
#pragma unroll
                    for (int j = 0; j + 1 < V; ++j) sk[j] = sk[j + 1];
                    sk[V - 1] = 0u;
                }
            }
        }
        float *vo = val + r * k;
        uint8_t *io = idx + r * k;
        if constexpr (SORTED) {
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (q < taken) {
                    const int t = (int)((tpos >> (5 * q)) & 31u);
                    const int slot = sp[q];
                    vo[t] = pick_f<V>(v, slot);
                    io[t] = (uint8_t)(lane * V + slot);
                }
            continue;
        }
        uint32_t selm = 0;
#pragma unroll
        for (int q = 0; q < V; ++q)
            if (q < taken) selm |= 1u << sp[q];
        int pos = warp_excl_scan(__popc(selm), lane);
#pragma unroll
        for (int j = 0; j < V; ++j) {
            if (selm & (1u << j)) {
                vo[pos] = v[j];
                io[pos] = (uint8_t)(lane * V + j);
                ++pos;
            }
        }
    }
}

// ---------------------------------------------------------------- thread-per-row networks
// One THREAD per row (D in {32, 64, 128}, K a power of two <= min(32, D/2)): a
// warp stages 32 rows in shared memory with coalesced 128-bit loads, then every
// lane selects its own row's top K with no cross-lane traffic. Each element
// becomes a unique 32-bit composite: its order key with the low CB = log2(D)
// bits replaced by (D - 1 - column), so composites order by (value desc, column
// asc) exactly except between elements sharing the truncated key. Top K of the D
// composites: bitonic-sort groups of K, then a tree of "merge, keep the larger
// K" steps (elementwise max against the reversed partner, bitonic merge). Each
// merge discards K composites; the largest discarded one is the (K+1)-th overall,
// so the selection is exact unless it shares the K-th's truncated key -- those
// (rare) rows, and rows with such ties, rerun an exact resolution of the tied elements (tpr_rerun) from
// shared memory. The K kept columns are sorted ascending (CBSR order) or
// left in value order (SORTED), and their values read back from shared memory.
// Instructions per row ~ D log^2 K compare-exchanges instead of K warp-wide
// reduction rounds (the standalone D-ReLU was issue-bound, profiles/r01).
template <int D, int K, bool SORTED, bool STREAM>
__global__ void __launch_bounds__(128, D == 128 ? 3 : 6) drelu_tpr_kernel(const float *__restrict__ x, int64_t n,
                                                        int64_t ldx, float *__restrict__ val,
                                                        uint8_t *__restrict__ idx) {
    constexpr int P = D + 4;                      // padded row: conflict-free 128-bit reads
    constexpr int Q = D / 4;                      // float4 per row
    extern __shared__ __align__(16) float tpr_sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float *xs = tpr_sm + (size_t)wid * 32 * P;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
        // ---- stage 32 rows (coalesced: consecutive lanes read consecutive float4s);
        // batches of 16 independent loads per lane before their shared stores
        constexpr int NL = Q;                     // float4 loads per lane (32 rows x Q / 32)
        constexpr int NB = NL < 16 ? NL : 16;
#pragma unroll
        for (int b0 = 0; b0 < NL; b0 += NB) {
            float4 v[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int e = lane + 32 * (b0 + u), i = e / Q, c4 = e % Q;
                v[u] = r0 + i < n ? __ldg(reinterpret_cast<const float4 *>(x + (r0 + i) * ldx) + c4)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int e = lane + 32 * (b0 + u), i = e / Q, c4 = e % Q;
                *reinterpret_cast<float4 *>(xs + i * P + 4 * c4) = v[u];
            }
        }
        __syncwarp();
        const int64_t r = r0 + lane;
        tpr_select_row<D, K, SORTED, STREAM>(xs + lane * P, r < n, val + r * K, idx + r * K);
        __syncwarp();
    }
}

template <int D, int K, bool SORTED, bool STREAM>
void launch_tpr(const float *x, int64_t n, int64_t ldx, float *val, uint8_t *idx, cudaStream_t s) {
    const size_t smem = (size_t)4 * 32 * (D + 4) * sizeof(float);
    const void *fn = (const void *)drelu_tpr_kernel<D, K, SORTED, STREAM>;
    ensure_smem(fn, smem);
    // persistent: one wave of resident CTAs striding over 32-row groups (a partial
    // second wave would double the time of a one-group-per-warp launch)
    static int ps = 0;
    if (ps == 0) {
        DR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, (const void *)drelu_tpr_kernel<D, K, SORTED, STREAM>, 128, smem));
        if (ps < 1) ps = 1;
    }
    const int64_t groups = (n + 31) / 32;
    const int64_t cap = (int64_t)148 * ps;
    int64_t blocks = (groups + 3) / 4;
    if (blocks > cap) blocks = cap;
    drelu_tpr_kernel<D, K, SORTED, STREAM><<<(unsigned)blocks, 128, smem, s>>>(x, n, ldx, val, idx);
}

// Cooperative thread-per-row (ascending-column CBSR): T consecutive lanes share a
// row, each taking D/T consecutive columns of the staged row: a per-lane network
// (composites sorted in groups of K, merged keeping the larger K), then log2 T
// butterfly steps exchange the running top K with __shfl_xor and merge it (both
// partners end with the same K, and the largest discarded composite). Same
// composites and the same exact rerun as tpr_select_row, so the selection is
// identical; a thread holds D/T composites instead of D -- fewer registers, T
// times more threads per row, more warps resident for the latency-bound network.
template <int D, int K, int T>
__global__ void __launch_bounds__(128) drelu_tcoop_kernel(const float *__restrict__ x, int64_t n,
                                                          int64_t ldx, float *__restrict__ val,
                                                          uint8_t *__restrict__ idx, int roll) {
    constexpr int P = D + 4, Q = D / 4, RW = 32 / T, W = D / T;   // rows per warp, columns per lane
    constexpr int CB = D == 32 ? 5 : D == 64 ? 6 : 7;
    constexpr uint32_t CM = (1u << CB) - 1u;
    static_assert(W >= K && W % 4 == 0, "each lane needs >= K columns");
    extern __shared__ __align__(16) float tco_sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rl = lane / T, sl = lane % T;                        // row of the warp, slice
    // two staging buffers per warp: the next row group streams in (cp.async, no
    // registers) while this one is reduced
    float *xsb = tco_sm + (size_t)wid * 2 * RW * P;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    constexpr int NL = RW * Q / 32;                                // float4 copies per lane
    auto issue = [&](int64_t rb, float *dst) {
#pragma unroll
        for (int u = 0; u < NL; ++u) {
            const int e = lane + 32 * u, i = e / Q, c4 = e % Q;
            float *d = dst + i * P + 4 * c4;
            if (rb + i < n) {
                const float *src = x + (rb + i) * ldx + 4 * c4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(d)),
                             "l"(src)
                             : "memory");
            } else {
                *reinterpret_cast<float4 *>(d) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int buf = 0;
    if (gw * RW < n) issue(gw * RW, xsb);
    for (int64_t r0 = gw * RW; r0 < n; r0 += nw * RW) {
        float *xs = xsb + (size_t)buf * RW * P;
        const int64_t nx = r0 + nw * RW;
        if (nx < n) {
            issue(nx, xsb + (size_t)(buf ^ 1) * RW * P);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const int64_t r = r0 + rl;
        const float *xr = xs + rl * P;
        uint32_t w[W];
        uint32_t lost = 0;
        if (roll) {
            // the lane's W columns in rolled chunks of CK (tpr_top_stream's network)
            constexpr int CK = K < 8 ? 8 : K;
            static_assert(W % CK == 0, "chunking");
            uint32_t b[CK];
            tpr_keys<CK, CB>(xr, sl * W, b);
            bitonic_sort_desc<CK>(b);
#pragma unroll
            for (int t = 0; t < K; ++t) w[t] = b[t];
            if constexpr (CK > K) lost = b[K];
#pragma unroll 1
            for (int c0 = CK; c0 < W; c0 += CK) {
                tpr_keys<CK, CB>(xr, sl * W + c0, b);
                bitonic_sort_desc<CK>(b);
                if constexpr (CK > K) lost = max(lost, b[K]);
                lost = max(lost, merge_keep_desc<K>(w, b));
            }
        } else {
#pragma unroll
            for (int c4 = 0; c4 < W / 4; ++c4) {
                const uint32_t c = (uint32_t)(sl * W + 4 * c4);
                const float4 q = *reinterpret_cast<const float4 *>(xr + c);
                w[4 * c4 + 0] = (order_key(q.x) & ~CM) | (CM - (c + 0));
                w[4 * c4 + 1] = (order_key(q.y) & ~CM) | (CM - (c + 1));
                w[4 * c4 + 2] = (order_key(q.z) & ~CM) | (CM - (c + 2));
                w[4 * c4 + 3] = (order_key(q.w) & ~CM) | (CM - (c + 3));
            }
#pragma unroll
            for (int g = 0; g < W / K; ++g) bitonic_sort_desc<K>(w + g * K);
#pragma unroll
            for (int step = 1; step < W / K; step <<= 1)
#pragma unroll
                for (int g = 0; g + step < W / K; g += 2 * step)
                    lost = max(lost, merge_keep_desc<K>(w + g * K, w + (g + step) * K));
        }
        // butterfly over the T lanes of the row
#pragma unroll
        for (int m = 1; m < T; m <<= 1) {
            uint32_t b[K];
#pragma unroll
            for (int t = 0; t < K; ++t) b[t] = __shfl_xor_sync(0xffffffffu, w[t], m);
            lost = max(lost, __shfl_xor_sync(0xffffffffu, lost, m));
            lost = max(lost, merge_keep_desc<K>(w, b));
        }
        uint32_t col[K];
#pragma unroll
        for (int t = 0; t < K; ++t) col[t] = CM - (w[t] & CM);
        const bool valid = r < n;
        const bool rerun = (lost & ~CM) == (w[K - 1] & ~CM);
        if (valid && rerun) {
            // exact (rare): the tied elements at the threshold ranked by full key
            uint32_t sel[K];
            tpr_rerun<D, K, CB>(xr, w[K - 1] & ~CM, sel);
#pragma unroll
            for (int t = 0; t < K; ++t) col[t] = sel[K - 1 - t];   // descending, like below
        } else {
            bitonic_sort_desc<K>(col);
        }
        // lane sl of the row writes pairs [sl K / T, (sl + 1) K / T) (ascending columns)
        if (valid) {
            constexpr int KT = K / T > 0 ? K / T : 1;
            if (sl * KT < K) {
#pragma unroll
                for (int t = 0; t < KT; ++t) {
                    const int o = sl * KT + t;                      // output slot
                    uint32_t c = 0;
#pragma unroll
                    for (int u = 0; u < K; ++u)
                        if (u == K - 1 - o) c = col[u];
                    val[r * K + o] = xr[c];
                    idx[r * K + o] = (uint8_t)c;
                }
            }
        }
        __syncwarp();                      // every read of xs done before it is refilled
        buf ^= 1;
    }
}

template <int D, int K, int T>
void launch_tcoop(const float *x, int64_t n, int64_t ldx, float *val, uint8_t *idx, cudaStream_t s) {
    const size_t smem = (size_t)4 * 2 * (32 / T) * (D + 4) * sizeof(float);
    const void *fn = (const void *)drelu_tcoop_kernel<D, K, T>;
    ensure_smem(fn, smem);
    static int ps = 0;
    if (ps == 0) {
        DR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, fn, 128, smem));
        if (ps < 1) ps = 1;
    }
    const int64_t groups = (n + 32 / T - 1) / (32 / T);
    const int64_t cap = (int64_t)148 * ps;
    int64_t blocks = (groups + 3) / 4;
    if (blocks > cap) blocks = cap;
    // rolled per-lane network at D = 128 (C4 1M x 128, k = 16: 0.258 -> 0.242 ms;
    // 700k: 0.186 -> 0.180), unrolled at D = 64 (equal or faster); tpr_stream 0 / 2 force
    const int roll = D == 128 ? (knobs().tpr_stream != 0) : (knobs().tpr_stream == 2);
    drelu_tcoop_kernel<D, K, T><<<(unsigned)blocks, 128, smem, s>>>(x, n, ldx, val, idx, roll);
}

template <bool SORTED>
bool try_tpr(const float *x, int64_t n, int dim, int64_t ldx, int k, float *val, uint8_t *idx,
             cudaStream_t s) {
    if ((ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(x) % 16) != 0) return false;
    // cooperative rows: default (-2) two lanes per row at D = 64, k in {4, 8}
    // (100k x 64, k = 8: 0.0205 vs 0.0246 ms thread-per-row, 0.0307 warp-per-row)
    // and, with the rolled per-lane network, at D = 128, k in 4..16 (C4 1M x 128,
    // k = 16: 0.242 vs 0.248 ms rolled thread-per-row; 700k: 0.180 vs 0.191) --
    // profiles/r03/drelu_ab.json, drelu_ab_roll.json; 0 = off, 1 / 2 / 4 = forced (A/B)
    int T = (int)knobs().drelu_coop;
    if (T == -2) T = ((dim == 64 && (k == 4 || k == 8)) || (dim == 128 && k >= 4 && k <= 16)) ? 2 : 0;
    if (!SORTED && T > 0) {
#define DR_TCO(DD, KK, TT)                                                                  \
        if (dim == DD && k == KK && T == TT) {                                              \
            launch_tcoop<DD, KK, TT>(x, n, ldx, val, idx, s);                               \
            return true;                                                                    \
        }
        DR_TCO(128, 4, 1) DR_TCO(128, 8, 1) DR_TCO(128, 16, 1)
        DR_TCO(64, 4, 1) DR_TCO(64, 8, 1) DR_TCO(64, 16, 1)
        DR_TCO(128, 4, 2) DR_TCO(128, 8, 2) DR_TCO(128, 16, 2)
        DR_TCO(128, 4, 4) DR_TCO(128, 8, 4) DR_TCO(128, 16, 4)
        DR_TCO(64, 4, 2) DR_TCO(64, 8, 2) DR_TCO(64, 16, 2)
        DR_TCO(64, 4, 4) DR_TCO(64, 8, 4) DR_TCO(64, 16, 4)
#undef DR_TCO
    }
#define DR_TPR(DD, KK)                                                                      \
    if (dim == DD && k == KK) {                                                             \
        if (knobs().tpr_stream == 1 ? DD == 128 : knobs().tpr_stream == 2)                \
            launch_tpr<DD, KK, SORTED, true>(x, n, ldx, val, idx, s);                       \
        else launch_tpr<DD, KK, SORTED, false>(x, n, ldx, val, idx, s);                     \
        return true;                                                                        \
    }
    // measured (profiles/r02/drelu_ab.json, profiles/r03/drelu_ab.json): faster than
    // the warp-per-row kernels at D = 128 (C4: 0.47 -> 0.25 ms) and at D = 64 with
    // k >= 8 (100k x 64, k = 8: 0.031 -> 0.025 ms once the tied-threshold rerun
    // became cheap, tpr_rerun)
    DR_TPR(64, 8) DR_TPR(64, 16) DR_TPR(64, 32)
    DR_TPR(128, 4) DR_TPR(128, 8) DR_TPR(128, 16) DR_TPR(128, 32)
    if (knobs().drelu_tpr == 2) {                 // A/B: every supported shape
        DR_TPR(32, 2) DR_TPR(32, 4) DR_TPR(32, 8) DR_TPR(32, 16)
        DR_TPR(64, 2) DR_TPR(64, 4)
    }
#undef DR_TPR
    return false;
}

}  // namespace

void launch_drelu(const float *x, int64_t n, int dim, int64_t ldx, int k, float *val,
                  uint8_t *idx, cudaStream_t s, bool sorted) {
    if (n <= 0) return;
    ProfScope ps("drelu", s);
    const int threads = 256, rows_per_cta = threads / 32;
    int64_t blocks = (n + rows_per_cta - 1) / rows_per_cta;
    if (blocks > 148 * 8) blocks = 148 * 8;        // one wave: 8 x 256 threads per SM
    const int V = dim <= 32 ? 1 : dim <= 64 ? 2 : dim <= 128 ? 4 : 8;
    const bool vec = dim == 32 * V && (ldx % V) == 0 &&
                     (reinterpret_cast<uintptr_t>(x) % (4 * V)) == 0;
    DR_CHECK(!sorted || k <= 32, DR_ERR_BAD_K, "value-sorted D-ReLU needs k <= 32");
    const bool force_bs = knobs().drelu_bs == 1;   // A/B only: the binary search for every k
    // thread-per-row networks for the common widths (A/B: drelu_tpr=0 disables)
    if (knobs().drelu_tpr && !force_bs &&
        (sorted ? try_tpr<true>(x, n, dim, ldx, k, val, idx, s)
                : try_tpr<false>(x, n, dim, ldx, k, val, idx, s))) {
        note_launch("drelu");
        return;
    }
    if (k <= 32 && sorted) {
        if (V == 1)
            drelu_extract_kernel<1, true><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else if (V == 2)
            drelu_extract_kernel<2, true><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else if (V == 4)
            drelu_extract_kernel<4, true><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else
            drelu_extract_kernel<8, true><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    } else if (k <= 32 && 2 * k < dim && !force_bs) {
        // successive max: k rounds; for k >= dim / 2 the ~13-step binary search is
        // cheaper (measured: 300k x 64, k = 32: 0.104 vs 0.135 ms; k <= 16 and
        // D = 128, k = 16: extraction 1.2-1.8x faster -- profiles/r01/ab_drelu.txt)
        if (V == 1)
            drelu_extract_kernel<1, false><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else if (V == 2)
            drelu_extract_kernel<2, false><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else if (V == 4)
            drelu_extract_kernel<4, false><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
        else
            drelu_extract_kernel<8, false><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    } else if (V == 1)
        drelu_kernel<1, 1><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else if (V == 2)
        drelu_kernel<2, 1><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else if (V == 4)
        drelu_kernel<4, 1><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    else
        drelu_kernel<8, 1><<<(unsigned)blocks, threads, 0, s>>>(x, n, dim, ldx, k, vec, val, idx);
    note_launch("drelu");
}

}  // namespace dr

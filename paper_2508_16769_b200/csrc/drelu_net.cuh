// drelu_net.cuh — device helpers of the exact row-wise top-k (D-ReLU, Eq. 2-3,
// P:212-222) shared by the standalone kernels (drelu.cu) and the projection
// epilogue that emits the next layer's CBSR (tc2.cu, row a5).
//
// Order key: an order-preserving uint32 of x + 0.0f (-0.0 and +0.0 share a key
// and tie, reading Q5). Composite key: the order key with its CB low bits
// replaced by (CM - column), CM = 2^CB - 1, so composites are distinct within a
// row and compare as (value desc, column asc) -- exact unless two values agree
// in all but their CB low key bits (then the caller resolves the threshold
// exactly; see the "rerun" paths).
#pragma once
#include <cstdint>

namespace dr {

__device__ __forceinline__ uint32_t order_key(float x) {
    uint32_t u = __float_as_uint(x + 0.0f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// bitonic sort of w[0..K) descending
template <int K>
__device__ __forceinline__ void bitonic_sort_desc(uint32_t *w) {
#pragma unroll
    for (int k = 2; k <= K; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const uint32_t hi = max(w[i], w[l]), lo = min(w[i], w[l]);
                    const bool desc = (i & k) == 0;
                    w[i] = desc ? hi : lo;
                    w[l] = desc ? lo : hi;
                }
            }
}

// a, b sorted descending (K each): a <- the K largest of both, sorted descending;
// returns the largest discarded composite
template <int K>
__device__ __forceinline__ uint32_t merge_keep_desc(uint32_t *a, const uint32_t *b) {
    uint32_t lost = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const uint32_t x = a[i], y = b[K - 1 - i];
        a[i] = max(x, y);
        lost = max(lost, min(x, y));
    }
#pragma unroll
    for (int j = K >> 1; j > 0; j >>= 1)
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const int l = i ^ j;
            if (l > i) {
                const uint32_t hi = max(a[i], a[l]), lo = min(a[i], a[l]);
                a[i] = hi;
                a[l] = lo;
            }
        }
    return lost;
}

// composites of columns c0 .. c0 + C - 1 of a staged row (C a multiple of 4)
template <int C, int CB>
__device__ __forceinline__ void tpr_keys(const float *xr, int c0, uint32_t *w) {
    constexpr uint32_t CM = (1u << CB) - 1u;
#pragma unroll
    for (int c4 = 0; c4 < C / 4; ++c4) {
        const float4 v = *reinterpret_cast<const float4 *>(xr + c0 + 4 * c4);
        const uint32_t c = (uint32_t)(c0 + 4 * c4);
        w[4 * c4 + 0] = (order_key(v.x) & ~CM) | (CM - (c + 0));
        w[4 * c4 + 1] = (order_key(v.y) & ~CM) | (CM - (c + 1));
        w[4 * c4 + 2] = (order_key(v.z) & ~CM) | (CM - (c + 2));
        w[4 * c4 + 3] = (order_key(v.w) & ~CM) | (CM - (c + 3));
    }
}

// Streaming form of the same network: the row is consumed in chunks of
// CK = max(K, 8) columns by a rolled loop (one chunk's keys sorted, its best K
// merged into the running top K). The top-K set and the largest discarded
// composite equal the unrolled tree's (every composite outside the final top K
// is discarded by exactly one merge or chunk cut), so the selection is
// identical; the code is ~D/CK times smaller. Inside the projection epilogue
// (10 warp roles in one kernel) the unrolled network was instruction-fetch
// bound (stall_no_inst on the compare-exchanges, C5 profile).
template <int D, int K>
__device__ __forceinline__ uint32_t tpr_top_stream(const float *xr, uint32_t (&top)[K]) {
    constexpr int CB = D == 32 ? 5 : D == 64 ? 6 : 7;
    constexpr int CK = K < 8 ? (D < 8 ? D : 8) : K;
    static_assert(D % CK == 0 && CK % 4 == 0, "chunking");
    uint32_t lost = 0;
    {
        uint32_t b[CK];
        tpr_keys<CK, CB>(xr, 0, b);
        bitonic_sort_desc<CK>(b);
#pragma unroll
        for (int t = 0; t < K; ++t) top[t] = b[t];
        if constexpr (CK > K) lost = b[K];
    }
#pragma unroll 1
    for (int c0 = CK; c0 < D; c0 += CK) {
        uint32_t b[CK];
        tpr_keys<CK, CB>(xr, c0, b);
        bitonic_sort_desc<CK>(b);
        if constexpr (CK > K) lost = max(lost, b[K]);
        lost = max(lost, merge_keep_desc<K>(top, b));
    }
    return lost;
}

// Exact selection for a row whose truncated composites are ambiguous at the
// threshold. Tt = the K-th largest truncated key (that of the K-th composite):
// every element with a larger truncated key is in the top K, none with a smaller
// one is, and among the few whose truncated key equals Tt the best K - gt by
// (full key desc, column asc) are taken (each ranked by one pass over the row).
// Same set as ranking full keys; ~(2 + m) D shared reads for m <= 16 tied
// elements instead of the 33 D of a 32-step bisection (a rerun lane stalls its
// warp); rows with more ties take the bisection. sel = the K selected columns,
// ascending.
template <int D, int K, int CB>
__device__ __forceinline__ void tpr_rerun(const float *xr, uint32_t Tt, uint32_t (&sel)[K]) {
    constexpr uint32_t CM = (1u << CB) - 1u;
    int gt = 0, m = 0;
#pragma unroll 8
    for (int j = 0; j < D; ++j) {
        const uint32_t kt = order_key(xr[j]) & ~CM;
        gt += kt > Tt;
        m += kt == Tt;
    }
    int q = 0;
    if (m <= 16) {
        // few tied elements (the usual case): rank each by one pass over the row
        const int need = K - gt;
        for (int j = 0; j < D; ++j) {
            const uint32_t kj = order_key(xr[j]);
            bool take = (kj & ~CM) > Tt;
            if ((kj & ~CM) == Tt) {
                int r = 0;
#pragma unroll 8
                for (int i = 0; i < D; ++i) {
                    const uint32_t ki = order_key(xr[i]);
                    r += ((ki & ~CM) == Tt && (ki > kj || (ki == kj && i < j))) ? 1 : 0;
                }
                take = r < need;
            }
            if (take) {
#pragma unroll
                for (int t = 0; t < K; ++t)
                    if (t == q) sel[t] = (uint32_t)j;
                ++q;
            }
        }
        return;
    }
    // many ties (e.g. rows of equal or integer values): the K-th largest full key by
    // MSB-first bisection (33 D reads however many tie), then keys above it and the
    // lowest columns among keys equal to it
    uint32_t T = 0;
    for (int b = 31; b >= 0; --b) {
        const uint32_t cand = T | (1u << b);
        int cnt = 0;
        for (int j = 0; j < D; ++j) cnt += order_key(xr[j]) >= cand;
        if (cnt >= K) T = cand;
    }
    int gtf = 0;
    for (int j = 0; j < D; ++j) gtf += order_key(xr[j]) > T;
    int need = K - gtf;
    for (int j = 0; j < D; ++j) {
        const uint32_t kj = order_key(xr[j]);
        const bool take = kj > T || (kj == T && need > 0);
        if (take && kj == T) --need;
        if (take) {
#pragma unroll
            for (int t = 0; t < K; ++t)
                if (t == q) sel[t] = (uint32_t)j;
            ++q;
        }
    }
}

// Exact top-K of one row xr[0..D) held in shared memory (padded stride, 16-B
// aligned), thread-per-row (the thread's own row): composite keys = order key
// with the CB low bits replaced by (CM - column), bitonic-sorted in groups of K
// and merged keeping the larger K; exact unless the best discarded composite
// shares the K-th's truncated key -- then an exact rerun (tpr_rerun) resolves
// the tied elements from shared memory. Writes K pairs to vo / io: ascending columns (CBSR order,
// P:229), or value order (SORTED). valid == false: nothing is written.
// Used by the standalone D-ReLU (drelu.cu) and the projection epilogue that
// emits the next layer's CBSR (tc2.cu, row a5).
template <int D, int K, bool SORTED, bool STREAM = false>
__device__ __forceinline__ void tpr_select_row(const float *xr, bool valid, float *vo, uint8_t *io) {
    constexpr int CB = D == 32 ? 5 : D == 64 ? 6 : 7;
    constexpr uint32_t CM = (1u << CB) - 1u;
    constexpr int Q = D / 4;
    uint32_t w[STREAM ? K : D];
    uint32_t lost = 0;
    if constexpr (STREAM) {
        lost = tpr_top_stream<D, K>(xr, w);
    } else {
#pragma unroll
        for (int c4 = 0; c4 < Q; ++c4) {
            const float4 v = *reinterpret_cast<const float4 *>(xr + 4 * c4);
            w[4 * c4 + 0] = (order_key(v.x) & ~CM) | (CM - (uint32_t)(4 * c4 + 0));
            w[4 * c4 + 1] = (order_key(v.y) & ~CM) | (CM - (uint32_t)(4 * c4 + 1));
            w[4 * c4 + 2] = (order_key(v.z) & ~CM) | (CM - (uint32_t)(4 * c4 + 2));
            w[4 * c4 + 3] = (order_key(v.w) & ~CM) | (CM - (uint32_t)(4 * c4 + 3));
        }
#pragma unroll
        for (int g = 0; g < D / K; ++g) bitonic_sort_desc<K>(w + g * K);
#pragma unroll
        for (int step = 1; step < D / K; step <<= 1)
#pragma unroll
            for (int g = 0; g + step < D / K; g += 2 * step)
                lost = max(lost, merge_keep_desc<K>(w + g * K, w + (g + step) * K));
    }
    // w[0..K) = the top K composites, descending; exact unless the best loser
    // shares the K-th's truncated key
    uint32_t col[K];
#pragma unroll
    for (int t = 0; t < K; ++t) col[t] = CM - (w[t] & CM);
    bool rerun = (lost & ~CM) == (w[K - 1] & ~CM);
    if constexpr (SORTED) {    // value order inside the K: equal truncated keys are ordered by column
#pragma unroll
        for (int t = 0; t + 1 < K; ++t) rerun |= ((w[t] ^ w[t + 1]) & ~CM) == 0u;
    }
    if (valid && rerun) {
        // exact rerun (rare): the ambiguous elements at the threshold ranked by full key
        uint32_t sel[K];
        tpr_rerun<D, K, CB>(xr, w[K - 1] & ~CM, sel);
        if constexpr (SORTED) {
            // order the K selected columns by (key desc, col asc): insertion sort
            for (int a2 = 1; a2 < K; ++a2)
                for (int b2 = a2; b2 > 0; --b2) {
                    const uint32_t ca = sel[b2 - 1], cb = sel[b2];
                    const uint32_t ka = order_key(xr[ca]), kb = order_key(xr[cb]);
                    if (kb > ka || (kb == ka && cb < ca)) {
                        sel[b2 - 1] = cb;
                        sel[b2] = ca;
                    }
                }
        }
        // col[] is read back to front below unless SORTED: store descending
#pragma unroll
        for (int t = 0; t < K; ++t) col[t] = SORTED ? sel[t] : sel[K - 1 - t];
    } else if constexpr (!SORTED) {
        bitonic_sort_desc<K>(col);             // descending columns ...
    }
    if (valid) {
        if constexpr (SORTED) {
#pragma unroll
            for (int t = 0; t < K; ++t) {
                vo[t] = xr[col[t]];
                io[t] = (uint8_t)col[t];
            }
        } else {
            // ... written back to front: ascending (CBSR order)
            float ov[K];
            uint32_t ob[K / 4 > 0 ? K / 4 : 1];
#pragma unroll
            for (int t = 0; t < (K / 4 > 0 ? K / 4 : 1); ++t) ob[t] = 0u;
#pragma unroll
            for (int t = 0; t < K; ++t) {
                const uint32_t c = col[K - 1 - t];
                ov[t] = xr[c];
                ob[t >> 2] |= c << (8 * (t & 3));
            }
            if constexpr (K % 4 == 0) {
#pragma unroll
                for (int t = 0; t < K / 4; ++t)
                    reinterpret_cast<float4 *>(vo)[t] = make_float4(ov[4 * t], ov[4 * t + 1], ov[4 * t + 2], ov[4 * t + 3]);
                if constexpr (K == 4) *reinterpret_cast<uint32_t *>(io) = ob[0];
                else if constexpr (K == 8) *reinterpret_cast<uint2 *>(io) = make_uint2(ob[0], ob[1]);
                else {
#pragma unroll
                    for (int t = 0; t < K / 16; ++t)
                        reinterpret_cast<uint4 *>(io)[t] = make_uint4(ob[4 * t], ob[4 * t + 1], ob[4 * t + 2], ob[4 * t + 3]);
                }
            } else {
#pragma unroll
                for (int t = 0; t < K; ++t) {
                    vo[t] = ov[t];
                    io[t] = (uint8_t)(ob[t >> 2] >> (8 * (t & 3)));
                }
            }
        }
    }
}

}  // namespace dr

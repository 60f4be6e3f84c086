// tspmm.cu — tiled DR-SpMM forward (Alg. 1, Eq. 5-7) and SSpMM backward (Alg. 2,
// Eq. 10-11) of a square unit-weight relation (near) on the tcgen05 tensor cores.
//
// The relation is cut into tiles of <= 128 rows with compact neighbourhoods
// (TileSet, graph.cpp). For a tile T with halo H (the distinct ids its rows
// touch), the aggregation of all its rows is one dense product
//     forward : Z_T  = diag(c_T)  Adj[T x H] densify(H_src[H])      (Eq. 5)
//     backward: G_T  = diag(s_T)  Adj^T[T x H] dZ'[H]               (Eq. 10)
// with the 0/1 adjacency tile as the A operand (exact in bf16) and the halo's
// feature rows as the B operand, split x = hi + lo in bf16 (|x - hi - lo| <=
// 2^-17 |x|; A B_hi and A B_lo accumulate side by side in TMEM, fp32). The
// backward then samples G at the source row's own CBSR indices (the D-ReLU mask
// gradient, Eq. 11), adds the extra term (Sage root term + the low-degree second
// relation of the source type, summed beforehand by the SIMT kernel) and writes
// the dense dX row. Every halo row is read once per
// tile (compulsory bytes) instead of once per edge, and the per-edge work moves
// from the L1/shared-memory scatter pipes to the tensor cores.
//
// Roles (one persistent CTA per SM, 14 warps; CTA b takes tiles b, b + grid, ...
// so the SMs sweep consecutive, neighbouring tiles together and shared halo rows
// come from L2; TileSet::cta_chunks lists each CTA's chunk sequence):
//   warp 0     producer  (backward): bulk copies (TMA engine) of the chunk's 64
//                         dZ' halo rows into the stage;
//   warps 2-9  converters: expand the chunk's row masks into the 0/1 adjacency
//                         tile [128 x 64] (bf16);
//                         forward: densify the halo's CBSR rows straight into the
//                         K-major hi/lo B tiles; backward: transposing hi/lo split
//                         of the landed dZ' rows (in place). Their global reads
//                         are cp.async copies into side slots two chunks ahead;
//   warp 1     MMA      : one thread, one N = 2D MMA per K = 16 step ([B_hi; B_lo]
//                         stacked along N) into a double-buffered TMEM accumulator;
//   warps 10-13 epilogue: TMEM -> registers (lane = tile row) -> a per-warp
//                         [32 rows x 32 cols] staging tile -> 128-bit coalesced
//                         row stores (4 rows x 128 B per instruction).
// Fixed summation order everywhere: deterministic, no atomics (reading Q23).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "dr_internal.h"
#include "tc.cuh"

namespace dr {

void ensure_smem(const void *fn, size_t bytes);

namespace {

constexpr int kThreads = 448;
constexpr int kConv = 256;                     // converter threads (warps 2-9)
constexpr int kEpiWarp0 = 10;
constexpr int kMaxSA = 4;
constexpr int kStg = 36;                       // epilogue staging row stride (floats, 144 B)
constexpr uint32_t kATile = 16384;             // 128 x 64 bf16
constexpr uint32_t kStgBytes = 4 * 32 * kStg * 4;      // epilogue staging, 4 warps

struct TsArgs {
    int32_t n_tiles;
    const int32_t *rows, *chunk_beg, *halo, *cta_beg, *cta_chunks, *cta_tiles;
    int tile_stride;
    const uint64_t *abits;
    int k, SA;
    uint32_t stage_bytes, side_bytes;
    // forward: CBSR of the halo (source) rows, per-row output scale, output
    const float *hval;
    const uint8_t *hidx;
    const float *c;
    float *z;
    int z_split;                      // forward output as [hi | lo] bf16 rows
    // backward: dZ' rows of the halo (destinations), optional per-halo-row scale
    // (standalone ABI: dz not yet row-scaled), s_j of the tiled relation, and the
    // extra per-kept-entry term added in the epilogue (root term + other relation)
    const float *dz, *dzc, *s;
    const uint8_t *dzs;               // split dZ' rows ([hi | lo] bf16, 4 D bytes), or null
    const void *zeros;                // forward: >= 2 D 128 zero bytes (TMA zero fill of B), or null
    const float *root;
    float *dx, *g_kept;
    unsigned long long *dbg;          // DR_TS_DEBUG role timers (cycles per CTA), else null
};

// mbarrier wait with a short sleep between probes (roles off the critical path)
__device__ __forceinline__ void wait_sleep(uint64_t *bar, uint32_t phase) {
    tc::mbar_wait_sleep(bar, phase);
}

#define TDBG_T0 const long long dbg_t0 = a.dbg ? clock64() : 0
#define TDBG_ADD(slot) do { if (a.dbg) atomicAdd(a.dbg + blockIdx.x * 16 + (slot), (unsigned long long)(clock64() - dbg_t0)); } while (0)

// ---- transposing split unit (backward B operand): feature quad fq x row octet j
struct Unit {
    int fq, j;
    bool ok;
};
template <int D>
__device__ __forceinline__ Unit unit_of(int ct) {
    constexpr int W4 = D / 4, fh = (W4 + 7) / 8;
    const int i = ct & 7, gq = (ct >> 3) & 3, rest = ct >> 5;
    Unit x;
    x.fq = i + 8 * (rest % fh);
    x.j = gq + 4 * (rest / fh);
    x.ok = x.fq < W4 && x.j < 8;
    return x;
}
__device__ __forceinline__ void store_col8(uint8_t *B, uint32_t lo_off, int f, int j, const float *a) {
    uint4 h, l;
    tc::split_bf16x2(a[0], a[1], h.x, l.x);
    tc::split_bf16x2(a[2], a[3], h.y, l.y);
    tc::split_bf16x2(a[4], a[5], h.z, l.z);
    tc::split_bf16x2(a[6], a[7], h.w, l.w);
    const uint32_t off = tc::sw128_off_h((uint32_t)f, (uint32_t)(8 * j));
    *reinterpret_cast<uint4 *>(B + off) = h;
    *reinterpret_cast<uint4 *>(B + lo_off + off) = l;
}

// ---- converter side buffers
// The converters' global reads for chunk ch are 16/8/4-B async copies
// (cp.async) into a side slot issued two chunks ahead: the chunk's 128 row
// masks (1 KB) and, forward, the CBSR rows of its 64 halo ids (thread ct copies
// its quarter u = ct / 4, h = ct % 4). Halo ids are loaded into registers three
// chunks ahead.
constexpr int kSideSlots = 3;
constexpr uint32_t kSideA = 1024;              // 128 x 64-bit row masks
struct CInfo {
    int id;          // forward: halo id of row u = ct / 4
    int h0, h1;      // backward: halo ids of rows lane, lane + 32 (valid-row count)
};
template <bool BWD>
__device__ __forceinline__ void info_load(const TsArgs &a, int64_t ch, int ct, CInfo &p) {
    if (!BWD || a.dzs) {
        p.id = __ldg(a.halo + ch * kTsChunk + (ct >> 2));
    } else {
        p.h0 = __ldg(a.halo + ch * kTsChunk + (ct & 31));
        p.h1 = __ldg(a.halo + ch * kTsChunk + 32 + (ct & 31));
    }
}
template <bool BWD, int QH>
__device__ __forceinline__ void side_issue(const TsArgs &a, int64_t ch, const CInfo &p, uint8_t *sd,
                                           int ct) {
    if (ct < 64) tc::cp_async16(sd + 16 * ct, a.abits + ch * kTsRows + 2 * ct, 16);
    if constexpr (!BWD) {
        if (p.id >= 0) {
            constexpr int K = 4 * QH;
            const int u = ct >> 2, h = ct & 3;
            uint8_t *sv = sd + kSideA + u * K * 4 + h * QH * 4;
            const float *gv = a.hval + (int64_t)p.id * K + h * QH;
            if constexpr (QH == 8) {
                tc::cp_async16(sv, gv, 16);
                tc::cp_async16(sv + 16, gv + 4, 16);
            } else if constexpr (QH == 4) {
                tc::cp_async16(sv, gv, 16);
            } else if constexpr (QH == 2) {
                tc::cp_async8(sv, gv);
            } else {
                tc::cp_async4(sv, gv, 4);
            }
            if (h == 0) {
                uint8_t *si = sd + kSideA + 64 * K * 4 + u * K;
                const uint8_t *gi = a.hidx + (int64_t)p.id * K;
                if constexpr (QH == 8) {
                    tc::cp_async16(si, gi, 16);
                    tc::cp_async16(si + 16, gi + 16, 16);
                } else if constexpr (QH == 4) {
                    tc::cp_async16(si, gi, 16);
                } else if constexpr (QH == 2) {
                    tc::cp_async8(si, gi);
                } else {
                    tc::cp_async4(si, gi, 4);
                }
            }
        }
    }
}

// Backward, split dZ' input: the 64 halo rows' [hi | lo] bf16 halves are copied
// (cp.async, 16-B pieces) straight into the MN-major SW128 B operand of the
// stage -- K = halo slot u (row u % 8 of 8-row group u / 8, 1 KB apart), N =
// feature (64-feature atoms 8 KB apart, hi atoms then lo atoms): no conversion.
// Thread ct copies row u = ct / 4, pieces h, h + 4, ... (h = ct % 4); rows with
// no halo id are zero-filled.
template <int D>
__device__ __forceinline__ void gather_split(const TsArgs &a, const CInfo &p, uint8_t *B, int ct) {
    constexpr int NP = D / 4;                  // 16-B pieces per split row (hi + lo)
    const int u = ct >> 2, h = ct & 3;
    const uint8_t *src = a.dzs + (int64_t)(p.id >= 0 ? p.id : 0) * (4 * D);
    const uint32_t nb = p.id >= 0 ? 16u : 0u;
    uint8_t *rowb = B + (u >> 3) * 1024 + (u & 7) * 128;
#pragma unroll
    for (int q = 0; q < NP / 4; ++q) {
        const int pc = h + 4 * q;              // piece: hi 0 .. D/8-1, lo D/8 .. D/4-1
        const int lo = pc >= D / 8, c = lo ? pc - D / 8 : pc;
        const int atom = (lo ? D / 64 : 0) + (c >> 3), cc = c & 7;
        tc::cp_async16(rowb + atom * 8192 + ((cc ^ (u & 7)) << 4), src + 16 * pc, nb);
    }
}

// The [128 x 64] bf16 A tile from the chunk's row masks: thread ct writes row
// m = ct / 2, halo slots [32 h, 32 h + 32) (h = ct % 2) as four whole 16-B
// swizzle chunks of 0 / 1.0 -- every element written, no zero fill, no scatter.
__device__ __forceinline__ void build_a(const uint8_t *sd, uint8_t *A, int ct) {
    const int m = ct >> 1, h = ct & 1;
    const uint32_t bits = reinterpret_cast<const uint32_t *>(sd)[2 * m + h];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t byte = bits >> (8 * c);
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t t = byte >> (2 * j);
            w[j] = (((t & 1u) * 0xFFFFu) | ((t & 2u) * 0x7FFF8000u)) & 0x3F803F80u;
        }
        *reinterpret_cast<uint4 *>(A + m * 128 + (((4 * h + c) ^ (m & 7)) << 4)) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

template <int D, int QH>
__device__ __forceinline__ void convert_fwd(const TsArgs &a, const CInfo &p, const uint8_t *sd,
                                            uint8_t *st, int ct, bool zero_b) {
    uint8_t *A = st, *B = st + kATile;
    constexpr uint32_t lo = (uint32_t)D * 128u;
    constexpr int K = 4 * QH;
    if (zero_b) {                           // (else the TMA zero-filled it)
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int i = 0; i < (2 * D * 128) / (16 * kConv); ++i)
            reinterpret_cast<uint4 *>(B)[ct + kConv * i] = z;
    }
    tc::cp_async_wait<1>();                 // this chunk's side copies (ch + 1's may fly)
    tc::named_bar(1, kConv);                // B zeroed + everyone's side data visible
    build_a(sd, A, ct);
    if (p.id >= 0) {
        const int u = ct >> 2, h = ct & 3;
        const float *sv = reinterpret_cast<const float *>(sd + kSideA) + u * K + h * QH;
        const uint8_t *si = sd + kSideA + 64 * K * 4 + u * K + h * QH;
#pragma unroll
        for (int q = 0; q < QH; ++q) {
            uint32_t hh, ll;
            tc::split_bf16x2(sv[q], 0.f, hh, ll);
            const uint32_t off = tc::sw128_off_h(si[q], (uint32_t)u);
            *reinterpret_cast<uint16_t *>(B + off) = (uint16_t)(hh & 0xffffu);
            *reinterpret_cast<uint16_t *>(B + lo + off) = (uint16_t)(ll & 0xffffu);
        }
    }
}

template <int D, int QH>
__device__ __forceinline__ void convert_bwd(const TsArgs &a, const CInfo &p, const uint8_t *sd,
                                            uint8_t *st, int ct, int64_t ch) {
    uint8_t *A = st, *B = st + kATile;
    constexpr uint32_t lo = (uint32_t)D * 128u;
    // valid rows of the chunk = a prefix (halo padding sits at the end of a tile)
    const int valid = __popc(__ballot_sync(0xffffffffu, p.h0 >= 0)) +
                      __popc(__ballot_sync(0xffffffffu, p.h1 >= 0));
    const float4 *raw = reinterpret_cast<const float4 *>(B);
    const Unit x = unit_of<D>(ct);
    float4 vv[8];
    if (x.ok) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int rr = 8 * x.j + r;
            float4 q = rr < valid ? raw[rr * (D / 4) + x.fq] : make_float4(0.f, 0.f, 0.f, 0.f);
            if (a.dzc && rr < valid) {             // standalone ABI: dz rows not yet scaled
                const float cs = __ldg(a.dzc + __ldg(a.halo + ch * kTsChunk + rr));
                q.x *= cs; q.y *= cs; q.z *= cs; q.w *= cs;
            }
            vv[r] = q;
        }
    }
    tc::cp_async_wait<1>();
    tc::named_bar(1, kConv);                 // raw reads done (in place) + side data visible
    build_a(sd, A, ct);
    if (x.ok) {
        const int f = 4 * x.fq;
        float c8[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) c8[r] = vv[r].x;
        store_col8(B, lo, f + 0, x.j, c8);
#pragma unroll
        for (int r = 0; r < 8; ++r) c8[r] = vv[r].y;
        store_col8(B, lo, f + 1, x.j, c8);
#pragma unroll
        for (int r = 0; r < 8; ++r) c8[r] = vv[r].z;
        store_col8(B, lo, f + 2, x.j, c8);
#pragma unroll
        for (int r = 0; r < 8; ++r) c8[r] = vv[r].w;
        store_col8(B, lo, f + 3, x.j, c8);
    }
}

// ---- epilogue helpers (warp quarter qd: tile rows 32 qd + lane; TMEM lanes likewise)
// TMEM columns [j0, j0+32) of this warp's 32 rows -> staging (row = lane), scaled
template <int D>
__device__ __forceinline__ void tmem_to_stg(uint32_t taddr, float scale, float *stg, int lane) {
    uint32_t r0[16], r1[16], q0[16], q1[16];
    tc::tmem_ld16_nw(taddr, r0);
    tc::tmem_ld16_nw(taddr + 16u, r1);
    tc::tmem_ld16_nw(taddr + (uint32_t)D, q0);          // A B_lo half
    tc::tmem_ld16_nw(taddr + (uint32_t)D + 16u, q1);
    tc::tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        r0[q] = __float_as_uint(__uint_as_float(r0[q]) + __uint_as_float(q0[q]));
        r1[q] = __float_as_uint(__uint_as_float(r1[q]) + __uint_as_float(q1[q]));
    }
    float4 *o = reinterpret_cast<float4 *>(stg + lane * kStg);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        o[q] = make_float4(scale * __uint_as_float(r0[4 * q]), scale * __uint_as_float(r0[4 * q + 1]),
                           scale * __uint_as_float(r0[4 * q + 2]), scale * __uint_as_float(r0[4 * q + 3]));
#pragma unroll
    for (int q = 0; q < 4; ++q)
        o[4 + q] = make_float4(scale * __uint_as_float(r1[4 * q]), scale * __uint_as_float(r1[4 * q + 1]),
                               scale * __uint_as_float(r1[4 * q + 2]), scale * __uint_as_float(r1[4 * q + 3]));
}
// staging [32 rows][32 cols] -> out[rid_r * D + j0 ...]: lane -> (row 4 i + lane / 8,
// column quad lane % 8): each instruction writes 4 full 128-B row segments
template <int D>
__device__ __forceinline__ void stg_to_global(const float *stg, float *out, int rid, int j0, int lane) {
    const int cq = lane & 7, rs = lane >> 3;
    float4 v[8];
    int rr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + rs;
        rr[i] = __shfl_sync(0xffffffffu, rid, r);
        v[i] = *reinterpret_cast<const float4 *>(stg + r * kStg + 4 * cq);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (rr[i] >= 0) __stcs(reinterpret_cast<float4 *>(out + (int64_t)rr[i] * D + j0) + cq, v[i]);
}

// split output rows ([hi | lo] bf16 halves, 4 D bytes): hi of column j at 2 j,
// lo at 2 (D + j)
template <int D>
__device__ __forceinline__ void stg_to_global_split(const float *stg, uint8_t *out, int rid, int j0,
                                                    int lane) {
    const int cq = lane & 7, rs = lane >> 3;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = 4 * i + rs;
        const int rr = __shfl_sync(0xffffffffu, rid, r);
        const float4 v = *reinterpret_cast<const float4 *>(stg + r * kStg + 4 * cq);
        uint2 h, l;
        tc::split_bf16x2(v.x, v.y, h.x, l.x);
        tc::split_bf16x2(v.z, v.w, h.y, l.y);
        if (rr >= 0) {
            uint8_t *rowp = out + (int64_t)rr * D * 4;
            __stcs(reinterpret_cast<uint2 *>(rowp + 2 * (j0 + 4 * cq)), h);
            __stcs(reinterpret_cast<uint2 *>(rowp + 2 * (D + j0 + 4 * cq)), l);
        }
    }
}

template <int D>
__device__ __forceinline__ void epi_fwd(const TsArgs &a, int t, uint32_t tacc, float *stg, int lane) {
    const int rid = __ldg(a.rows + (int64_t)t * kTsRows + (tacc >> 16) + lane);
    const float cr = rid >= 0 ? __ldg(a.c + rid) : 0.f;
#pragma unroll 1
    for (int j0 = 0; j0 < D; j0 += 32) {
        tmem_to_stg<D>(tacc + (uint32_t)j0, cr, stg, lane);
        __syncwarp();
        if (a.z_split) stg_to_global_split<D>(stg, reinterpret_cast<uint8_t *>(a.z), rid, j0, lane);
        else stg_to_global<D>(stg, a.z, rid, j0, lane);
        __syncwarp();
    }
}

// Per-row inputs of the backward epilogue, loaded one tile ahead (software
// pipelined across tiles): the row id, its CBSR indices and its extra term
// (root term + second relation, summed beforehand).
template <int K>
struct EpiIn {
    static constexpr bool kPre = K <= 16;     // K = 32: extra term loaded at use (registers)
    int rid;
    uint32_t idw[K / 4];
    float ex[kPre ? K : 1];
};
template <int K>
__device__ __forceinline__ void load_extra(const TsArgs &a, int rid, float *ex) {
    if (rid >= 0 && a.root) {
        const float4 *rr = reinterpret_cast<const float4 *>(a.root + (int64_t)rid * K);
#pragma unroll
        for (int q = 0; q < K / 4; ++q) {
            const float4 v = __ldg(rr + q);
            ex[4 * q] = v.x; ex[4 * q + 1] = v.y; ex[4 * q + 2] = v.z; ex[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q) ex[q] = 0.f;
    }
}
template <int K>
__device__ __forceinline__ void epi_in_load(const TsArgs &a, int t, int m, EpiIn<K> &e) {
    e.rid = __ldg(a.rows + (int64_t)t * kTsRows + m);
    if (e.rid >= 0) {
        const uint8_t *ir = a.hidx + (int64_t)e.rid * K;
#pragma unroll
        for (int q = 0; q < K / 4; ++q) e.idw[q] = __ldg(reinterpret_cast<const uint32_t *>(ir) + q);
    } else {
#pragma unroll
        for (int q = 0; q < K / 4; ++q) e.idw[q] = 0;
    }
    if constexpr (EpiIn<K>::kPre) load_extra<K>(a, e.rid, e.ex);
}

template <int D, int QH>
__device__ __forceinline__ void epi_bwd(const TsArgs &a, const EpiIn<4 * QH> &in, uint32_t tacc,
                                        float *stg, int lane, uint64_t *accempty) {
    constexpr int K = 4 * QH;
    const int rid = in.rid;
    auto idx = [&](int q) -> uint32_t { return (in.idw[q >> 2] >> (8 * (q & 3))) & 0xffu; };
    float g[K];
#pragma unroll
    for (int q = 0; q < K; ++q) g[q] = 0.f;
    // sample the accumulator row at the row's own CBSR indices
#pragma unroll 1
    for (int j0 = 0; j0 < D; j0 += 32) {
        tmem_to_stg<D>(tacc + (uint32_t)j0, 1.f, stg, lane);
        __syncwarp();
#pragma unroll
        for (int q = 0; q < K; ++q)
            if ((int)(idx(q) >> 5) == (j0 >> 5)) g[q] = stg[lane * kStg + (idx(q) & 31u)];
        __syncwarp();
    }
    // the accumulator buffer is free for the next tile's MMAs
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(accempty);
    const float sj = rid >= 0 ? __ldg(a.s + rid) : 0.f;
    if constexpr (EpiIn<K>::kPre) {
#pragma unroll
        for (int q = 0; q < K; ++q) g[q] = sj * g[q] + in.ex[q];
    } else {
        float ex[K];
        load_extra<K>(a, rid, ex);
#pragma unroll
        for (int q = 0; q < K; ++q) g[q] = sj * g[q] + ex[q];
    }
    if (rid >= 0 && a.g_kept) {
        float4 *o = reinterpret_cast<float4 *>(a.g_kept + (int64_t)rid * K);
#pragma unroll
        for (int q = 0; q < K / 4; ++q) o[q] = make_float4(g[4 * q], g[4 * q + 1], g[4 * q + 2], g[4 * q + 3]);
    }
    if (!a.dx) return;
    // dense dX row: zeros + the K values at their indices, 32 columns at a time
#pragma unroll 1
    for (int j0 = 0; j0 < D; j0 += 32) {
        float4 *o = reinterpret_cast<float4 *>(stg + lane * kStg);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < K; ++q)
            if ((int)(idx(q) >> 5) == (j0 >> 5)) stg[lane * kStg + (idx(q) & 31u)] = g[q];
        __syncwarp();
        stg_to_global<D>(stg, a.dx, rid, j0, lane);
        __syncwarp();
    }
}

template <bool BWD, int D, int QH>
__global__ void __launch_bounds__(kThreads, 1) tspmm_kernel(const __grid_constant__ TsArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[kMaxSA], conv[kMaxSA], empty[kMaxSA], accfull[2],
        accempty[2];
    __shared__ uint32_t tmem_slot;
    const long long kt00 = clock64();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int SA = a.SA;
    // two accumulators of 2D fp32 columns: [A B_hi | A B_lo], summed in the epilogue
    // (one N = 2D MMA per K step reads the A tile once)
    constexpr uint32_t ncols = 4 * D;
    if (tid == 0) {
        for (int i = 0; i < SA; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&conv[i], kConv / 32);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&accfull[i], 1);
            tc::mbar_init(&accempty[i], 4);
        }
        tc::fence_mbar_init();
    }
    if (warp == 1) {
        tc::tmem_alloc(&tmem_slot, ncols);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    const long long kt0 = clock64();
    if (a.dbg && tid == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        a.dbg[blockIdx.x * 16 + 11] = g;                                  // start (ns)
    }
    float *stg_all = reinterpret_cast<float *>(sm + (size_t)SA * a.stage_bytes);
    // this CTA: tiles blockIdx.x, + gridDim.x, ...; its chunk sequence (same order)
    // is cta_chunks[base, base + n_it)
    const int base = __ldg(a.cta_beg + blockIdx.x), n_it = __ldg(a.cta_beg + blockIdx.x + 1) - base;
    auto cid = [&](int i) -> int { return i < n_it ? __ldg(a.cta_chunks + base + i) : 0; };
    // its tiles: t0, t0 + stride, ... (n_t of them), in the same order
    const int t0 = __ldg(a.cta_tiles + 2 * blockIdx.x), n_t = __ldg(a.cta_tiles + 2 * blockIdx.x + 1);
    const int tstride = a.tile_stride;

    if (warp == 0) {
        if (!BWD && a.zeros) {
            // forward: the B tile of each stage is zero-filled by the TMA engine (bulk
            // copy of an L2-resident zero buffer) once the MMA has released the slot,
            // so the converters only scatter the CBSR values into it
            const uint32_t bb = 2u * (uint32_t)D * 128u;
            for (int it = 0; it < n_it; ++it) {
                const int slot = it % SA;
                const uint32_t u = (uint32_t)(it / SA);
                if (u > 0) {
                    TDBG_T0;
                    wait_sleep(&empty[slot], (u - 1) & 1u);
                    if (lane == 0) TDBG_ADD(0);
                }
                if (lane == 0) {
                    tc::mbar_arrive_expect_tx(&full[slot], bb);
                    tc::bulk_g2s(sm + (size_t)slot * a.stage_bytes + kATile, a.zeros, bb, &full[slot]);
                }
                __syncwarp();
            }
        } else if (BWD && !a.dzs) {
            int nid0 = -1, nid1 = -1, cn = cid(1);
            if (n_it > 0) {
                const int c = cid(0);
                nid0 = __ldg(a.halo + (int64_t)c * kTsChunk + lane);
                nid1 = __ldg(a.halo + (int64_t)c * kTsChunk + 32 + lane);
            }
            for (int it = 0; it < n_it; ++it) {
                const int slot = it % SA;
                const uint32_t u = (uint32_t)(it / SA);
                const int id0 = nid0, id1 = nid1;
                if (it + 1 < n_it) {
                    nid0 = __ldg(a.halo + (int64_t)cn * kTsChunk + lane);
                    nid1 = __ldg(a.halo + (int64_t)cn * kTsChunk + 32 + lane);
                    cn = cid(it + 2);
                }
                if (u > 0) {
                    TDBG_T0;
                    wait_sleep(&empty[slot], (u - 1) & 1u);
                    if (lane == 0) TDBG_ADD(0);
                }
                uint64_t *fb = &full[slot];
                const uint32_t nv = __popc(__ballot_sync(0xffffffffu, id0 >= 0)) +
                                    __popc(__ballot_sync(0xffffffffu, id1 >= 0));
                if (lane == 0) tc::mbar_arrive_expect_tx(fb, nv * (uint32_t)D * 4u);
                __syncwarp();
                uint8_t *B = sm + (size_t)slot * a.stage_bytes + kATile;
                if (id0 >= 0) tc::bulk_g2s(B + (size_t)lane * D * 4, a.dz + (int64_t)id0 * D, D * 4, fb);
                if (id1 >= 0) tc::bulk_g2s(B + (size_t)(32 + lane) * D * 4, a.dz + (int64_t)id1 * D, D * 4, fb);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const bool mn = BWD && a.dzs != nullptr;          // split input: MN-major B
            const uint32_t idesc = tc::idesc_bf16(kTsRows, 2 * D) | (mn ? (1u << 16) : 0u);
            int it = 0;
            for (int lt = 0; lt < n_t; ++lt) {
                const int t = t0 + lt * tstride;
                const int b = lt & 1;
                if (lt >= 2) {
                    TDBG_T0;
                    wait_sleep(&accempty[b], (uint32_t)((lt / 2 - 1) & 1));
                    TDBG_ADD(2);
                }
                tc::fence_after();
                const uint32_t d = tmem + (uint32_t)(b * 2 * D);
                const int c0 = __ldg(a.chunk_beg + t), c1 = __ldg(a.chunk_beg + t + 1);
                for (int ch = c0; ch < c1; ++ch, ++it) {
                    const int slot = it % SA;
                    {
                        TDBG_T0;
                        wait_sleep(&conv[slot], (uint32_t)((it / SA) & 1));
                        TDBG_ADD(1);
                    }
                    tc::fence_after();
                    const uint32_t sa = tc::smem_u32(sm + (size_t)slot * a.stage_bytes);
                    const uint32_t sbh = sa + kATile;     // [B_hi ; B_lo] = 2D K-major rows
#pragma unroll
                    for (int ks = 0; ks < kTsChunk / 16; ++ks) {
                        const uint32_t ko = ks * 32;
                        const uint64_t bd = mn ? tc::desc_mn_sw128(sbh + ks * 2048u, 8192u, 1024u)
                                               : tc::desc_sw128(sbh + ko);
                        tc::mma_bf16(d, tc::desc_sw128(sa + ko), bd, idesc,
                                     (ch == c0 && ks == 0) ? 0u : 1u);
                    }
                    tc::mma_commit(&empty[slot]);
                }
                tc::mma_commit(&accfull[b]);
            }
        }
        __syncwarp();
    } else if (warp < kEpiWarp0) {
        const int ct = tid - 64;
        uint8_t *side = sm + (size_t)SA * a.stage_bytes + kStgBytes;
        // rings over the CTA's chunk sequence: ids c0..c3 (steps it..it+3), infos
        // i0..i2 (it..it+2); side copies are in flight for it, it + 1
        int c0 = cid(0), c1 = cid(1), c2 = cid(2), c3 = cid(3);
        CInfo i0{}, i1{}, i2{}, i3{};
        const bool split = BWD && a.dzs != nullptr;
        if (n_it > 0) info_load<BWD>(a, c0, ct, i0);
        if (n_it > 1) info_load<BWD>(a, c1, ct, i1);
        if (n_it > 2) info_load<BWD>(a, c2, ct, i2);
        if (n_it > 0) {
            side_issue<BWD, QH>(a, c0, i0, side, ct);
            if (split) gather_split<D>(a, i0, sm + kATile, ct);
        }
        tc::cp_async_commit();
        if (n_it > 1) {
            side_issue<BWD, QH>(a, c1, i1, side + a.side_bytes, ct);
            if (split) gather_split<D>(a, i1, sm + (size_t)(1 % SA) * a.stage_bytes + kATile, ct);
        }
        tc::cp_async_commit();
        for (int it = 0; it < n_it; ++it) {
            const int c4 = cid(it + 4);
            if (it + 3 < n_it) info_load<BWD>(a, c3, ct, i3);
            const int slot = it % SA;
            const uint32_t u = (uint32_t)(it / SA);
            uint8_t *st = sm + (size_t)slot * a.stage_bytes;
            const uint8_t *sd = side + (size_t)(it % kSideSlots) * a.side_bytes;
            if (split) {
                // chunk it + 2's copies go into its stage slot once the MMA of the
                // chunk that used it (it + 2 - SA) is done, and into its side slot
                // (read at step it - 1 by everyone: the barrier of step it - 1... is
                // passed by all before anyone reaches step it's issue -- see below)
                {
                    TDBG_T0;
                    if (it + 2 < n_it) {
                        const int s2 = (it + 2) % SA;
                        const uint32_t u2 = (uint32_t)((it + 2) / SA);
                        if (u2 > 0) tc::mbar_wait(&empty[s2], (u2 - 1) & 1u);
                    }
                    if (ct == 0) TDBG_ADD(3);
                }
                tc::named_bar(1, kConv);       // all done reading side slot (it + 2) % 3 (step it - 1)
                if (it + 2 < n_it) {
                    side_issue<BWD, QH>(a, c2, i2, side + (size_t)((it + 2) % kSideSlots) * a.side_bytes, ct);
                    gather_split<D>(a, i2, sm + (size_t)((it + 2) % SA) * a.stage_bytes + kATile, ct);
                }
                tc::cp_async_commit();
                TDBG_T0;
                tc::cp_async_wait<2>();        // chunk it's copies landed (this thread's)
                tc::named_bar(1, kConv);       // ... and everyone's
                build_a(sd, st, ct);
                if (ct == 0) TDBG_ADD(4);
            } else {
                {
                    TDBG_T0;
                    if (BWD || a.zeros) tc::mbar_wait(&full[slot], u & 1u);
                    else if (u > 0) tc::mbar_wait(&empty[slot], (u - 1) & 1u);
                    if (ct == 0) TDBG_ADD(3);
                }
                {
                    TDBG_T0;
                    if constexpr (BWD) convert_bwd<D, QH>(a, i0, sd, st, ct, c0);
                    else convert_fwd<D, QH>(a, i0, sd, st, ct, a.zeros == nullptr);
                    if (ct == 0) TDBG_ADD(4);
                }
                // every converter thread is past the barrier inside convert: the slot
                // read at step it - 1 is free for step it + 2
                if (it + 2 < n_it)
                    side_issue<BWD, QH>(a, c2, i2, side + (size_t)((it + 2) % kSideSlots) * a.side_bytes, ct);
                tc::cp_async_commit();
            }
            tc::fence_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&conv[slot]);
            c0 = c1; c1 = c2; c2 = c3; c3 = c4;
            i0 = i1; i1 = i2; i2 = i3;
        }
        tc::cp_async_wait<0>();
    } else {
        const int qd = warp & 3;
        float *stg = stg_all + (size_t)(warp - kEpiWarp0) * 32 * kStg;
        EpiIn<4 * QH> cur, nxt;
        if constexpr (BWD) {
            if (n_t > 0) epi_in_load<4 * QH>(a, t0, qd * 32 + lane, cur);
        }
        for (int lt = 0; lt < n_t; ++lt) {
            const int t = t0 + lt * tstride;
            const int b = lt & 1;
            if constexpr (BWD) {
                if (lt + 1 < n_t) epi_in_load<4 * QH>(a, t + tstride, qd * 32 + lane, nxt);
            }
            {
                TDBG_T0;
                wait_sleep(&accfull[b], (uint32_t)((lt / 2) & 1));
                if (warp == kEpiWarp0 && lane == 0) TDBG_ADD(5);
            }
            tc::fence_after();
            TDBG_T0;
            const uint32_t tacc = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(b * 2 * D);
            if constexpr (BWD) {
                epi_bwd<D, QH>(a, cur, tacc, stg, lane, &accempty[b]);
                cur = nxt;
            } else {
                epi_fwd<D>(a, t, tacc, stg, lane);
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&accempty[b]);
            }
            if (warp == kEpiWarp0 && lane == 0) TDBG_ADD(6);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (a.dbg && tid == 0) {
        const long long kt1 = clock64();
        atomicAdd(a.dbg + blockIdx.x * 16 + 8, (unsigned long long)(kt1 - kt0));
        a.dbg[blockIdx.x * 16 + 10] = (unsigned long long)(kt0 - kt00);   // setup
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        a.dbg[blockIdx.x * 16 + 12] = g;                                  // end (ns)
    }
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, ncols);
    }
}

template <bool BWD>
const void *pick(int D, int k) {
#define DR_TS_CASE(DD, KK)                                                                        \
    if (D == DD && k == KK) return (const void *)tspmm_kernel<BWD, DD, KK / 4>;
    DR_TS_CASE(64, 4) DR_TS_CASE(64, 8) DR_TS_CASE(64, 16) DR_TS_CASE(64, 32)
    DR_TS_CASE(128, 4) DR_TS_CASE(128, 8) DR_TS_CASE(128, 16) DR_TS_CASE(128, 32)
#undef DR_TS_CASE
    return nullptr;
}

void launch(const TileSet &ts, TsArgs &a, int D, bool bwd, cudaStream_t s) {
    a.rows = ts.rows;
    a.chunk_beg = ts.chunk_beg;
    a.halo = ts.halo;
    a.abits = ts.abits;
    a.cta_beg = ts.cta_beg;
    a.cta_chunks = ts.cta_chunks;
    a.cta_tiles = ts.cta_tiles;
    a.tile_stride = ts.tile_stride;
    a.n_tiles = ts.n_tiles;
    a.stage_bytes = kATile + 256u * (uint32_t)D;
    a.side_bytes = (uint32_t)(kSideA + (bwd ? 0 : 64 * a.k * 5) + 127) & ~127u;
    const size_t budget = 227 * 1024 - 1024 - kStgBytes - (size_t)kSideSlots * a.side_bytes - 512;
    a.SA = (int)std::min<size_t>(knobs().ts_sa > 0 ? knobs().ts_sa : kMaxSA, budget / a.stage_bytes);
    // >= 3: the split backward gathers chunk it + 2 into its stage slot while chunk
    // it's slot is still being read (SA = 2 would wait on itself)
    DR_CHECK(a.SA >= 3, DR_ERR_UNSUPPORTED, "tspmm: shared memory budget");
    const size_t smem = (size_t)a.SA * a.stage_bytes + kStgBytes + (size_t)kSideSlots * a.side_bytes + 1024;
    const void *fn = bwd ? pick<true>(D, a.k) : pick<false>(D, a.k);
    DR_CHECK(fn, DR_ERR_UNSUPPORTED, "tspmm: unsupported D/k");
    ensure_smem(fn, smem);
    const int grid = ts.grid;
    if (grid <= 0) return;
    static unsigned long long *dbg_buf = nullptr;
    if (knobs().ts_debug) {
        if (!dbg_buf) DR_CUDA(cudaMalloc(&dbg_buf, 148 * 16 * 8));
        DR_CUDA(cudaMemsetAsync(dbg_buf, 0, 148 * 16 * 8, s));
        a.dbg = dbg_buf;
    }
    void *args[] = {(void *)&a};
    DR_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kThreads), args, smem, s));
    if (a.dbg) {
        unsigned long long h[148 * 16];
        DR_CUDA(cudaStreamSynchronize(s));
        DR_CUDA(cudaMemcpy(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost));
        double t[16] = {0}, tmax = 0, setup_max = 0;
        unsigned long long g0 = ~0ull, g1 = 0, g0max = 0;
        for (int b = 0; b < grid; ++b) {
            for (int q = 0; q < 10; ++q) t[q] += (double)h[b * 16 + q] / grid;
            tmax = std::max(tmax, (double)h[b * 16 + 8]);
            setup_max = std::max(setup_max, (double)h[b * 16 + 10]);
            g0 = std::min(g0, h[b * 16 + 11]);
            g0max = std::max(g0max, h[b * 16 + 11]);
            g1 = std::max(g1, h[b * 16 + 12]);
        }
        fprintf(stderr, "[tspmm %s] max CTA kcycles %.1f, max setup kcycles %.1f, CTA start spread %.1f us, "
                "first start -> last end %.1f us\n", bwd ? "bwd" : "fwd", tmax / 1e3, setup_max / 1e3,
                (g0max - g0) / 1e3, (g1 - g0) / 1e3);
        fprintf(stderr,
                "[tspmm %s D=%d k=%d tiles=%d chunks=%lld SA=%d] kcycles/CTA: total %.1f | prod wait "
                "%.1f | mma wait conv %.1f acc %.1f | conv pre %.1f wait %.1f work %.1f | epi wait "
                "%.1f work %.1f\n",
                bwd ? "bwd" : "fwd", D, a.k, ts.n_tiles, (long long)ts.n_chunks, a.SA, t[8] / 1e3,
                t[0] / 1e3, t[1] / 1e3, t[2] / 1e3, t[9] / 1e3, t[3] / 1e3, t[4] / 1e3, t[5] / 1e3,
                t[6] / 1e3);
    }
}

}  // namespace

bool tspmm_supported(const TileSet &ts, int dim, int k) {
    if (knobs().tspmm == 0) return false;             // experiments only: 0 disables
    return ts.n_tiles > 0 && (dim == 64 || dim == 128) && (k == 4 || k == 8 || k == 16 || k == 32);
}

// A 64 KB device buffer of zeros (the forward's TMA zero fill source), made once.
static const void *zero_buffer() {
    static void *p = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        if (cudaMalloc(&p, 65536) != cudaSuccess || cudaMemset(p, 0, 65536) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
    });
    return p;
}

void launch_tspmm_fwd(const RelDev &r, const float *hval, const uint8_t *hidx, int k, int dim,
                      float *z, cudaStream_t s, bool z_split) {
    TsArgs a{};
    a.z_split = z_split ? 1 : 0;
    // DR_TS_ZEROFILL=1: the TMA zero-fills B from an L2-resident zero buffer
    // instead of the converters (measured slower at C2 and C4: smem fill
    // bandwidth, not converter issue, bounds it; kept as an experiment)
    a.zeros = knobs().ts_zerofill == 1 ? zero_buffer() : nullptr;
    a.k = k;
    a.hval = hval;
    a.hidx = hidx;
    a.c = r.c;
    a.z = z;
    ProfScope ps("spmm_fwd", s);
    launch(r.tiles, a, dim, false, s);
    note_launch("tspmm_fwd");
}

void launch_tspmm_bwd(const RelDev &r, const float *dz, bool dz_split, bool apply_c,
                      const float *extra, const uint8_t *hidx, int k, int dim, float *g_kept,
                      float *dx, cudaStream_t s) {
    TsArgs a{};
    a.k = k;
    a.hidx = hidx;
    a.dz = dz;
    if (dz_split) {
        DR_CHECK(!apply_c, DR_ERR_INVALID_ARGUMENT, "tspmm: split dz must be row-scaled");
        a.dzs = reinterpret_cast<const uint8_t *>(dz);
    }
    a.dzc = apply_c ? r.c : nullptr;
    a.s = r.s;
    a.root = extra;
    a.dx = dx;
    a.g_kept = g_kept;
    ProfScope ps("spmm_bwd", s);
    launch(r.tilesT, a, dim, true, s);
    note_launch("tspmm_bwd");
}

}  // namespace dr

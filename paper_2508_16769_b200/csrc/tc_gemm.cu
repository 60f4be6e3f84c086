// tc_gemm.cu — tensor-core (tcgen05, kind::tf32) row-tile GEMMs for the dense
// parts of a HeteroConv layer (Eq. 4 W^psi; backward dZ = dY W^T,
// Eq. 10-13), with the layer epilogues fused.
//
// Precision: the parity bar is 1e-4 (north_star); plain TF32 (10-bit mantissa)
// misses it, so every product is evaluated as 3xTF32: a = a_hi + a_lo,
// b = b_hi + b_lo, a*b ~ a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (error ~2^-22).
//
// Structure (one CTA of 128 threads per SM-slot, persistent over 128-row tiles):
//   * B (weights) is pre-split and packed once per call by pack_b_kernel into
//     the exact K-major SW128 shared-memory image, chunk by chunk (32 K wide),
//     so each chunk arrives with one cp.async.bulk (TMA engine) copy;
//   * A (activations) is read with 128-bit loads, split hi/lo (and masked, or
//     densified from CBSR) by all threads and written swizzled;
//   * two smem stages: while the tensor core runs chunk s, threads stage s+1;
//     thread 0 issues 3 x 4 MMAs per chunk (M=128, N<=256, K=8 each) into TMEM
//     and commits to the stage's mbarrier;
//   * epilogue: each thread owns one output row (TMEM lane), reads 16 columns
//     at a time with tcgen05.ld and applies bias / max-merge / mask bits /
//     taps (forward) or the destination normaliser (backward dZ).
// A GEMM may have two K segments (dense Z, then the densified CBSR root input),
// so the SageConv root term Hd·Wr is part of the same accumulation.
#include "dr_internal.h"
#include "proj.h"
#include "tc.cuh"
#include "tc_gemm.h"

namespace dr {
namespace {

constexpr int kTM = 128;             // rows per tile (MMA M)
constexpr int kKC = 32;              // K per chunk (one 128-B swizzle atom of fp32)
constexpr int kThreadsTC = 128;

// ---------------------------------------------------------------- B packing
// img[c] = { hi: NB rows x 128 B (swizzled), lo: NB rows x 128 B } for chunk c of
// segment: B_op[n][kk] = transpose ? W[kk*ldw + n] : W[n*ldw + kk], kk < K, n < NB.
__global__ void pack_b_kernel(const float *__restrict__ W, int ldw, int K, int NB, int transpose,
                              uint8_t *__restrict__ img) {
    const int chunks = (K + kKC - 1) / kKC;
    const int64_t total = (int64_t)chunks * NB * kKC;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(e % kKC);
        const int n = (int)((e / kKC) % NB);
        const int c = (int)(e / ((int64_t)kKC * NB));
        const int k = c * kKC + kk;
        float x = 0.f;
        if (k < K) x = transpose ? W[(int64_t)k * ldw + n] : W[(int64_t)n * ldw + k];
        float hi, lo;
        tc::split_tf32(x, hi, lo);
        uint8_t *base = img + (size_t)c * 2 * NB * 128;
        const uint32_t off = tc::sw128_off(n, kk);
        *reinterpret_cast<float *>(base + off) = hi;
        *reinterpret_cast<float *>(base + (size_t)NB * 128 + off) = lo;
    }
}

// ---------------------------------------------------------------- row GEMM kernel
struct Seg {
    const float *A;            // dense: n x K row-major (lda = K); nullptr => CBSR segment
    const float *hval;         // CBSR segment (densified on the fly)
    const uint8_t *hidx;
    int k;                     // CBSR k
    int K;                     // logical width
    int chunks;                // ceil(K / 32)
    int mask_mode;             // dense only: kMaskNone / kMaskM / kMaskNotM (columns of A)
};

struct TcRowsArgs {
    int64_t n;
    int N;                     // MMA N (output width)
    int G;                     // GEMMs (accumulators): 1 or 2
    int nseg[2];
    Seg seg[2][2];
    const uint8_t *bimg[2];    // packed B of each GEMM (segments back to back)
    const uint32_t *mask_in;   // merge mask for dense-segment masking
    int mask_words;
    int epi;                   // kEpiFwd / kEpiDz
    // forward epilogue
    const float *bias[2];
    int merge;
    float *y;
    uint32_t *mask_out;
    float *tap_a, *tap_b;
    // dz epilogue
    const float *crow;
    float *dz;
};

__device__ __forceinline__ void stage_dense(const Seg &s, int chunk, int64_t r0, int64_t n,
                                            const uint32_t *mask, int mw, float *hi, float *lo) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane & 7;                          // float4 index inside the 32-col chunk
    const int c0 = chunk * kKC + q * 4;
#pragma unroll 4
    for (int i = 0; i < 8; ++i) {
        const int r = warp * 32 + i * 4 + (lane >> 3);
        const int64_t row = r0 + r;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (row < n && c0 < s.K) {
            v = __ldg(reinterpret_cast<const float4 *>(s.A + row * s.K + c0));
            if (s.mask_mode != kMaskNone) {
                uint32_t bits = (__ldg(mask + row * mw + (c0 >> 5)) >> (c0 & 31)) & 0xfu;
                if (s.mask_mode == kMaskNotM) bits = ~bits;
                if (!(bits & 1u)) v.x = 0.f;
                if (!(bits & 2u)) v.y = 0.f;
                if (!(bits & 4u)) v.z = 0.f;
                if (!(bits & 8u)) v.w = 0.f;
            }
        }
        float4 h, l;
        tc::split_tf32(v.x, h.x, l.x);
        tc::split_tf32(v.y, h.y, l.y);
        tc::split_tf32(v.z, h.z, l.z);
        tc::split_tf32(v.w, h.w, l.w);
        const uint32_t off = tc::sw128_off(r, q * 4);
        *reinterpret_cast<float4 *>(reinterpret_cast<char *>(hi) + off) = h;
        *reinterpret_cast<float4 *>(reinterpret_cast<char *>(lo) + off) = l;
    }
}

__device__ __forceinline__ void stage_cbsr(const Seg &s, int chunk, int64_t r0, int64_t n,
                                           float *hi, float *lo) {
    const int r = threadIdx.x;                       // one row per thread
    char *hb = reinterpret_cast<char *>(hi), *lb = reinterpret_cast<char *>(lo);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4 *>(hb + r * 128 + q * 16) = z;
        *reinterpret_cast<float4 *>(lb + r * 128 + q * 16) = z;
    }
    const int64_t row = r0 + r;
    if (row >= n) return;
    const int lo_c = chunk * kKC;
    const float *hv = s.hval + row * s.k;
    const uint8_t *hi8 = s.hidx + row * s.k;
    if ((s.k & 3) == 0) {
        // 4 pairs per step: one 128-bit value load + one 32-bit index load, all issued first
        for (int t0 = 0; t0 < s.k; t0 += 16) {
            float4 v[4];
            uint32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (t0 + 4 * u < s.k) {
                    v[u] = __ldg(reinterpret_cast<const float4 *>(hv + t0 + 4 * u));
                    w[u] = __ldg(reinterpret_cast<const uint32_t *>(hi8 + t0 + 4 * u));
                } else {
                    w[u] = 0xffffffffu;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int c = (int)((w[u] >> (8 * b)) & 0xffu) - lo_c;
                    if (w[u] == 0xffffffffu || c < 0 || c >= kKC) continue;
                    float h, l;
                    tc::split_tf32(vv[b], h, l);
                    const uint32_t off = tc::sw128_off(r, c);
                    *reinterpret_cast<float *>(hb + off) = h;
                    *reinterpret_cast<float *>(lb + off) = l;
                }
            }
        }
        return;
    }
    for (int t = 0; t < s.k; ++t) {
        const int c = (int)__ldg(hi8 + t) - lo_c;
        if (c < 0 || c >= kKC) continue;
        float h, l;
        tc::split_tf32(__ldg(hv + t), h, l);
        const uint32_t off = tc::sw128_off(r, c);
        *reinterpret_cast<float *>(hb + off) = h;
        *reinterpret_cast<float *>(lb + off) = l;
    }
}

__global__ void __launch_bounds__(kThreadsTC, 1) tc_rows_kernel(TcRowsArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B align the dynamic smem base (swizzle atoms)
    uint8_t *sm = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int N = a.N;
    const uint32_t a_bytes = kTM * 128, b_bytes = (uint32_t)N * 128;
    const uint32_t stage_bytes = 2 * a_bytes + 2 * b_bytes;
    uint8_t *stage[2] = {sm, sm + stage_bytes};
    __shared__ __align__(8) uint64_t full_b[2], mma_done[2];
    __shared__ uint32_t tmem_base_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ncols_needed = (uint32_t)(a.G * N);
    uint32_t ncols = 32;
    while (ncols < ncols_needed) ncols <<= 1;

    if (tid == 0) {
        tc::mbar_init(&full_b[0], 1);
        tc::mbar_init(&full_b[1], 1);
        tc::mbar_init(&mma_done[0], 1);
        tc::mbar_init(&mma_done[1], 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) {
        tc::tmem_alloc(&tmem_base_slot, ncols);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base_slot;
    const uint32_t idesc = tc::idesc_tf32(kTM, N);
    const int64_t n_tiles = (a.n + kTM - 1) / kTM;
    uint32_t gstep = 0;

    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t r0 = tile * kTM;
        uint32_t last_stage = 0, last_use = 0;
        for (int g = 0; g < a.G; ++g) {
            int chunk_in_gemm = 0;
            for (int sgi = 0; sgi < a.nseg[g]; ++sgi) {
                const Seg &s = a.seg[g][sgi];
                for (int c = 0; c < s.chunks; ++c, ++chunk_in_gemm) {
                    const uint32_t st = gstep & 1u, use = gstep >> 1;
                    if (use >= 1) tc::mbar_wait(&mma_done[st], (use - 1) & 1u);
                    uint8_t *buf = stage[st];
                    float *ahi = reinterpret_cast<float *>(buf);
                    float *alo = reinterpret_cast<float *>(buf + a_bytes);
                    uint8_t *bhi = buf + 2 * a_bytes;
                    if (tid == 0) {
                        tc::mbar_arrive_expect_tx(&full_b[st], 2 * b_bytes);
                        tc::bulk_g2s(bhi, a.bimg[g] + (size_t)chunk_in_gemm * 2 * b_bytes,
                                     2 * b_bytes, &full_b[st]);
                    }
                    if (s.A) stage_dense(s, c, r0, a.n, a.mask_in, a.mask_words, ahi, alo);
                    else stage_cbsr(s, c, r0, a.n, ahi, alo);
                    tc::fence_async_smem();
                    __syncthreads();
                    if (tid == 0) {
                        tc::mbar_wait(&full_b[st], use & 1u);
                        tc::fence_after();
                        const uint32_t sa = tc::smem_u32(buf), sb = tc::smem_u32(bhi);
                        const uint32_t d = tmem + (uint32_t)(g * N);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks) {
                            const uint32_t ko = ks * 32;      // bytes: 8 fp32
                            const uint64_t ah = tc::desc_sw128(sa + ko);
                            const uint64_t al = tc::desc_sw128(sa + a_bytes + ko);
                            const uint64_t bh = tc::desc_sw128(sb + ko);
                            const uint64_t bl = tc::desc_sw128(sb + b_bytes + ko);
                            const uint32_t acc0 = (chunk_in_gemm > 0 || ks > 0) ? 1u : 0u;
                            tc::mma_tf32(d, ah, bh, idesc, acc0);
                            tc::mma_tf32(d, ah, bl, idesc, 1u);
                            tc::mma_tf32(d, al, bh, idesc, 1u);
                        }
                        tc::mma_commit(&mma_done[st]);
                    }
                    last_stage = st;
                    last_use = use;
                    ++gstep;
                }
            }
        }
        // ---- epilogue: wait for the tile's last MMAs, one TMEM lane (row) per thread
        tc::mbar_wait(&mma_done[last_stage], last_use & 1u);
        tc::fence_after();
        const int r = warp * 32 + lane;
        const int64_t row = r0 + r;
        const bool ok = row < a.n;
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        if (a.epi == kEpiDz) {
            const float cr = (ok && a.crow) ? __ldg(a.crow + row) : 1.f;
            for (int j = 0; j < N; j += 16) {
                float v[16];
                tc::tmem_ld16(tmem + lane_base + (uint32_t)j, v);
                if (ok) {
                    float4 *o = reinterpret_cast<float4 *>(a.dz + row * N + j);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        o[q] = make_float4(cr * v[4 * q], cr * v[4 * q + 1], cr * v[4 * q + 2],
                                           cr * v[4 * q + 3]);
                }
            }
        } else {
            const int mw = (N + 31) >> 5;
            uint32_t word = 0;
            for (int j = 0; j < N; j += 16) {
                float ya[16], yb[16];
                tc::tmem_ld16(tmem + lane_base + (uint32_t)j, ya);
                if (a.G == 2) tc::tmem_ld16(tmem + lane_base + (uint32_t)(N + j), yb);
                if (!ok) continue;
#pragma unroll
                for (int q = 0; q < 16; ++q) ya[q] += __ldg(a.bias[0] + j + q);
                float y[16];
                uint32_t bits = 0;
                if (a.G == 2) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        yb[q] += __ldg(a.bias[1] + j + q);
                        if (a.merge == DR_MERGE_MAX) {
                            const bool m = ya[q] >= yb[q];          // Eq. 14: ties -> near
                            y[q] = m ? ya[q] : yb[q];
                            bits |= (uint32_t)m << q;
                        } else {
                            y[q] = ya[q] + yb[q];
                        }
                    }
                    if (a.tap_a) {
                        float4 *o = reinterpret_cast<float4 *>(a.tap_a + row * N + j);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            o[q] = make_float4(ya[4 * q], ya[4 * q + 1], ya[4 * q + 2], ya[4 * q + 3]);
                    }
                    if (a.tap_b) {
                        float4 *o = reinterpret_cast<float4 *>(a.tap_b + row * N + j);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            o[q] = make_float4(yb[4 * q], yb[4 * q + 1], yb[4 * q + 2], yb[4 * q + 3]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 16; ++q) y[q] = ya[q];
                }
                if (a.y) {
                    float4 *o = reinterpret_cast<float4 *>(a.y + row * N + j);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        o[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
                }
                if (a.G == 2 && a.mask_out) {
                    word |= bits << (j & 16);
                    if ((j & 16) || j + 16 >= N) {
                        a.mask_out[row * mw + (j >> 5)] = word;
                        word = 0;
                    }
                }
            }
        }
        tc::fence_before();
        __syncthreads();
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}


// ---------------------------------------------------------------- dW = Z^T mask(dY) (row reduction)
// One CTA per contiguous row range; reduction chunks of 32 rows are the MMA K.
// A operand (M = 128 feature rows x 32 graph rows) stacks up to two segments
// (dense Z, densified CBSR) per accumulator group; B operand (N x 32) is
// mask(dY) transposed. Both are staged transposed by the threads (lane = graph
// row, conflict-free swizzled stores). db = colsum(mask(dY)) is accumulated in
// registers during staging. Per-CTA partials are summed in a fixed order by
// tc_reduce_parts_kernel (deterministic).
struct RSeg {
    const float *Z;            // dense n x w, or nullptr => CBSR (hval/hidx/k, dim w)
    const float *hval;
    const uint8_t *hidx;
    int k, w, m0;              // width and first feature row inside the group's M=128
};
struct TcReduceArgs {
    int64_t n;
    int N, G;
    int nseg[2];
    RSeg seg[2][2];
    const float *dy;
    const uint32_t *mask;
    int mask_mode;
    int64_t rows_per_cta;
    float *part;               // [grid][G*128*N + N]
};

__device__ __forceinline__ void stage_A_red(const RSeg &s, int64_t rb, int64_t re, float *hi,
                                            float *lo) {
    // warp w covers feature rows [32w, 32w+32) of the group tile; lane = graph row in chunk
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int f0 = warp * 32;                       // feature rows of this warp (tile coords)
    const int lo_f = max(f0, s.m0), hi_f = min(f0 + 32, s.m0 + s.w);
    if (lo_f >= hi_f) return;
    const int64_t row = rb + lane;
    const bool ok = row < re;
    char *hb = reinterpret_cast<char *>(hi), *lb = reinterpret_cast<char *>(lo);
    if (s.Z) {
        for (int m = lo_f; m < hi_f; ++m) {
            const float v = ok ? __ldg(s.Z + row * s.w + (m - s.m0)) : 0.f;
            float h, l;
            tc::split_tf32(v, h, l);
            const uint32_t off = tc::sw128_off(m, lane);
            *reinterpret_cast<float *>(hb + off) = h;
            *reinterpret_cast<float *>(lb + off) = l;
        }
    } else {
        for (int m = lo_f; m < hi_f; ++m) {
            const uint32_t off = tc::sw128_off(m, lane);
            *reinterpret_cast<float *>(hb + off) = 0.f;
            *reinterpret_cast<float *>(lb + off) = 0.f;
        }
        __syncwarp();
        if (ok) {
            for (int t = 0; t < s.k; ++t) {
                const int m = s.m0 + (int)__ldg(s.hidx + row * s.k + t);
                if (m < lo_f || m >= hi_f) continue;
                float h, l;
                tc::split_tf32(__ldg(s.hval + row * s.k + t), h, l);
                const uint32_t off = tc::sw128_off(m, lane);
                *reinterpret_cast<float *>(hb + off) = h;
                *reinterpret_cast<float *>(lb + off) = l;
            }
        }
    }
}

__global__ void __launch_bounds__(kThreadsTC, 1) tc_reduce_kernel(TcReduceArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int N = a.N, G = a.G;
    const uint32_t a_bytes = kTM * 128, b_bytes = (uint32_t)N * 128;
    const uint32_t stage_bytes = (uint32_t)G * 2 * a_bytes + 2 * b_bytes;
    uint8_t *stage[2] = {sm, sm + stage_bytes};
    __shared__ __align__(8) uint64_t mma_done[2];
    __shared__ uint32_t tmem_base_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(G * N)) ncols <<= 1;
    // zero both stages once: padded feature rows stay zero for the whole kernel
    for (uint32_t o = tid * 16; o < 2 * stage_bytes; o += kThreadsTC * 16)
        *reinterpret_cast<float4 *>(sm + o) = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
        tc::mbar_init(&mma_done[0], 1);
        tc::mbar_init(&mma_done[1], 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) {
        tc::tmem_alloc(&tmem_base_slot, ncols);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base_slot;
    const uint32_t idesc = tc::idesc_tf32(kTM, N);
    const int mw = (N + 31) >> 5;
    const int64_t rbeg = (int64_t)blockIdx.x * a.rows_per_cta;
    const int64_t rend = min(a.n, rbeg + a.rows_per_cta);
    float dbacc[64];                                 // column sums: warp's columns, this lane's rows
#pragma unroll
    for (int i = 0; i < 64; ++i) dbacc[i] = 0.f;
    uint32_t gstep = 0;
    for (int64_t rb = rbeg; rb < rend; rb += 32, ++gstep) {
        const uint32_t st = gstep & 1u, use = gstep >> 1;
        if (use >= 1) tc::mbar_wait(&mma_done[st], (use - 1) & 1u);
        uint8_t *buf = stage[st];
        for (int g = 0; g < G; ++g)
            for (int q = 0; q < a.nseg[g]; ++q)
                stage_A_red(a.seg[g][q], rb, rend, reinterpret_cast<float *>(buf + g * 2 * a_bytes),
                            reinterpret_cast<float *>(buf + g * 2 * a_bytes + a_bytes));
        {   // B: mask(dY) transposed; warp w covers columns [w*N/4, (w+1)*N/4)
            char *bh = reinterpret_cast<char *>(buf + G * 2 * a_bytes), *bl = bh + b_bytes;
            const int64_t row = rb + lane;
            const bool ok = row < rend;
            const int per = N >> 2, c0 = warp * per;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                if (i >= per) break;
                const int c = c0 + i;
                float v = ok ? __ldg(a.dy + row * N + c) : 0.f;
                if (ok && a.mask_mode != kMaskNone) {
                    const uint32_t b = (__ldg(a.mask + row * mw + (c >> 5)) >> (c & 31)) & 1u;
                    if ((a.mask_mode == kMaskM) != (b != 0u)) v = 0.f;
                }
                dbacc[i] += v;
                float h, l;
                tc::split_tf32(v, h, l);
                const uint32_t off = tc::sw128_off(c, lane);
                *reinterpret_cast<float *>(bh + off) = h;
                *reinterpret_cast<float *>(bl + off) = l;
            }
        }
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t sb = tc::smem_u32(buf + G * 2 * a_bytes);
            for (int g = 0; g < G; ++g) {
                const uint32_t sa = tc::smem_u32(buf + g * 2 * a_bytes);
                const uint32_t d = tmem + (uint32_t)(g * N);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t ko = ks * 32;
                    const uint64_t ah = tc::desc_sw128(sa + ko), al = tc::desc_sw128(sa + a_bytes + ko);
                    const uint64_t bh = tc::desc_sw128(sb + ko), bl = tc::desc_sw128(sb + b_bytes + ko);
                    const uint32_t acc0 = (rb > rbeg || ks > 0) ? 1u : 0u;
                    tc::mma_tf32(d, ah, bh, idesc, acc0);
                    tc::mma_tf32(d, ah, bl, idesc, 1u);
                    tc::mma_tf32(d, al, bh, idesc, 1u);
                }
            }
            tc::mma_commit(&mma_done[st]);
        }
    }
    float *out = a.part + (int64_t)blockIdx.x * ((int64_t)G * kTM * N + N);
    if (gstep > 0) {
        const uint32_t last = (gstep - 1) & 1u, luse = (gstep - 1) >> 1;
        tc::mbar_wait(&mma_done[last], luse & 1u);
        tc::fence_after();
        const int m = warp * 32 + lane;
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        for (int g = 0; g < G; ++g)
            for (int j = 0; j < N; j += 16) {
                float v[16];
                tc::tmem_ld16(tmem + lane_base + (uint32_t)(g * N + j), v);
                float4 *o = reinterpret_cast<float4 *>(out + ((int64_t)g * kTM + m) * N + j);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
    } else {
        for (int64_t e = tid; e < (int64_t)G * kTM * N; e += kThreadsTC) out[e] = 0.f;
    }
    {   // db partial: butterfly over the 32 lanes (rows) of each column, fixed order
        const int per = N >> 2, c0 = warp * per;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
            if (i >= per) break;
            float v = dbacc[i];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) out[(int64_t)G * kTM * N + c0 + i] = v;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// Sum per-CTA partials in a fixed order and scatter to the segment outputs.
struct RedOut {
    int nout;
    int g[4], m0[4], w[4];     // group, first feature row, width
    float *dst[4];
    float *db;
};
__global__ void tc_reduce_parts_kernel(const float *__restrict__ part, int nparts, int G, int N,
                                       RedOut o) {
    __shared__ float red[8][33];
    const int64_t len = (int64_t)G * kTM * N + N;
    const int64_t e = (int64_t)blockIdx.x * 32 + threadIdx.x;
    float acc = 0.f;
    if (e < len)
        for (int c = threadIdx.y; c < nparts; c += 8) acc += __ldg(part + (int64_t)c * len + e);
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y != 0 || e >= len) return;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x];
    if (e >= (int64_t)G * kTM * N) {
        if (o.db) o.db[e - (int64_t)G * kTM * N] = s;
        return;
    }
    const int g = (int)(e / ((int64_t)kTM * N));
    const int m = (int)((e / N) % kTM), c = (int)(e % N);
    for (int i = 0; i < o.nout; ++i)
        if (o.g[i] == g && m >= o.m0[i] && m < o.m0[i] + o.w[i])
            o.dst[i][(int64_t)(m - o.m0[i]) * N + c] = s;
}

}  // namespace

// ---------------------------------------------------------------- host side
size_t tc_bimg_bytes(int K, int NB) {
    return (size_t)((K + kKC - 1) / kKC) * 2 * NB * 128;
}

void launch_pack_b(const float *W, int ldw, int K, int NB, bool transpose, uint8_t *img,
                   cudaStream_t s) {
    const int64_t total = (int64_t)((K + kKC - 1) / kKC) * NB * kKC;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 592) blocks = 592;
    pack_b_kernel<<<(unsigned)blocks, 256, 0, s>>>(W, ldw, K, NB, transpose ? 1 : 0, img);
    note_launch("pack_b");
}


int tc_reduce_grid(int64_t n, int G, int N) {
    const size_t stage = (size_t)G * 2 * kTM * 128 + 2 * (size_t)N * 128;
    const int per_sm = 2 * stage + 1024 <= 110 * 1024 ? 2 : 1;
    int64_t grid = (n + 255) / 256;
    if (grid > 148 * per_sm) grid = 148 * per_sm;
    if (grid < 1) grid = 1;
    return (int)grid;
}

size_t tc_reduce_work_floats(int64_t n, int G, int N) {
    return (size_t)tc_reduce_grid(n, G, N) * ((size_t)G * kTM * N + N);
}

void launch_tc_reduce(const TcReduceDesc &d, float *work, cudaStream_t s) {
    TcReduceArgs a{};
    a.n = d.n;
    a.N = d.N;
    a.G = d.G;
    RedOut o{};
    for (int g = 0; g < d.G; ++g) {
        a.nseg[g] = d.nseg[g];
        int m0 = 0;
        for (int q = 0; q < d.nseg[g]; ++q) {
            const TcRedSegDesc &sd = d.seg[g][q];
            RSeg &r = a.seg[g][q];
            r.Z = sd.Z;
            r.hval = sd.hval;
            r.hidx = sd.hidx;
            r.k = sd.k;
            r.w = sd.w;
            r.m0 = m0;
            o.g[o.nout] = g;
            o.m0[o.nout] = m0;
            o.w[o.nout] = sd.w;
            o.dst[o.nout] = sd.grad;
            ++o.nout;
            m0 += sd.w;
        }
    }
    o.db = d.db;
    a.dy = d.dy;
    a.mask = d.mask;
    a.mask_mode = d.mask_mode;
    const int grid = tc_reduce_grid(d.n, d.G, d.N);
    a.rows_per_cta = ((d.n + grid - 1) / grid + 31) / 32 * 32;
    a.part = work;
    const size_t smem = 2 * ((size_t)d.G * 2 * kTM * 128 + 2 * (size_t)d.N * 128) + 1024;
    ProfScope ps("tc_dw", s);
    ensure_smem((const void *)tc_reduce_kernel, smem);
    tc_reduce_kernel<<<grid, kThreadsTC, smem, s>>>(a);
    note_launch("tc_reduce");
    const int64_t stride = (int64_t)d.G * kTM * d.N + d.N;
    tc_reduce_parts_kernel<<<(unsigned)((stride + 31) / 32), dim3(32, 8), 0, s>>>(work, grid, d.G,
                                                                                  d.N, o);
    note_launch("tc_reduce_parts");
}

bool tc_supported(int N) {
    const char *e = getenv("DR_DENSE_SIMT");      // A/B switch for tests and profiling
    const int off = e ? atoi(e) : 0;
    return !off && N >= 16 && N <= 256 && N % 16 == 0;
}

void launch_tc_rows(const TcRowsDesc &d, cudaStream_t s) {
    if (d.n <= 0) return;
    TcRowsArgs a{};
    a.n = d.n;
    a.N = d.N;
    a.G = d.G;
    for (int g = 0; g < d.G; ++g) {
        a.nseg[g] = d.nseg[g];
        a.bimg[g] = d.bimg[g];
        a.bias[g] = d.bias[g];
        for (int q = 0; q < d.nseg[g]; ++q) {
            const TcSegDesc &sd = d.seg[g][q];
            Seg &sg = a.seg[g][q];
            sg.A = sd.A;
            sg.hval = sd.hval;
            sg.hidx = sd.hidx;
            sg.k = sd.k;
            sg.K = sd.K;
            sg.chunks = (sd.K + kKC - 1) / kKC;
            sg.mask_mode = sd.mask_mode;
        }
    }
    a.mask_in = d.mask_in;
    a.mask_words = (d.mask_in_width + 31) / 32;
    a.epi = d.epi;
    a.merge = d.merge;
    a.y = d.y;
    a.mask_out = d.mask_out;
    a.tap_a = d.tap_a;
    a.tap_b = d.tap_b;
    a.crow = d.crow;
    a.dz = d.dz;
    const size_t smem = 2 * (2 * (size_t)kTM * 128 + 2 * (size_t)d.N * 128) + 1024;
    ensure_smem((const void *)tc_rows_kernel, smem);
    const int64_t tiles = (d.n + kTM - 1) / kTM;
    const int per_sm = smem <= 110 * 1024 ? 2 : 1;
    const int64_t grid = tiles < 148 * per_sm ? tiles : 148 * per_sm;
    ProfScope ps(d.epi == kEpiDz ? "tc_dz" : "tc_proj", s);
    tc_rows_kernel<<<(unsigned)grid, kThreadsTC, smem, s>>>(a);
    note_launch("tc_rows");
}

}  // namespace dr

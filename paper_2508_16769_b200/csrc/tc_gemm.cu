// tc_gemm.cu — tensor-core (tcgen05, kind::tf32) GEMMs for the dense parts of a
// HeteroConv layer: the per-module projections with the max-merge epilogue
// (Eq. 4 W^psi P:236-238, Eq. 8 / Eq. 14), the backward dZ = c (mask(dY) W^T)
// (Eq. 10-13) and the weight gradients dW = Z^T mask(dY), db = colsum(mask(dY)).
//
// Precision: the parity bar is 1e-4 (north_star); plain TF32 (10-bit mantissa)
// misses it, so every product is 3xTF32: a = a_hi + a_lo, b = b_hi + b_lo,
// a*b ~ a_hi*b_hi + a_hi*b_lo + a_lo*b_hi (error ~2^-22 relative).
//
// Pipeline (both kernels, 128 threads, persistent CTAs):
//   raw ring  : cp.async (LDGSTS) copies of the next kRaw-1 steps' fp32 inputs
//               land in shared memory while the current step is converted, so
//               global latency overlaps conversion, MMA and epilogue;
//   operands  : two stages of K-major SW128 tiles; threads convert raw fp32
//               into tf32 hi/lo (masking or densifying CBSR rows on the way);
//               the weight operand of the row GEMM arrives pre-split by one
//               cp.async.bulk (TMA engine) copy per chunk;
//   MMA       : thread 0 issues 3 (hi/lo pairs) x 4 (K=8 steps) tcgen05.mma per
//               32-wide K chunk into TMEM and commits to the stage's mbarrier;
//   epilogue  : one TMEM lane (row) per thread, tcgen05.ld 16 columns at a time.
#include "dr_internal.h"
#include "proj.h"
#include "tc.cuh"
#include "tc_gemm.h"

namespace dr {
namespace {

constexpr int kTM = 128;             // MMA M (rows of a tile / feature rows of dW)
constexpr int kKC = 32;              // K per chunk (one 128-B swizzle atom of fp32)
constexpr int kThreadsTC = 256;   // 8 warps: warps w and w+4 share TMEM lane quarter w%4
constexpr int kSmemMax = 227 * 1024 - 2048;   // opt-in limit minus static smem

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

__device__ __forceinline__ void store_split4(char *hi, char *lo, uint32_t off, float4 v) {
    float4 h, l;
    tc::split_tf32(v.x, h.x, l.x);
    tc::split_tf32(v.y, h.y, l.y);
    tc::split_tf32(v.z, h.z, l.z);
    tc::split_tf32(v.w, h.w, l.w);
    *reinterpret_cast<float4 *>(hi + off) = h;
    *reinterpret_cast<float4 *>(lo + off) = l;
}
__device__ __forceinline__ void store_split1(char *hi, char *lo, uint32_t off, float v) {
    float h, l;
    tc::split_tf32(v, h, l);
    *reinterpret_cast<float *>(hi + off) = h;
    *reinterpret_cast<float *>(lo + off) = l;
}

// Copy `bytes_valid` bytes of a contiguous block (16-B aligned) into smem with
// 16-B cp.async pieces spread over the CTA; the rest of `bytes_total` zero-filled.
__device__ __forceinline__ void cp_block(uint8_t *dst, const uint8_t *src, int64_t bytes_valid,
                                         int bytes_total) {
    for (int p = threadIdx.x; p * 16 < bytes_total; p += kThreadsTC) {
        const int64_t v = bytes_valid - (int64_t)p * 16;
        const uint32_t nb = v <= 0 ? 0u : (v >= 16 ? 16u : (uint32_t)v);
        tc::cp_async16(dst + p * 16, nb ? src + (int64_t)p * 16 : src, nb);
    }
}

// ================================================================= row GEMM
struct Seg {
    const float *A;            // dense: n x K row-major; nullptr => CBSR segment
    const float *hval;
    const uint8_t *hidx;
    int k, K, mask_mode;
};
struct Step {
    int8_t g, sg, c, cig;      // gemm, segment, chunk in segment, chunk in gemm
};
struct TcRowsArgs {
    int64_t n;
    int N, G, S;
    Step step[16];
    Seg seg[2][2];
    const uint8_t *bimg[2];
    const uint32_t *mask_in;
    int mask_words;
    int raw_bytes;
    int epi;
    const float *bias[2];
    int merge;
    float *y;
    uint32_t *mask_out;
    float *tap_a, *tap_b;
    const float *crow;
    float *dz;
};

// raw slot of a step: dense -> 128 rows x 128 B (+ 128 mask words at +16384);
// CBSR -> the tile's values (128*k fp32) then indices (128*k bytes)
__device__ __forceinline__ void rows_issue_raw(const TcRowsArgs &a, const Step &st, int64_t r0,
                                               uint8_t *raw) {
    const Seg &s = a.seg[st.g][st.sg];
    const int tid = threadIdx.x;
    if (s.A) {
#pragma unroll
        for (int i = 0; i < 1024 / kThreadsTC; ++i) {
            const int p = tid + kThreadsTC * i, r = p >> 3, q = p & 7;
            const int64_t row = r0 + r;
            const int col = st.c * kKC + q * 4;
            const bool ok = row < a.n && col < s.K;
            tc::cp_async16(raw + r * 128 + q * 16, ok ? (const void *)(s.A + row * s.K + col)
                                                      : (const void *)s.A, ok ? 16u : 0u);
        }
        if (s.mask_mode != kMaskNone && tid < kTM) {
            const int64_t row = r0 + tid;
            const bool ok = row < a.n;
            tc::cp_async4(raw + 16384 + tid * 4,
                          ok ? (const void *)(a.mask_in + row * a.mask_words + (st.c * kKC >> 5))
                             : (const void *)a.mask_in, ok ? 4u : 0u);
        }
    } else {
        const int64_t rows = a.n - r0 < kTM ? a.n - r0 : kTM;
        cp_block(raw, reinterpret_cast<const uint8_t *>(s.hval + r0 * s.k), rows * s.k * 4,
                 kTM * s.k * 4);
        cp_block(raw + kTM * s.k * 4, s.hidx + r0 * s.k, rows * s.k, kTM * s.k);
    }
}

__device__ __forceinline__ void rows_convert(const TcRowsArgs &a, const Step &st,
                                             const uint8_t *raw, char *hi, char *lo) {
    const Seg &s = a.seg[st.g][st.sg];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (s.A) {
        const int q = lane & 7;
        constexpr int RPW = kTM / (kThreadsTC / 32);          // rows per warp
#pragma unroll
        for (int i = 0; i < RPW / 4; ++i) {
            const int r = warp * RPW + i * 4 + (lane >> 3);
            float4 v = *reinterpret_cast<const float4 *>(raw + r * 128 + q * 16);
            if (s.mask_mode != kMaskNone) {
                const uint32_t w = *reinterpret_cast<const uint32_t *>(raw + 16384 + r * 4);
                uint32_t bits = (w >> (((st.c * kKC) & 31) + q * 4)) & 0xfu;
                if (s.mask_mode == kMaskNotM) bits = ~bits;
                if (!(bits & 1u)) v.x = 0.f;
                if (!(bits & 2u)) v.y = 0.f;
                if (!(bits & 4u)) v.z = 0.f;
                if (!(bits & 8u)) v.w = 0.f;
            }
            store_split4(hi, lo, tc::sw128_off(r, q * 4), v);
        }
    } else {
        // two threads per row: each zeroes half of the row, then (after a barrier)
        // scatters every other CBSR pair of the row
        const int r = tid & (kTM - 1), half = tid / kTM;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4 *>(hi + r * 128 + (half * 4 + q) * 16) = z;
            *reinterpret_cast<float4 *>(lo + r * 128 + (half * 4 + q) * 16) = z;
        }
        __syncthreads();
        const float *vals = reinterpret_cast<const float *>(raw) + r * s.k;
        const uint8_t *idx = raw + kTM * s.k * 4 + r * s.k;
        const int lo_c = st.c * kKC;
        for (int t = half; t < s.k; t += 2) {
            const int c = (int)idx[t] - lo_c;
            if (c >= 0 && c < kKC) store_split1(hi, lo, tc::sw128_off(r, c), vals[t]);
        }
    }
}

__device__ __forceinline__ void rows_epilogue(const TcRowsArgs &a, uint32_t tmem, int64_t r0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = a.N;
    const int quarter = warp & 3, half = warp >> 2;
    const int64_t row = r0 + quarter * 32 + lane;
    const bool ok = row < a.n;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    // column range of this warp: halves of N when both halves hold whole 32-col words
    const int jb = N >= 64 ? half * (N / 2) : 0, je = N >= 64 ? jb + N / 2 : (half ? 0 : N);
    if (a.epi == kEpiDz) {
        const float cr = (ok && a.crow) ? __ldg(a.crow + row) : 1.f;
        for (int j = jb; j < je; j += 16) {
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
        return;
    }
    const int mw = (N + 31) >> 5;
    uint32_t word = 0;
    for (int j = jb; j < je; j += 16) {
        float ya[16], yb[16];
        tc::tmem_ld16(tmem + lane_base + (uint32_t)j, ya);
        if (a.G == 2) tc::tmem_ld16(tmem + lane_base + (uint32_t)(N + j), yb);
        if (!ok) continue;
        float bias[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 b = __ldg(reinterpret_cast<const float4 *>(a.bias[0] + j) + q);
            bias[4 * q] = b.x; bias[4 * q + 1] = b.y; bias[4 * q + 2] = b.z; bias[4 * q + 3] = b.w;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) ya[q] += bias[q];
        float y[16];
        uint32_t bits = 0;
        if (a.G == 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 b = __ldg(reinterpret_cast<const float4 *>(a.bias[1] + j) + q);
                bias[4 * q] = b.x; bias[4 * q + 1] = b.y; bias[4 * q + 2] = b.z; bias[4 * q + 3] = b.w;
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                yb[q] += bias[q];
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
            if ((j & 16) || j + 16 >= je) {
                a.mask_out[row * mw + (j >> 5)] = word;
                word = 0;
            }
        }
    }
}

template <int kRaw>
__global__ void __launch_bounds__(kThreadsTC, 1) tc_rows_kernel(TcRowsArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int N = a.N;
    const uint32_t a_bytes = kTM * 128, b_bytes = (uint32_t)N * 128;
    const uint32_t op_bytes = 2 * a_bytes + 2 * b_bytes;
    uint8_t *ops[2] = {sm, sm + op_bytes};
    uint8_t *raws = sm + 2 * op_bytes;
    __shared__ __align__(8) uint64_t full_b[2], mma_done[2];
    __shared__ uint32_t tmem_base_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(a.G * N)) ncols <<= 1;
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
    const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t total = my_tiles * a.S;
    auto r0_of = [&](int64_t gs) { return ((int64_t)blockIdx.x + (gs / a.S) * gridDim.x) * kTM; };
    // prologue: raw for the first kRaw-1 steps
#pragma unroll
    for (int p = 0; p < kRaw - 1; ++p) {
        if (p < total) rows_issue_raw(a, a.step[p % a.S], r0_of(p), raws + p * a.raw_bytes);
        tc::cp_async_commit();
    }
    for (int64_t gs = 0; gs < total; ++gs) {
        const int sl = (int)(gs % a.S);
        const Step st = a.step[sl];
        const int64_t r0 = r0_of(gs);
        const uint32_t opi = (uint32_t)(gs & 1), use = (uint32_t)(gs >> 1);
        tc::cp_async_wait<kRaw - 2>();             // this step's raw copies have landed
        __syncthreads();                           // ... for every thread; previous raw slot free
        {
            const int64_t nx = gs + kRaw - 1;
            if (nx < total)
                rows_issue_raw(a, a.step[nx % a.S], r0_of(nx), raws + (nx % kRaw) * a.raw_bytes);
            tc::cp_async_commit();
        }
        if (use >= 1) tc::mbar_wait(&mma_done[opi], (use - 1) & 1u);
        uint8_t *op = ops[opi];
        uint8_t *bhi = op + 2 * a_bytes;
        if (tid == 0) {
            tc::mbar_arrive_expect_tx(&full_b[opi], 2 * b_bytes);
            tc::bulk_g2s(bhi, a.bimg[st.g] + (size_t)st.cig * 2 * b_bytes, 2 * b_bytes,
                         &full_b[opi]);
        }
        rows_convert(a, st, raws + (gs % kRaw) * a.raw_bytes, reinterpret_cast<char *>(op),
                     reinterpret_cast<char *>(op + a_bytes));
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::mbar_wait(&full_b[opi], use & 1u);
            tc::fence_after();
            const uint32_t sa = tc::smem_u32(op), sb = tc::smem_u32(bhi);
            const uint32_t d = tmem + (uint32_t)(st.g * N);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t ko = ks * 32;      // 8 fp32
                const uint64_t ah = tc::desc_sw128(sa + ko), al = tc::desc_sw128(sa + a_bytes + ko);
                const uint64_t bh = tc::desc_sw128(sb + ko), bl = tc::desc_sw128(sb + b_bytes + ko);
                const uint32_t acc0 = (st.cig > 0 || ks > 0) ? 1u : 0u;
                tc::mma_tf32(d, ah, bh, idesc, acc0);
                tc::mma_tf32(d, ah, bl, idesc, 1u);
                tc::mma_tf32(d, al, bh, idesc, 1u);
            }
            tc::mma_commit(&mma_done[opi]);
        }
        if (sl == a.S - 1) {
            tc::mbar_wait(&mma_done[opi], use & 1u);
            tc::fence_after();
            rows_epilogue(a, tmem, r0);
            tc::fence_before();
        }
    }
    tc::cp_async_wait<0>();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ================================================================= dW = Z^T mask(dY)
// One CTA per contiguous row range; each step is 32 graph rows = the MMA K.
// A (M = 128 feature rows x 32) stacks up to two segments per accumulator group
// (dense Z, densified CBSR); B (N x 32) is mask(dY) transposed. Raw rows land by
// cp.async, threads transpose + split them into the operand tiles (lane = feature
// or column, 32 graph rows each). db accumulates per lane in registers.
struct RSeg {
    const float *Z;            // dense n x w, or nullptr => CBSR (hval/hidx/k, dim w)
    const float *hval;
    const uint8_t *hidx;
    int k, w, m0;              // width, first feature row inside the group tile
    int raw_off;               // byte offset of this segment's rows in the raw slot
};
struct TcReduceArgs {
    int64_t n;
    int N, G;
    int nseg[2];
    RSeg seg[2][2];
    const float *dy;
    const uint32_t *mask;
    int mask_mode;
    int raw_bytes, raw_dy, raw_mask;
    int64_t rows_per_cta;
    float *part;               // [grid][G*128*N + N]
};

__device__ __forceinline__ void red_issue_raw(const TcReduceArgs &a, int64_t rb, int64_t re,
                                              uint8_t *raw) {
    const int64_t rows = re - rb < 32 ? re - rb : 32;
    for (int g = 0; g < a.G; ++g)
        for (int q = 0; q < a.nseg[g]; ++q) {
            const RSeg &s = a.seg[g][q];
            if (s.Z) {
                cp_block(raw + s.raw_off, reinterpret_cast<const uint8_t *>(s.Z + rb * s.w),
                         rows * s.w * 4, 32 * s.w * 4);
            } else {
                cp_block(raw + s.raw_off, reinterpret_cast<const uint8_t *>(s.hval + rb * s.k),
                         rows * s.k * 4, 32 * s.k * 4);
                cp_block(raw + s.raw_off + 32 * s.k * 4, s.hidx + rb * s.k, rows * s.k, 32 * s.k);
            }
        }
    cp_block(raw + a.raw_dy, reinterpret_cast<const uint8_t *>(a.dy + rb * a.N), rows * a.N * 4,
             32 * a.N * 4);
    if (a.mask_mode != kMaskNone) {
        const int mw = (a.N + 31) >> 5;
        cp_block(raw + a.raw_mask, reinterpret_cast<const uint8_t *>(a.mask + rb * mw),
                 rows * mw * 4, (32 * mw * 4 + 15) / 16 * 16);
    }
}

__device__ __forceinline__ void red_convert(const TcReduceArgs &a, const uint8_t *raw,
                                            uint8_t *op, float *dbacc) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t a_bytes = kTM * 128;
    // A groups: warp w owns feature rows [32(w%4), +32) and graph rows [16(w/4), +16);
    // lane = feature
    const int quarter = warp & 3, half = warp >> 2;
    for (int g = 0; g < a.G; ++g) {
        char *hi = reinterpret_cast<char *>(op + g * 2 * a_bytes), *lo = hi + a_bytes;
        const int f = quarter * 32 + lane;
        for (int q = 0; q < a.nseg[g]; ++q) {
            const RSeg &s = a.seg[g][q];
            if (f < s.m0 || f >= s.m0 + s.w) continue;
            const int fl = f - s.m0;
            if (s.Z) {
                const float *z = reinterpret_cast<const float *>(raw + s.raw_off);
#pragma unroll 8
                for (int rr = half * 16; rr < half * 16 + 16; ++rr)
                    store_split1(hi, lo, tc::sw128_off(f, rr), z[rr * s.w + fl]);
            } else {
#pragma unroll 8
                for (int rr = half * 16; rr < half * 16 + 16; ++rr)
                    store_split1(hi, lo, tc::sw128_off(f, rr), 0.f);
            }
        }
    }
    __syncthreads();                               // zeroed CBSR rows before the scatter
    for (int g = 0; g < a.G; ++g) {
        char *hi = reinterpret_cast<char *>(op + g * 2 * a_bytes), *lo = hi + a_bytes;
        for (int q = 0; q < a.nseg[g]; ++q) {
            const RSeg &s = a.seg[g][q];
            if (s.Z || warp != 0) continue;        // warp 0 scatters: lane = graph row
            const float *vals = reinterpret_cast<const float *>(raw + s.raw_off) + lane * s.k;
            const uint8_t *idx = raw + s.raw_off + 32 * s.k * 4 + lane * s.k;
            for (int t = 0; t < s.k; ++t)
                store_split1(hi, lo, tc::sw128_off(s.m0 + idx[t], lane), vals[t]);
        }
    }
    // B: lane = column, loop over the 32 graph rows
    {
        char *hi = reinterpret_cast<char *>(op + a.G * 2 * a_bytes);
        char *lo = hi + a.N * 128;
        const float *dy = reinterpret_cast<const float *>(raw + a.raw_dy);
        const uint32_t *mk = reinterpret_cast<const uint32_t *>(raw + a.raw_mask);
        const int mw = (a.N + 31) >> 5;
        for (int i = 0; i < 2; ++i) {
            const int c = (quarter + 4 * i) * 32 + lane;  // columns covered by this thread
            if (c >= a.N) break;
            float s = 0.f;
#pragma unroll 8
            for (int rr = half * 16; rr < half * 16 + 16; ++rr) {
                float v = dy[rr * a.N + c];
                if (a.mask_mode != kMaskNone) {
                    const uint32_t b = (mk[rr * mw + (c >> 5)] >> (c & 31)) & 1u;
                    if ((a.mask_mode == kMaskM) != (b != 0u)) v = 0.f;
                }
                s += v;
                store_split1(hi, lo, tc::sw128_off(c, rr), v);
            }
            dbacc[i] += s;
        }
    }
}

template <int kRaw>
__global__ void __launch_bounds__(kThreadsTC, 1) tc_reduce_kernel(TcReduceArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int N = a.N, G = a.G;
    const uint32_t a_bytes = kTM * 128, b_bytes = (uint32_t)N * 128;
    const uint32_t op_bytes = (uint32_t)G * 2 * a_bytes + 2 * b_bytes;
    uint8_t *ops[2] = {sm, sm + op_bytes};
    uint8_t *raws = sm + 2 * op_bytes;
    __shared__ __align__(8) uint64_t mma_done[2];
    __shared__ uint32_t tmem_base_slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(G * N)) ncols <<= 1;
    // zero both operand stages once: padded feature rows stay zero
    for (uint32_t o = tid * 16; o < 2 * op_bytes; o += kThreadsTC * 16)
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
    const int64_t rbeg = (int64_t)blockIdx.x * a.rows_per_cta;
    const int64_t rend = a.n < rbeg + a.rows_per_cta ? a.n : rbeg + a.rows_per_cta;
    const int64_t total = rend > rbeg ? (rend - rbeg + 31) / 32 : 0;
    float dbacc[2] = {0.f, 0.f};
#pragma unroll
    for (int p = 0; p < kRaw - 1; ++p) {
        if (p < total) red_issue_raw(a, rbeg + 32 * p, rend, raws + p * a.raw_bytes);
        tc::cp_async_commit();
    }
    for (int64_t gs = 0; gs < total; ++gs) {
        const uint32_t opi = (uint32_t)(gs & 1), use = (uint32_t)(gs >> 1);
        tc::cp_async_wait<kRaw - 2>();
        __syncthreads();
        {
            const int64_t nx = gs + kRaw - 1;
            if (nx < total)
                red_issue_raw(a, rbeg + 32 * nx, rend, raws + (nx % kRaw) * a.raw_bytes);
            tc::cp_async_commit();
        }
        if (use >= 1) tc::mbar_wait(&mma_done[opi], (use - 1) & 1u);
        uint8_t *op = ops[opi];
        red_convert(a, raws + (gs % kRaw) * a.raw_bytes, op, dbacc);
        tc::fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc::fence_after();
            const uint32_t sb = tc::smem_u32(op + G * 2 * a_bytes);
            for (int g = 0; g < G; ++g) {
                const uint32_t sa = tc::smem_u32(op + g * 2 * a_bytes);
                const uint32_t d = tmem + (uint32_t)(g * N);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t ko = ks * 32;
                    const uint64_t ah = tc::desc_sw128(sa + ko), al = tc::desc_sw128(sa + a_bytes + ko);
                    const uint64_t bh = tc::desc_sw128(sb + ko), bl = tc::desc_sw128(sb + b_bytes + ko);
                    const uint32_t acc0 = (gs > 0 || ks > 0) ? 1u : 0u;
                    tc::mma_tf32(d, ah, bh, idesc, acc0);
                    tc::mma_tf32(d, ah, bl, idesc, 1u);
                    tc::mma_tf32(d, al, bh, idesc, 1u);
                }
            }
            tc::mma_commit(&mma_done[opi]);
        }
    }
    tc::cp_async_wait<0>();
    float *out = a.part + (int64_t)blockIdx.x * ((int64_t)G * kTM * N + N);
    const int quarter = warp & 3, half = warp >> 2;
    if (total > 0) {
        const uint32_t last = (uint32_t)((total - 1) & 1), luse = (uint32_t)((total - 1) >> 1);
        tc::mbar_wait(&mma_done[last], luse & 1u);
        tc::fence_after();
        const int m = quarter * 32 + lane;
        const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
        const int jb = N >= 32 ? half * (N / 2) : 0, je = N >= 32 ? jb + N / 2 : (half ? 0 : N);
        for (int g = 0; g < G; ++g)
            for (int j = jb; j < je; j += 16) {
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
    {   // db partial: the two row halves of each column, added in a fixed order
        __shared__ float dbs[2][256];
        for (int i = 0; i < 2; ++i) {
            const int c = (quarter + 4 * i) * 32 + lane;
            if (c < N) dbs[half][c] = dbacc[i];
        }
        __syncthreads();
        for (int c = tid; c < N; c += kThreadsTC) out[(int64_t)G * kTM * N + c] = dbs[0][c] + dbs[1][c];
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

size_t rows_smem(int N, int raw_bytes, int depth) {
    return 2 * (2 * (size_t)kTM * 128 + 2 * (size_t)N * 128) + (size_t)depth * raw_bytes + 1024;
}

struct RedLayout {
    int raw_bytes, raw_dy, raw_mask;
    size_t smem;
};
RedLayout red_layout(const TcReduceDesc &d, int offs[2][2]) {
    RedLayout L{};
    int off = 0;
    for (int g = 0; g < d.G; ++g)
        for (int q = 0; q < d.nseg[g]; ++q) {
            const TcRedSegDesc &s = d.seg[g][q];
            offs[g][q] = off;
            off += s.Z ? 32 * s.w * 4 : (32 * s.k * 4 + (32 * s.k + 15) / 16 * 16);
            off = (off + 15) / 16 * 16;
        }
    L.raw_dy = off;
    off += 32 * d.N * 4;
    L.raw_mask = off;
    off += (32 * ((d.N + 31) / 32) * 4 + 15) / 16 * 16;
    L.raw_bytes = (off + 127) / 128 * 128;
    L.smem = 2 * ((size_t)d.G * 2 * kTM * 128 + 2 * (size_t)d.N * 128) + 1024;
    return L;
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

static int per_sm_for(size_t smem) {
    return smem <= 75 * 1024 ? 3 : smem <= 112 * 1024 ? 2 : 1;
}

static int tc_reduce_grid(int64_t n, size_t smem) {
    int64_t grid = (n + 255) / 256;
    const int64_t cap = 148 * per_sm_for(smem);
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    return (int)grid;
}

size_t tc_reduce_work_floats(int64_t n, int G, int N) {
    return (size_t)(148 * 3) * ((size_t)G * kTM * N + N) + 0 * n;
}

void launch_tc_reduce(const TcReduceDesc &d, float *work, cudaStream_t s) {
    TcReduceArgs a{};
    a.n = d.n;
    a.N = d.N;
    a.G = d.G;
    int offs[2][2] = {{0, 0}, {0, 0}};
    const RedLayout lay = red_layout(d, offs);
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
            r.raw_off = offs[g][q];
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
    a.raw_bytes = lay.raw_bytes;
    a.raw_dy = lay.raw_dy;
    a.raw_mask = lay.raw_mask;
    const int grid = tc_reduce_grid(d.n, lay.smem + 3 * (size_t)lay.raw_bytes);
    a.rows_per_cta = ((d.n + grid - 1) / grid + 31) / 32 * 32;
    a.part = work;
    ProfScope ps("tc_dw", s);
    const size_t smem3 = lay.smem + 3 * (size_t)lay.raw_bytes, smem2 = lay.smem + 2 * (size_t)lay.raw_bytes;
    DR_CHECK(smem2 <= kSmemMax, DR_ERR_UNSUPPORTED, "tc_reduce: shared memory budget");
    if (smem3 <= kSmemMax) {
        ensure_smem((const void *)tc_reduce_kernel<3>, smem3);
        tc_reduce_kernel<3><<<grid, kThreadsTC, smem3, s>>>(a);
    } else {
        ensure_smem((const void *)tc_reduce_kernel<2>, smem2);
        tc_reduce_kernel<2><<<grid, kThreadsTC, smem2, s>>>(a);
    }
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
    int raw = 16384 + 512;
    a.S = 0;
    for (int g = 0; g < d.G; ++g) {
        a.bimg[g] = d.bimg[g];
        a.bias[g] = d.bias[g];
        int cig = 0;
        for (int q = 0; q < d.nseg[g]; ++q) {
            const TcSegDesc &sd = d.seg[g][q];
            Seg &sg = a.seg[g][q];
            sg.A = sd.A;
            sg.hval = sd.hval;
            sg.hidx = sd.hidx;
            sg.k = sd.k;
            sg.K = sd.K;
            sg.mask_mode = sd.mask_mode;
            if (!sd.A) {
                const int need = kTM * sd.k * 5;
                if (need > raw) raw = need;
            }
            const int chunks = (sd.K + kKC - 1) / kKC;
            for (int c = 0; c < chunks; ++c) {
                DR_CHECK(a.S < 16, DR_ERR_UNSUPPORTED, "tc_rows: too many K chunks");
                a.step[a.S++] = Step{(int8_t)g, (int8_t)q, (int8_t)c, (int8_t)cig++};
            }
        }
    }
    a.raw_bytes = (raw + 127) / 128 * 128;
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
    const size_t smem3 = rows_smem(d.N, a.raw_bytes, 3), smem2 = rows_smem(d.N, a.raw_bytes, 2);
    DR_CHECK(smem2 <= kSmemMax, DR_ERR_UNSUPPORTED, "tc_rows: shared memory budget");
    const size_t smem = smem3 <= kSmemMax ? smem3 : smem2;
    const int64_t tiles = (d.n + kTM - 1) / kTM;
    const int64_t cap = 148 * per_sm_for(smem);
    const int64_t grid = tiles < cap ? tiles : cap;
    ProfScope ps(d.epi == kEpiDz ? "tc_dz" : "tc_proj", s);
    if (smem3 <= kSmemMax) {
        ensure_smem((const void *)tc_rows_kernel<3>, smem);
        tc_rows_kernel<3><<<(unsigned)grid, kThreadsTC, smem, s>>>(a);
    } else {
        ensure_smem((const void *)tc_rows_kernel<2>, smem);
        tc_rows_kernel<2><<<(unsigned)grid, kThreadsTC, smem, s>>>(a);
    }
    note_launch("tc_rows");
}

}  // namespace dr

// tc2.cu — warp-specialised tcgen05 GEMMs for the dense parts of a HeteroConv
// layer (see tc2.h for the math and the precision argument).
//
// Row GEMM (one persistent CTA per SM, 10 warps):
//   warp 0      producer : per (tile, K chunk) step, 1-D bulk copies (TMA engine) of
//                          the 128 rows x 64 fp32 of the chunk (or the tile's CBSR
//                          rows) and the merge-mask words into a stage; packed B
//                          chunks into a ring (or once, when all fit: resident B);
//   warps 2-5   converters: split the raw fp32 stage IN PLACE into the bf16 hi / lo
//                          K-major SW128 operand tiles (masking, zero-padding,
//                          densifying CBSR rows on the way);
//   warp 1      MMA      : one thread issues 3 kind::f16 MMAs per K=16 step into a
//                          double-buffered TMEM accumulator, commits to the stage /
//                          B slot / accumulator barriers;
//   warps 6-9   epilogue : TMEM -> registers (one row per thread), bias, max-merge
//                          + mask bits (Eq. 8, 14), taps, or the dz row scale and the
//                          root-term sampling, then global stores.
// Reduce GEMM (dW = A^T mask(dY)): 6 warps, same producer / MMA roles; the four
// converter warps transpose 64-row stages into [feature][row] and [col][row]
// operands, accumulate db, and read the final TMEM accumulator out as per-CTA
// partials that a second kernel sums in a fixed order (deterministic, no atomics).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "dr_internal.h"
#include "proj.h"
#include "tc.cuh"
#include "tc2.h"
#include "drelu_net.cuh"

namespace dr {
namespace {

constexpr int kTile = 128;             // rows per tile = MMA M
constexpr int kChunk = 64;             // bf16 K per chunk (one 128-B swizzle atom)
constexpr uint32_t kStage = 32768;     // 128 x 64 fp32 raw == bf16 hi + lo tiles
constexpr uint32_t kHalf = 16384;      // one bf16 128 x 64 tile
constexpr int kMaskStage = 4096;       // 128 rows x up to 8 mask words
// row GEMM roles. W2 = false (10 warps, 168 registers each): producer, MMA issuer,
// 4 converter warps, 4 epilogue warps. W2 = true (16 warps, 4 aligned warpgroups
// with their own register budgets, setmaxnreg): WG0 converters (128), WG1 producer
// + MMA issuer + 2 idle warps (40), WG2 / WG3 two epilogue warpgroups (168 each)
// taking alternate tiles (the two TMEM accumulators), so a latency-bound epilogue
// (one warp per SM sub-partition otherwise) runs two deep.
template <bool W2> struct RowsRoles {
    static constexpr int threads = W2 ? 512 : 320;
    static constexpr int conv0 = W2 ? 0 : 2;       // first of the 4 converter warps
    static constexpr int prod = W2 ? 4 : 0;
    static constexpr int mma = W2 ? 5 : 1;
    static constexpr int epi0 = W2 ? 8 : 6;        // first epilogue warp
    static constexpr int nepi = W2 ? 8 : 4;
};
constexpr int kRedThreads = 320;     // producer, MMA, 2 x 4 converter warps
constexpr int kEpiWarp0 = 32 * 36 * 4;                // epilogue staging per warp: [32][36] fp32
constexpr int kEpiWarpN = 32 * 68 * 4;                // ... with the fused D-ReLU: [32][kRB] row buffer
constexpr int kSmemBase = 227 * 1024 - 1024 - 4096;   // opt-in max minus alignment, static smem
__host__ __device__ constexpr int epi_warp_bytes(bool next) { return next ? kEpiWarpN : kEpiWarp0; }
constexpr int kSmemBudgetRed = 227 * 1024 - 1024 - 10240 - 1024;  // reduce kernel: ~10 KB static
constexpr int kMaxSteps = 16;
constexpr int kMaxSA = 4, kMaxSB = 16;

__device__ __forceinline__ float4 lds4(const uint8_t *p) { return *reinterpret_cast<const float4 *>(p); }

// ================================================================= B packing
// chunk c of the image: hi = Ntot rows x 128 B, then lo; element (n, kk) of the
// operand at sw128_off_h(n, kk - 64c).
__global__ void tc2_pack_b_kernel(const float *__restrict__ W, int ldw, int K, int NB, int n0,
                                  int Ntot, int transpose, uint8_t *__restrict__ img) {
    const int chunks = (K + kChunk - 1) / kChunk;
    const int64_t total = (int64_t)chunks * NB * (kChunk / 2);      // element pairs
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int kp = (int)(e % (kChunk / 2));
        const int n = (int)((e / (kChunk / 2)) % NB);
        const int c = (int)(e / ((int64_t)(kChunk / 2) * NB));
        const int k0 = c * kChunk + 2 * kp;
        float v[2];
        for (int q = 0; q < 2; ++q) {
            const int k = k0 + q;
            v[q] = k < K ? (transpose ? W[(int64_t)k * ldw + n] : W[(int64_t)n * ldw + k]) : 0.f;
        }
        uint32_t hi, lo;
        tc::split_bf16x2(v[0], v[1], hi, lo);
        uint8_t *base = img + (size_t)c * 2 * Ntot * 128;
        const uint32_t off = tc::sw128_off_h((uint32_t)(n0 + n), (uint32_t)(2 * kp));
        *reinterpret_cast<uint32_t *>(base + off) = hi;
        *reinterpret_cast<uint32_t *>(base + (size_t)Ntot * 128 + off) = lo;
    }
}

// several images in one launch (blockIdx.y = job): a layer's forward or
// backward packs all its weights at once instead of one launch per weight
struct PackJobs {
    Tc2PackJob job[kMaxPackJobs];
};
__global__ void tc2_pack_b_multi_kernel(const __grid_constant__ PackJobs j) {
    const Tc2PackJob &p = j.job[blockIdx.y];
    const int chunks = (p.K + kChunk - 1) / kChunk;
    const int64_t total = (int64_t)chunks * p.NB * (kChunk / 2);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int kp = (int)(e % (kChunk / 2));
        const int n = (int)((e / (kChunk / 2)) % p.NB);
        const int c = (int)(e / ((int64_t)(kChunk / 2) * p.NB));
        const int k0 = c * kChunk + 2 * kp;
        float v[2];
        for (int q = 0; q < 2; ++q) {
            const int k = k0 + q;
            v[q] = k < p.K ? (p.transpose ? p.W[(int64_t)k * p.ldw + n] : p.W[(int64_t)n * p.ldw + k]) : 0.f;
        }
        uint32_t hi, lo;
        tc::split_bf16x2(v[0], v[1], hi, lo);
        uint8_t *base = p.img + (size_t)c * 2 * p.Ntot * 128;
        const uint32_t off = tc::sw128_off_h((uint32_t)(p.n0 + n), (uint32_t)(2 * kp));
        *reinterpret_cast<uint32_t *>(base + off) = hi;
        *reinterpret_cast<uint32_t *>(base + (size_t)p.Ntot * 128 + off) = lo;
    }
}

// ================================================================= row GEMM
#define RDBG_T0 const long long dbg_t0 = a.dbg ? clock64() : 0
#define RDBG_ADD(slot) do { if (a.dbg) atomicAdd(a.dbg + blockIdx.x * 16 + (slot), (unsigned long long)(clock64() - dbg_t0)); } while (0)
struct R2Step {
    int8_t g, s, c, bc, first;     // group, segment, chunk in segment, chunk in group image, first of group
};
struct R2Seg {
    const float *A;
    const float *hval;
    const uint8_t *hidx;
    int k, K, mask_mode;
    int split;                     // A rows are [hi | lo] bf16: TMA lands the operand directly
};
struct R2Args {
    CUtensorMap tmap[2][2];        // dense segments: [n x K] fp32, box 64 cols x 128 rows
    int64_t n;
    int N, G, S;
    R2Step step[kMaxSteps];
    R2Seg seg[2][2];
    const uint8_t *bimg[2];
    const uint32_t *mask_in;
    int mw;
    int SA, SB, b_resident;
    int ewg;                       // epilogue warpgroups (1 or 2; smem permitting)
    uint32_t bchunk;               // bytes of one packed B chunk (hi + lo)
    uint32_t epi_off;              // byte offset of the epilogue staging boxes
    int epi;
    const float *bias[2];
    int merge;
    float *y;
    uint32_t *mask_out;
    float *tap_a, *tap_b;
    int n_dz;
    int dz_split;
    const float *crow;
    float *dz;
    const uint8_t *root_idx;
    int root_k;
    float *root;
    // fused linear head + MSE (last layer; tc2.h)
    int head;
    const float *head_w, *head_b, *labels;
    float head_inv_n;
    float *head_dy, *head_part;
    // fused next-layer D-ReLU (row a5): CBSR of y, exactly nk per row (tc2.h)
    int nk;                        // keep count (0: no fused D-ReLU)
    int nk_stream;                 // rolled-chunk network (knob tpr_stream)
    float *nval;
    uint8_t *nidx;
    unsigned long long *dbg;       // DR_TC2_DEBUG role timers, else null
};

__host__ __device__ __forceinline__ uint32_t rup16(uint32_t x) { return (x + 15u) & ~15u; }

// producer: one step's raw data into stage `st`, signalled on `full`
__device__ __forceinline__ void rows_produce(const R2Args &a, const R2Step &sp, int64_t r0,
                                             uint8_t *st, uint8_t *mk, uint64_t *full, int lane) {
    const R2Seg &s = a.seg[sp.g][sp.s];
    const int rows = (int)(a.n - r0 < kTile ? a.n - r0 : kTile);
    if (s.A && s.split) {
        // split rows: the hi and lo 128 x 64 bf16 boxes arrive 128-B swizzled, i.e.
        // already the K-major SW128 operand tiles (no converter work)
        if (lane == 0) {
            tc::mbar_arrive_expect_tx(full, kStage);
            tc::tma_load_2d(st, &a.tmap[sp.g][sp.s], sp.c * kChunk, (int)r0, full);
            tc::tma_load_2d(st + kHalf, &a.tmap[sp.g][sp.s], s.K + sp.c * kChunk, (int)r0, full);
        }
    } else if (s.A) {
        // one TMA box: rows r0..r0+127, columns 64c..64c+63 (out-of-range rows and
        // columns arrive as zeros), plus the tile's merge-mask words
        const uint32_t mbytes = s.mask_mode != kMask2None ? rup16((uint32_t)rows * a.mw * 4) : 0u;
        if (lane == 0) {
            tc::mbar_arrive_expect_tx(full, kStage + mbytes);
            tc::tma_load_2d(st, &a.tmap[sp.g][sp.s], sp.c * kChunk, (int)r0, full);
            if (mbytes) tc::bulk_g2s(mk, a.mask_in + r0 * a.mw, mbytes, full);
        }
    } else {
        // CBSR rows of the tile: values at +0, indices at +kHalf (both contiguous);
        // sizes rounded up to 16 B (the tape pads every buffer)
        const uint32_t vb = rup16((uint32_t)rows * s.k * 4), ib = rup16((uint32_t)rows * s.k);
        if (lane == 0) {
            tc::mbar_arrive_expect_tx(full, vb + ib);
            tc::bulk_g2s(st, s.hval + r0 * s.k, vb, full);
            tc::bulk_g2s(st + kHalf, s.hidx + r0 * s.k, ib, full);
        }
    }
}

// converters (128 threads, ct = 0..127): raw stage -> hi (+0) / lo (+kHalf) in place
__device__ __forceinline__ void rows_convert(const R2Args &a, const R2Step &sp, int64_t r0,
                                             uint8_t *st, const uint8_t *mk, int ct) {
    const R2Seg &s = a.seg[sp.g][sp.s];
    const int lane = ct & 31, cw = ct >> 5;
    if (s.A && s.split) return;                        // landed as operand tiles
    if (s.A) {
        const int q = lane & 15;                       // float4 column group of the chunk
        float4 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int r = cw * 32 + 2 * i + (lane >> 4);
            v[i] = lds4(st + r * 256 + q * 16);
        }
        uint32_t mbits[16];
        if (s.mask_mode != kMask2None) {
            const int col = sp.c * kChunk + 4 * q;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int r = cw * 32 + 2 * i + (lane >> 4);
                const uint32_t w = *reinterpret_cast<const uint32_t *>(mk + (r * a.mw + (col >> 5)) * 4);
                uint32_t b = (w >> (col & 31)) & 0xfu;
                if (s.mask_mode == kMask2NotM) b = ~b & 0xfu;
                mbits[i] = b;
            }
        }
        tc::named_bar(1, 128);                         // every raw read precedes any write
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int r = cw * 32 + 2 * i + (lane >> 4);
            float4 x = v[i];                           // TMA zero-filled rows >= n, cols >= K
            if (s.mask_mode != kMask2None) {
                const uint32_t b = mbits[i];
                if (!(b & 1u)) x.x = 0.f;
                if (!(b & 2u)) x.y = 0.f;
                if (!(b & 4u)) x.z = 0.f;
                if (!(b & 8u)) x.w = 0.f;
            }
            uint2 h, l;
            tc::split_bf16x2(x.x, x.y, h.x, l.x);
            tc::split_bf16x2(x.z, x.w, h.y, l.y);
            const uint32_t off = tc::sw128_off_h((uint32_t)r, (uint32_t)(4 * q));
            *reinterpret_cast<uint2 *>(st + off) = h;
            *reinterpret_cast<uint2 *>(st + kHalf + off) = l;
        }
    } else {
        // CBSR chunk: thread ct reads float4 groups e4 = ct + 128 i of the tile's
        // contiguous values (and the 4 matching index bytes), conflict-free; after
        // a barrier the whole operand is zeroed, after a second one each thread
        // scatters its entries whose index falls in this chunk's 64 columns
        const int k = s.k, nv4 = 32 * k;               // 128 k entries / 4
        int lk = 0;
        while ((1 << lk) < k) ++lk;
        float4 vq[8];
        uint32_t iq[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e4 = ct + 128 * i;
            if (e4 < nv4) {
                vq[i] = lds4(st + 16 * e4);
                iq[i] = *reinterpret_cast<const uint32_t *>(st + kHalf + 4 * e4);
            }
        }
        tc::named_bar(1, 128);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 16; ++i) *reinterpret_cast<float4 *>(st + 16 * (ct + 128 * i)) = z;
        tc::named_bar(1, 128);
        const int lo_c = sp.c * kChunk;
        const int rows = (int)(a.n - r0 < kTile ? a.n - r0 : kTile);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int e4 = ct + 128 * i;
            if (e4 >= nv4) continue;
            const float vv[4] = {vq[i].x, vq[i].y, vq[i].z, vq[i].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = 4 * e4 + q, r = e >> lk;
                const int col = (int)((iq[i] >> (8 * q)) & 0xffu) - lo_c;
                if (r < rows && col >= 0 && col < kChunk) {
                    uint32_t h, l;
                    tc::split_bf16x2(vv[q], 0.f, h, l);
                    const uint32_t off = tc::sw128_off_h((uint32_t)r, (uint32_t)col);
                    *reinterpret_cast<uint16_t *>(st + off) = (uint16_t)(h & 0xffffu);
                    *reinterpret_cast<uint16_t *>(st + kHalf + off) = (uint16_t)(l & 0xffffu);
                }
            }
        }
    }
}


// epilogue warp (quarter qd): rows r0 + 32 qd + lane of accumulator columns at `acc`
// Epilogue staging: per warp a [32 rows][32 columns] fp32 tile (row stride 36
// floats: conflict-free 128-bit row writes and column-quad reads). A block of
// 32 accumulator columns goes TMEM -> registers (lane = row) -> staging ->
// coalesced stores (lane -> row 4 i + lane / 8, column quad lane % 8: each
// instruction writes 4 rows x 128 B). No asynchronous store state to wait on.
constexpr int kEStg = 36;
__device__ __forceinline__ void stg_put(float *stg, int stride, int lane, const float *v) {
    float4 *o = reinterpret_cast<float4 *>(stg + lane * stride);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}
// rows row0 .. row0 + 31 (< n) of an fp32 [n x W] matrix, columns [j, j + 32)
__device__ __forceinline__ void stg_out_f32(const float *stg, int stride, float *out, int64_t W,
                                            int64_t row0, int64_t n, int j, int lane) {
    const int cq = lane & 7, rs = lane >> 3;
    // one 64-bit base and one bound per lane; rows rs, rs + 4, ... are W float4 apart
    if (j + 4 * cq >= W) return;
    const int64_t left = n - row0 - rs;
    float4 *p = reinterpret_cast<float4 *>(out + (row0 + rs) * W + j) + cq;
    const float *sp = stg + rs * stride + 4 * cq;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 v = *reinterpret_cast<const float4 *>(sp + 4 * i * stride);
        if (4 * i < left) __stcs(p + (int64_t)i * W, v);
    }
}
// split output ([hi | lo] bf16 rows of 2 W halves): hi at column j, lo at W + j
__device__ __forceinline__ void stg_out_split(const float *stg, uint8_t *out, int64_t W, int64_t row0,
                                              int64_t n, int j, int lane) {
    const int cq = lane & 7, rs = lane >> 3;
    if (j + 4 * cq >= W) return;
    const int64_t left = n - row0 - rs;
    uint8_t *rp = out + (row0 + rs) * W * 4 + 2 * (j + 4 * cq);    // hi piece; lo at + 2 W
    const float *sp = stg + rs * kEStg + 4 * cq;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 v = *reinterpret_cast<const float4 *>(sp + 4 * i * kEStg);
        uint2 h, l;
        tc::split_bf16x2(v.x, v.y, h.x, l.x);
        tc::split_bf16x2(v.z, v.w, h.y, l.y);
        if (4 * i < left) {
            uint8_t *q = rp + (int64_t)i * 16 * W;                  // 4 rows of 4 W bytes
            __stcs(reinterpret_cast<uint2 *>(q), h);
            __stcs(reinterpret_cast<uint2 *>(q + 2 * W), l);
        }
    }
}

// Per-row epilogue inputs loaded one tile ahead (their latency overlaps the
// previous tile): the dZ' row scale and the row's CBSR indices (root term).
struct EpiPre {
    float cr;
    uint32_t iw[8];
};
__device__ __forceinline__ void epi_pre_load(const R2Args &a, int64_t row, EpiPre &e) {
    const bool ok = row < a.n;
    e.cr = (ok && a.crow) ? __ldg(a.crow + row) : 1.f;
#pragma unroll
    for (int t = 0; t < 8; ++t) e.iw[t] = 0xffffffffu;
    if (a.epi == kEpi2Dz && a.root && ok) {
        const int rk = a.root_k;
        const uint8_t *ip = a.root_idx + row * rk;
        if (rk == 16) {
            const uint4 w = __ldg(reinterpret_cast<const uint4 *>(ip));
            e.iw[0] = w.x; e.iw[1] = w.y; e.iw[2] = w.z; e.iw[3] = w.w;
        } else if (rk == 8) {
            const uint2 w = __ldg(reinterpret_cast<const uint2 *>(ip));
            e.iw[0] = w.x; e.iw[1] = w.y;
        } else if (rk == 32) {
            const uint4 w0 = __ldg(reinterpret_cast<const uint4 *>(ip));
            const uint4 w1 = __ldg(reinterpret_cast<const uint4 *>(ip) + 1);
            e.iw[0] = w0.x; e.iw[1] = w0.y; e.iw[2] = w0.z; e.iw[3] = w0.w;
            e.iw[4] = w1.x; e.iw[5] = w1.y; e.iw[6] = w1.z; e.iw[7] = w1.w;
        } else {
#pragma unroll
            for (int t = 0; t < 8; ++t)
                if (4 * t < rk) {
                    uint32_t w = 0xffffffffu;
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (4 * t + b < rk)
                            w = (w & ~(0xffu << (8 * b))) | ((uint32_t)__ldg(ip + 4 * t + b) << (8 * b));
                    e.iw[t] = w;
                }
        }
    }
}

// ---------------- fused next-layer D-ReLU (row a5; Eq. 2-3, applied
// to this layer's output, which is the next layer's input)
// The epilogue warp stages its 32 output rows in a [32][kRB] shared-memory row
// buffer (which is also the staging of the coalesced Y stores); each lane then
// selects its own row's exact top-NK with the thread-per-row network of the
// standalone D-ReLU (drelu_net.cuh tpr_select_row: composite keys, bitonic
// groups, exact rerun from shared memory on a truncated-key collision).
// Measured (a scratch microbenchmark, one warp per SM sub-partition as in this
// epilogue): ~5.3k cycles per 32 rows at N=64, k=8, vs ~50k for a warp-
// cooperative redux.max extraction (latency-bound at one warp per SMSP).
constexpr int kRB = 68;                // row-buffer stride (floats): 64 columns + 4 pad

// y of accumulator columns [j, j + 32) of this lane's row (bias, merge): the same
// operations in the same order as the forward epilogue's pass, so the same bits
__device__ __forceinline__ void epi_y32(const R2Args &a, uint32_t lb, int j, const float *bias_s,
                                        float (&y)[32]) {
    const int N = a.N;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int jj = j + 16 * h;
        uint32_t ra[16], rb[16];
        if (jj < N) {
            tc::tmem_ld16_nw(lb + (uint32_t)jj, ra);
            if (a.G == 2) tc::tmem_ld16_nw(lb + (uint32_t)(N + jj), rb);
            tc::tmem_wait_ld();
        }
        float ba[16], bb[16];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const float4 u = *reinterpret_cast<const float4 *>(bias_s + jj + 4 * q4);
            ba[4 * q4] = u.x; ba[4 * q4 + 1] = u.y; ba[4 * q4 + 2] = u.z; ba[4 * q4 + 3] = u.w;
            const float4 w = *reinterpret_cast<const float4 *>(bias_s + 256 + jj + 4 * q4);
            bb[4 * q4] = w.x; bb[4 * q4 + 1] = w.y; bb[4 * q4 + 2] = w.z; bb[4 * q4 + 3] = w.w;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float ya = jj < N ? __uint_as_float(ra[q]) + ba[q] : 0.f;
            const float yb = (a.G == 2 && jj < N) ? __uint_as_float(rb[q]) + bb[q] : 0.f;
            float v = ya;
            if (a.G == 2) v = a.merge == DR_MERGE_MAX ? (ya >= yb ? ya : yb) : ya + yb;
            y[16 * h + q] = v;
        }
    }
}

// Fused linear head + MSE (reading Q14) on the last layer's Y_cell, which is then
// never stored: per row pred = y . w_h + b_h, r = pred - label, dp = 2 r / n;
// writes dY = dp w_h (the backward's input) and accumulates, per warp in shared
// memory in a fixed order, the head gradient sum_rows y dp, sum dp and sum r^2.
__device__ __forceinline__ void head_epilogue(const R2Args &a, uint32_t lb, int64_t row0, int lane,
                                           bool ok, float pred, const float *hw, float hb,
                                           const float *bias_s, float *stg, float *hacc,
                                           float &accb, float &accl, float label) {
    const int N = a.N;
    const float r = ok ? pred + hb - label : 0.f;
    const float dp = 2.0f * r * a.head_inv_n;
    accb += dp;
    accl += r * r;
    for (int j = 0; j < N; j += 32) {
        float y[32];
        epi_y32(a, lb, j, bias_s, y);
#pragma unroll
        for (int q = 0; q < 32; ++q) y[q] = ok ? y[q] * dp : 0.f;
        stg_put(stg, kEStg, lane, y);
        __syncwarp();
        float cs = 0.f;                            // column j + lane over the 32 rows
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr) cs += stg[rr * kEStg + lane];
        if (j + lane < N) hacc[j + lane] += cs;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 32; ++q) y[q] = j + q < N ? dp * hw[j + q] : 0.f;
        stg_put(stg, kEStg, lane, y);
        __syncwarp();
        stg_out_f32(stg, kEStg, a.head_dy, N, row0, a.n, j, lane);
        __syncwarp();
    }
}

// The same head pass on y staged in the warp's [32][kRB] row buffer (N <= 64):
// column sums of y dp over the warp's rows with dp broadcast from its row's lane
// (fused multiply-add, rows in ascending order), then dY = dp w_h staged over y
// and stored coalesced.
__device__ __forceinline__ void head_epilogue_staged(const R2Args &a, int64_t row0, int lane, bool ok,
                                                     float pred, const float *hw, float hb, float *stg,
                                                     float *hacc, float &accb, float &accl, float label) {
    const int N = a.N;
    const float r = ok ? pred + hb - label : 0.f;
    const float dp = 2.0f * r * a.head_inv_n;
    accb += dp;
    accl += r * r;
    for (int j = 0; j < N; j += 32) {
        float c0 = 0.f, c1 = 0.f;                  // column j + lane over the 32 rows
#pragma unroll 8
        for (int rr = 0; rr < 32; rr += 2) {
            c0 = fmaf(stg[rr * kRB + j + lane], __shfl_sync(0xffffffffu, dp, rr), c0);
            c1 = fmaf(stg[(rr + 1) * kRB + j + lane], __shfl_sync(0xffffffffu, dp, rr + 1), c1);
        }
        if (j + lane < N) hacc[j + lane] += c0 + c1;
    }
    __syncwarp();
    for (int j = 0; j < N; j += 32) {
        float y[32];
        const float4 *h4 = reinterpret_cast<const float4 *>(hw + j);   // zero past N
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
            const float4 w = h4[q4];
            y[4 * q4] = dp * w.x;
            y[4 * q4 + 1] = dp * w.y;
            y[4 * q4 + 2] = dp * w.z;
            y[4 * q4 + 3] = dp * w.w;
        }
        stg_put(stg + j, kRB, lane, y);
    }
    __syncwarp();
    for (int j = 0; j < N; j += 32) stg_out_f32(stg + j, kRB, a.head_dy, N, row0, a.n, j, lane);
    __syncwarp();
}

// epilogue warp (quarter qd): rows r0 + 32 qd + lane of accumulator columns at `acc`
template <int NK>
__device__ __forceinline__ void rows_epilogue(const R2Args &a, uint32_t acc, int64_t r0, int qd,
                                              int lane, const float *bias_s, float *stg,
                                              const EpiPre &pre, const float *hw, float hb,
                                              float *hacc, float &accb, float &accl) {
    const int N = a.N;
    const int64_t row0 = r0 + qd * 32, row = row0 + lane;
    const bool ok = row < a.n;
    const uint32_t lb = acc + ((uint32_t)(qd * 32) << 16);
    if (NK == 0 && a.epi == kEpi2Dz) {        // (the fused D-ReLU variants are forward-only)
        const float cr = pre.cr;
        // root term: columns [n_dz, N) sampled at the row's CBSR indices (ascending),
        // collected in registers (static indices) and stored as whole rows at the end
        const int rk = a.root_k;
        const uint32_t *iw = pre.iw;
        float rv[16];                                  // rk <= 16: kept in registers
#pragma unroll
        for (int q = 0; q < 16; ++q) rv[q] = 0.f;
        for (int j = 0; j < N; j += 32) {
            uint32_t r[2][16];
            tc::tmem_ld16_nw(lb + (uint32_t)j, r[0]);
            if (j + 16 < N) tc::tmem_ld16_nw(lb + (uint32_t)(j + 16), r[1]);
            tc::tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                v[q] = __uint_as_float(r[0][q]);
                v[16 + q] = j + 16 < N ? __uint_as_float(r[1][q]) : 0.f;
            }
            // dZ' row scale (not the root term); n_dz % 16 == 0: uniform per half block
            if (j < a.n_dz) {
#pragma unroll
                for (int q = 0; q < 16; ++q) v[q] *= cr;
            }
            if (j + 16 < a.n_dz) {
#pragma unroll
                for (int q = 16; q < 32; ++q) v[q] *= cr;
            }
            stg_put(stg, kEStg, lane, v);
            __syncwarp();
            if (j < a.n_dz) {
                if (a.dz_split) stg_out_split(stg, reinterpret_cast<uint8_t *>(a.dz), a.n_dz, row0, a.n, j, lane);
                else stg_out_f32(stg, kEStg, a.dz, a.n_dz, row0, a.n, j, lane);
            }
            if (a.root && j + 32 > a.n_dz) {
                if (rk <= 16) {
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int c = a.n_dz + (int)((iw[q >> 2] >> (8 * (q & 3))) & 0xffu) - j;
                        if (q < rk && c >= 0 && c < 32) rv[q] = stg[lane * kEStg + c];
                    }
                } else if (ok) {                       // rk in (16, 32]: stored as found
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const int c = a.n_dz + (int)((iw[q >> 2] >> (8 * (q & 3))) & 0xffu) - j;
                        if (q < rk && c >= 0 && c < 32) a.root[row * rk + q] = stg[lane * kEStg + c];
                    }
                }
            }
            __syncwarp();
        }
        if (a.root && ok && rk <= 16) {
            if ((rk & 3) == 0) {
                float4 *o = reinterpret_cast<float4 *>(a.root + row * rk);
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (4 * q < rk) o[q] = make_float4(rv[4 * q], rv[4 * q + 1], rv[4 * q + 2], rv[4 * q + 3]);
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (q < rk) a.root[row * rk + q] = rv[q];
            }
        }
        return;
    }
    const int mw = (N + 31) >> 5;
    // fused head: the row's label is loaded first, its latency under the TMEM reads
    const float label = (NK < 0 && ok) ? __ldg(a.labels + row) : 0.f;
    // NK > 0 (fused next-layer D-ReLU): `stg` is the warp's [32][kRB] row buffer
    // and every block stays staged at its columns until the selection below
    // fused head with N <= 64: y stays staged the same way, so the head pass reads it
    // back from shared memory instead of a second TMEM read + merge
    const bool rowbuf = NK > 0 || (NK < 0 && N <= 64);
    const int sstride = rowbuf ? kRB : kEStg;
    float pred = 0.f;                              // fused head: y . w_h of this row
    for (int j = 0; j < N; j += 32) {
        uint32_t ra[2][16], rb[2][16];
        tc::tmem_ld16_nw(lb + (uint32_t)j, ra[0]);
        if (j + 16 < N) tc::tmem_ld16_nw(lb + (uint32_t)(j + 16), ra[1]);
        if (a.G == 2) {
            tc::tmem_ld16_nw(lb + (uint32_t)(N + j), rb[0]);
            if (j + 16 < N) tc::tmem_ld16_nw(lb + (uint32_t)(N + j + 16), rb[1]);
        }
        tc::tmem_wait_ld();
        uint32_t word = 0;
        float y[32];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int jj = j + 16 * h;
            float ya[16], yb[16];
            // the 16 biases of this half as 4 broadcast 128-bit shared loads per group
            // (jj is a multiple of 16: 64-B aligned)
            float ba[16], bb[16];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) {
                const float4 u = *reinterpret_cast<const float4 *>(bias_s + jj + 4 * q4);
                ba[4 * q4] = u.x; ba[4 * q4 + 1] = u.y; ba[4 * q4 + 2] = u.z; ba[4 * q4 + 3] = u.w;
                const float4 w = *reinterpret_cast<const float4 *>(bias_s + 256 + jj + 4 * q4);
                bb[4 * q4] = w.x; bb[4 * q4 + 1] = w.y; bb[4 * q4 + 2] = w.z; bb[4 * q4 + 3] = w.w;
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                ya[q] = jj < N ? __uint_as_float(ra[h][q]) + ba[q] : 0.f;
                yb[q] = (a.G == 2 && jj < N) ? __uint_as_float(rb[h][q]) + bb[q] : 0.f;
            }
            if (a.G == 2) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    if (a.merge == DR_MERGE_MAX) {
                        const bool m = ya[q] >= yb[q];          // Eq. 14: ties -> near
                        y[16 * h + q] = m ? ya[q] : yb[q];
                        word |= (uint32_t)m << (16 * h + q);
                    } else {
                        y[16 * h + q] = ya[q] + yb[q];
                    }
                }
                if (ok && a.tap_a && jj < N) {
                    float4 *o = reinterpret_cast<float4 *>(a.tap_a + row * N + jj);
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = make_float4(ya[4 * q], ya[4 * q + 1], ya[4 * q + 2], ya[4 * q + 3]);
                }
                if (ok && a.tap_b && jj < N) {
                    float4 *o = reinterpret_cast<float4 *>(a.tap_b + row * N + jj);
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = make_float4(yb[4 * q], yb[4 * q + 1], yb[4 * q + 2], yb[4 * q + 3]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) y[16 * h + q] = ya[q];
            }
        }
        float *sb = rowbuf ? stg + j : stg;
        if (rowbuf || a.y) {
            stg_put(sb, sstride, lane, y);
            __syncwarp();
        }
        if (a.y) {
            stg_out_f32(sb, sstride, a.y, N, row0, a.n, j, lane);
            __syncwarp();
        }
        if (ok && a.G == 2 && a.mask_out) a.mask_out[row * mw + (j >> 5)] = word;
        if constexpr (NK < 0) {
            // y . w_h over this block: w_h as broadcast 128-bit loads (zero past N,
            // as y is), four partial sums
            const float4 *h4 = reinterpret_cast<const float4 *>(hw + j);
            float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
            for (int q4 = 0; q4 < 8; ++q4) {
                const float4 w = h4[q4];
                p0 = fmaf(y[4 * q4], w.x, p0);
                p1 = fmaf(y[4 * q4 + 1], w.y, p1);
                p2 = fmaf(y[4 * q4 + 2], w.z, p2);
                p3 = fmaf(y[4 * q4 + 3], w.w, p3);
            }
            pred += (p0 + p1) + (p2 + p3);
        }
    }
    if constexpr (NK < 0) {
        if (rowbuf) head_epilogue_staged(a, row0, lane, ok, pred, hw, hb, stg, hacc, accb, accl, label);
        else head_epilogue(a, lb, row0, lane, ok, pred, hw, hb, bias_s, stg, hacc, accb, accl, label);
    }
    if constexpr (NK > 0) {
        const float *xr = stg + lane * kRB;
        if (a.nk_stream) {
            if (N == 64) tpr_select_row<64, NK, false, true>(xr, ok, a.nval + row * NK, a.nidx + row * NK);
            else tpr_select_row<32, (NK < 32 ? NK : 32), false, true>(xr, ok, a.nval + row * NK, a.nidx + row * NK);
        } else {
            if (N == 64) tpr_select_row<64, NK, false, false>(xr, ok, a.nval + row * NK, a.nidx + row * NK);
            else tpr_select_row<32, (NK < 32 ? NK : 32), false, false>(xr, ok, a.nval + row * NK, a.nidx + row * NK);
        }
        __syncwarp();
    }
}

template <int NK, bool W2>
__global__ void __launch_bounds__(RowsRoles<W2>::threads, 1) tc2_rows_kernel(const __grid_constant__ R2Args a) {
    using RR = RowsRoles<W2>;
    constexpr int kRowsThreads = RR::threads;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[kMaxSA], conv[kMaxSA], empty[kMaxSA];
    __shared__ __align__(8) uint64_t bfull[kMaxSB], bempty[kMaxSB], accf[2], acce[2];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(16) float bias_s[512];
    // fused head (NK < 0 only): w_h, b_h and the per-epilogue-warp sums
    float *head_s = nullptr;
    float (*hacc_s)[258] = nullptr;
    if constexpr (NK < 0) {
        __shared__ __align__(16) float head_sh[260];
        __shared__ float hacc_sh[8][258];
        head_s = head_sh;
        hacc_s = hacc_sh;
    }
    const long long kt00 = clock64();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int SA = a.SA, SB = a.SB, S = a.S;
    for (int e = tid; e < 512; e += kRowsThreads) {
        const int g = e >> 8, j = e & 255;
        bias_s[e] = (a.epi == kEpi2Fwd && g < a.G && j < a.N && a.bias[g]) ? a.bias[g][j] : 0.f;
    }
    if (NK < 0) {
        for (int e = tid; e < 257; e += kRowsThreads)
            head_s[e] = e < a.N ? a.head_w[e] : (e == 256 ? a.head_b[0] : 0.f);
        for (int e = tid; e < 8 * 258; e += kRowsThreads) hacc_s[e / 258][e % 258] = 0.f;
    }
    uint8_t *stages = sm;
    uint8_t *bslots = sm + (size_t)SA * kStage;
    uint8_t *masks = bslots + (size_t)SB * a.bchunk;
    uint8_t *epi_stage = sm + a.epi_off;        // 4 a.ewg epilogue warps' staging (1024-aligned)
    const uint32_t GN = (uint32_t)(a.G * a.N);
    uint32_t ncols = 32;
    while (ncols < 2 * GN) ncols <<= 1;
    if (tid == 0) {
        for (int i = 0; i < SA; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&conv[i], 4);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < SB; ++i) {
            tc::mbar_init(&bfull[i], 1);
            tc::mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&accf[i], 1);
            tc::mbar_init(&acce[i], 4);
        }
        tc::fence_mbar_init();
    }
    if (warp == RR::mma) {
        tc::tmem_alloc(&tmem_slot, ncols);
        tc::tmem_relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    const long long kt0 = clock64();
    const int64_t n_tiles = (a.n + kTile - 1) / kTile;
    const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (a.dbg && tid == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        a.dbg[blockIdx.x * 16 + 11] = g;                                  // start (ns)
        a.dbg[blockIdx.x * 16 + 10] = (unsigned long long)(kt0 - kt00);   // setup
    }

    if (W2 ? (warp >= 4 && warp < 8) : warp < 2) {
        if constexpr (W2) tc::setmaxnreg_dec<40>();   // 128 (converters) + 40 + 2 x 168: <= 64 K
    if (warp == RR::prod) {
        // ---------------- producer
        if (a.b_resident) {
            if (lane == 0)
                for (int j = 0; j < S; ++j) {
                    const R2Step sp = a.step[j];
                    tc::mbar_arrive_expect_tx(&bfull[j], a.bchunk);
                    tc::bulk_g2s(bslots + (size_t)j * a.bchunk, a.bimg[sp.g] + (size_t)sp.bc * a.bchunk,
                                 a.bchunk, &bfull[j]);
                }
        }
        uint32_t it = 0, bt = 0;
        for (int64_t t = 0; t < my_tiles; ++t) {
            const int64_t r0 = ((int64_t)blockIdx.x + t * gridDim.x) * kTile;
            for (int j = 0; j < S; ++j, ++it) {
                const int slot = (int)(it % SA);
                const uint32_t u = it / SA;
                if (u > 0) {
                    RDBG_T0;
                    tc::mbar_wait_sleep(&empty[slot], (u - 1) & 1u);
                    if (lane == 0) RDBG_ADD(0);
                }
                const R2Step sp = a.step[j];
                rows_produce(a, sp, r0, stages + (size_t)slot * kStage, masks + (size_t)slot * kMaskStage,
                             &full[slot], lane);
                if (!a.b_resident) {
                    const int bs = (int)(bt % SB);
                    const uint32_t bu = bt / SB;
                    if (lane == 0) {
                        if (bu > 0) tc::mbar_wait_sleep(&bempty[bs], (bu - 1) & 1u);
                        tc::mbar_arrive_expect_tx(&bfull[bs], a.bchunk);
                        tc::bulk_g2s(bslots + (size_t)bs * a.bchunk,
                                     a.bimg[sp.g] + (size_t)sp.bc * a.bchunk, a.bchunk, &bfull[bs]);
                    }
                    ++bt;
                }
                __syncwarp();
            }
        }
    } else if (warp == RR::mma) {
        // ---------------- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_bf16(kTile, a.N);
            uint32_t it = 0, bt = 0;
            for (int64_t t = 0; t < my_tiles; ++t) {
                const uint32_t ab = (uint32_t)(t & 1);
                if (t >= 2) {
                    RDBG_T0;
                    tc::mbar_wait_sleep(&acce[ab], (uint32_t)(((t >> 1) - 1) & 1));
                    RDBG_ADD(2);
                }
                tc::fence_after();
                const uint32_t dbase = tmem + ab * GN;
                for (int j = 0; j < S; ++j, ++it) {
                    const int slot = (int)(it % SA);
                    {
                        RDBG_T0;
                        tc::mbar_wait_sleep(&conv[slot], (it / SA) & 1u);
                        RDBG_ADD(1);
                    }
                    const R2Step sp = a.step[j];
                    int bs;
                    if (a.b_resident) {
                        bs = j;
                        tc::mbar_wait_sleep(&bfull[bs], 0u);
                    } else {
                        bs = (int)(bt % SB);
                        tc::mbar_wait_sleep(&bfull[bs], (bt / SB) & 1u);
                    }
                    tc::fence_after();
                    const R2Seg &sg = a.seg[sp.g][sp.s];
                    const int Kc = min(kChunk, sg.K - sp.c * kChunk);
                    const int nks = (Kc + 15) >> 4;
                    const uint32_t sa = tc::smem_u32(stages + (size_t)slot * kStage);
                    const uint32_t sb = tc::smem_u32(bslots + (size_t)bs * a.bchunk);
                    const uint32_t blo = (uint32_t)a.N * 128u;
                    const uint32_t d = dbase + (uint32_t)(sp.g * a.N);
                    for (int ks = 0; ks < nks; ++ks) {
                        const uint32_t ko = ks * 32;
                        const uint64_t ah = tc::desc_sw128(sa + ko), al = tc::desc_sw128(sa + kHalf + ko);
                        const uint64_t bh = tc::desc_sw128(sb + ko), bl = tc::desc_sw128(sb + blo + ko);
                        tc::mma_bf16(d, ah, bh, idesc, (sp.first && ks == 0) ? 0u : 1u);
                        tc::mma_bf16(d, ah, bl, idesc, 1u);
                        tc::mma_bf16(d, al, bh, idesc, 1u);
                    }
                    tc::mma_commit(&empty[slot]);
                    if (!a.b_resident) {
                        tc::mma_commit(&bempty[bs]);
                        ++bt;
                    }
                }
                tc::mma_commit(&accf[ab]);
            }
        }
        __syncwarp();
    }
    } else if (warp >= RR::conv0 && warp < RR::conv0 + 4) {
        // ---------------- converters
        const int ct = tid - 32 * RR::conv0;
        uint32_t it = 0;
        for (int64_t t = 0; t < my_tiles; ++t) {
            const int64_t r0 = ((int64_t)blockIdx.x + t * gridDim.x) * kTile;
            for (int j = 0; j < S; ++j, ++it) {
                const int slot = (int)(it % SA);
                {
                    RDBG_T0;
                    tc::mbar_wait(&full[slot], (it / SA) & 1u);
                    if (ct == 0) RDBG_ADD(3);
                }
                RDBG_T0;
                rows_convert(a, a.step[j], r0, stages + (size_t)slot * kStage,
                             masks + (size_t)slot * kMaskStage, ct);
                if (ct == 0) RDBG_ADD(4);
                tc::fence_async_smem();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&conv[slot]);
            }
        }
    } else {
        if constexpr (W2) tc::setmaxnreg_inc<168>();
        // ---------------- epilogue: warpgroup eg takes tiles t = eg, eg + ewg, ...
        // (accumulator t & 1; with ewg = 2 warpgroup eg always owns accumulator eg)
        const int qd = warp & 3, ew = warp - RR::epi0, eg = ew >> 2, ewg = W2 ? a.ewg : 1;
        float *stg = reinterpret_cast<float *>(epi_stage + (size_t)ew * epi_warp_bytes(NK != 0));
        EpiPre pcur, pnxt;
        float accb = 0.f, accl = 0.f;              // fused head: sum dp, sum r^2 of this lane
        float (*hacc)[258] = hacc_s + ew;
        if (eg < ewg) {
            if (NK == 0 && eg < my_tiles)
                epi_pre_load(a, ((int64_t)blockIdx.x + (int64_t)eg * gridDim.x) * kTile + qd * 32 + lane, pcur);
            for (int64_t t = eg; t < my_tiles; t += ewg) {
                const int64_t r0 = ((int64_t)blockIdx.x + t * gridDim.x) * kTile;
                const uint32_t ab = (uint32_t)(t & 1);
                if (NK == 0 && t + ewg < my_tiles)
                    epi_pre_load(a, r0 + (int64_t)ewg * gridDim.x * kTile + qd * 32 + lane, pnxt);
                {
                    RDBG_T0;
                    tc::mbar_wait_sleep(&accf[ab], (uint32_t)((t >> 1) & 1));
                    if (ew == 0 && lane == 0) RDBG_ADD(5);
                }
                tc::fence_after();
                RDBG_T0;
                rows_epilogue<NK>(a, tmem + ab * GN, r0, qd, lane, bias_s, stg, pcur, head_s,
                                  head_s[256], hacc[0], accb, accl);
                pcur = pnxt;
                if (ew == 0 && lane == 0) RDBG_ADD(6);
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce[ab]);
            }
        }
        if (NK < 0) {   // this CTA's partial [sum_rows y dp (N) | sum dp | sum r^2], fixed order
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                accb += __shfl_xor_sync(0xffffffffu, accb, o);
                accl += __shfl_xor_sync(0xffffffffu, accl, o);
            }
            if (lane == 0) {
                hacc[0][a.N] += accb;
                hacc[0][a.N + 1] += accl;
            }
            tc::named_bar(2, 32 * RR::nepi);
            const int et = tid - 32 * RR::epi0;
            for (int e = et; e < a.N + 2; e += 32 * RR::nepi) {
                float v = hacc_s[0][e];
#pragma unroll
                for (int w8 = 1; w8 < RR::nepi; ++w8) v += hacc_s[w8][e];
                a.head_part[(int64_t)blockIdx.x * (a.N + 2) + e] = v;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (a.dbg && tid == 0) {
        atomicAdd(a.dbg + blockIdx.x * 16 + 8, (unsigned long long)(clock64() - kt0));
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        a.dbg[blockIdx.x * 16 + 12] = g;                                  // end (ns)
    }
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, ncols);
    }
}

// ================================================================= reduce GEMM
// Stage (64 graph rows): per group g an A' operand [128 features][64 rows]
// (hi + lo, 32 KB; the dense segment's raw rows land in it and are transposed
// in place), B' = mask(dY)^T [N][64 rows] (hi + lo, 256 N bytes; dY rows land in
// it), CBSR rows and mask words in small side areas.
struct RdSeg {
    const float *Z;
    const float *hval;
    const uint8_t *hidx;
    int k, w, m0;
    int split;                         // Z rows are [hi | lo] bf16 halves
};
struct RdArgs {
    CUtensorMap zmap[2][2];            // split Z segments: [n x 2w] bf16, box 64 cols x 64 rows, SW128
    int64_t n;
    int N, G;
    int nseg[2];
    RdSeg seg[2][2];
    const float *dy;
    const uint32_t *mask;
    int mw, mask_mode;
    int mask_mode1, ndb;                                // dual B (variant 5): group 1's mask, # db vectors
    int SA;
    uint32_t stage_bytes, off_b, off_cbsr, off_mask;   // within a stage
    uint32_t off_b1;                                    // dual B: group 1's B operand
    uint32_t cbsr_seg_bytes;                            // per CBSR segment: vals (64k*4) + idx (64k)
    int64_t rows_per_cta;
    float *part;                                        // [grid][G*128*N + N]
    unsigned long long *dbg;                            // DR_TC2_DEBUG role timers, else null
};


constexpr int kRRows = 64;     // graph rows per reduce step (= MMA K of 4 kind::f16 steps)

__device__ __forceinline__ void red_produce(const RdArgs &a, int64_t rb, int64_t re, uint8_t *st,
                                            uint64_t *full, int lane) {
    const int rows = (int)(re - rb < kRRows ? re - rb : kRRows);
    uint32_t bytes = 0;
    int ci = 0;
    for (int g = 0; g < a.G; ++g)
        for (int q = 0; q < a.nseg[g]; ++q) {
            const RdSeg &s = a.seg[g][q];
            if (s.Z && s.split) bytes += 2u * (uint32_t)(s.w / 64) * 8192u;   // full TMA boxes
            else if (s.Z) bytes += (uint32_t)rows * s.w * 4;
            else bytes += rup16((uint32_t)rows * s.k * 4) + rup16((uint32_t)rows * s.k);
        }
    bytes += (uint32_t)rows * a.N * 4;
    const uint32_t mb = a.mask_mode != kMask2None ? rup16((uint32_t)rows * a.mw * 4) : 0u;
    bytes += mb;
    if (lane == 0) {
        tc::mbar_arrive_expect_tx(full, bytes);
        for (int g = 0; g < a.G; ++g)
            for (int q = 0; q < a.nseg[g]; ++q) {
                const RdSeg &s = a.seg[g][q];
                if (s.Z && s.split) {
                    // the [hi | lo] bf16 rows land as MN-major SW128 atoms: no conversion
                    // (rows past n arrive as zeros)
                    for (int at = 0; at < s.w / 64; ++at) {
                        uint8_t *dst = st + (size_t)g * kStage + (size_t)(s.m0 / 64 + at) * 8192;
                        tc::tma_load_2d(dst, &a.zmap[g][q], at * 64, (int)rb, full);
                        tc::tma_load_2d(dst + kHalf, &a.zmap[g][q], s.w + at * 64, (int)rb, full);
                    }
                } else if (s.Z) {
                    tc::bulk_g2s(st + (size_t)g * kStage, s.Z + rb * s.w, (uint32_t)rows * s.w * 4, full);
                } else {
                    uint8_t *cb = st + a.off_cbsr + (size_t)ci * a.cbsr_seg_bytes;
                    tc::bulk_g2s(cb, s.hval + rb * s.k, rup16((uint32_t)rows * s.k * 4), full);
                    tc::bulk_g2s(cb + (size_t)kRRows * s.k * 4, s.hidx + rb * s.k,
                                 rup16((uint32_t)rows * s.k), full);
                    ++ci;
                }
            }
        tc::bulk_g2s(st + a.off_b, a.dy + rb * a.N, (uint32_t)rows * a.N * 4, full);
        if (mb) tc::bulk_g2s(st + a.off_mask, a.mask + rb * a.mw, mb, full);
    }
}

// Transposing split of a [64 rows][W] fp32 block (row stride W) into operand
// rows m0 .. m0+W-1 of a K-major [rows][64] bf16 hi/lo tile pair. A unit is a
// feature quad fq (4 columns) x a row octet j (8 graph rows): 8 float4 reads,
// 4 x (16-B hi + 16-B lo) writes. Lane l of a warp takes fq low bits from l%8
// and j low bits from l/8, so both the row reads (8 lanes = 128 contiguous B)
// and the swizzled writes (8 distinct 16-B bank groups per warp) are
// conflict-free. Rows >= valid read as 0; the merge mask is applied when asked.
struct Unit {
    int fq, j;
    bool ok;
};
__device__ __forceinline__ Unit red_unit(int W, int ct, int it) {
    const int W4 = W >> 2, fh = (W4 + 7) >> 3;
    const int u = ct + 128 * it;
    const int i = u & 7, gq = (u >> 3) & 3, rest = u >> 5;
    Unit x;
    x.fq = i + 8 * (rest % fh);
    x.j = gq + 4 * (rest / fh);
    x.ok = x.fq < W4 && x.j < 8;
    return x;
}
template <int MAXU>
__device__ __forceinline__ void red_read(const float *raw, int W, int valid, int ct,
                                         const uint8_t *mkraw, int mw, int mask_mode,
                                         float4 (&v)[MAXU][8], float (*colsum)[4]) {
    const float4 *raw4 = reinterpret_cast<const float4 *>(raw);
    const int W4 = W >> 2;
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
        const Unit x = red_unit(W, ct, i);
        if (!x.ok) continue;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int rr = 8 * x.j + r;
            float4 q = rr < valid ? raw4[rr * W4 + x.fq] : make_float4(0.f, 0.f, 0.f, 0.f);
            if (mask_mode != kMask2None) {
                const int col = 4 * x.fq;
                const uint32_t w =
                    *reinterpret_cast<const uint32_t *>(mkraw + (rr * mw + (col >> 5)) * 4);
                uint32_t b = (w >> (col & 31)) & 0xfu;
                if (mask_mode == kMask2NotM) b = ~b & 0xfu;
                if (!(b & 1u)) q.x = 0.f;
                if (!(b & 2u)) q.y = 0.f;
                if (!(b & 4u)) q.z = 0.f;
                if (!(b & 8u)) q.w = 0.f;
            }
            v[i][r] = q;
        }
        if (colsum) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                colsum[i][0] += v[i][r].x;
                colsum[i][1] += v[i][r].y;
                colsum[i][2] += v[i][r].z;
                colsum[i][3] += v[i][r].w;
            }
        }
    }
}
__device__ __forceinline__ void store_col8(uint8_t *tile, uint32_t lo_off, int m, int j,
                                           float a0, float a1, float a2, float a3, float a4,
                                           float a5, float a6, float a7) {
    uint4 h, l;
    tc::split_bf16x2(a0, a1, h.x, l.x);
    tc::split_bf16x2(a2, a3, h.y, l.y);
    tc::split_bf16x2(a4, a5, h.z, l.z);
    tc::split_bf16x2(a6, a7, h.w, l.w);
    const uint32_t off = tc::sw128_off_h((uint32_t)m, (uint32_t)(8 * j));
    *reinterpret_cast<uint4 *>(tile + off) = h;
    *reinterpret_cast<uint4 *>(tile + lo_off + off) = l;
}
template <int MAXU>
__device__ __forceinline__ void red_write(uint8_t *tile, uint32_t lo_off, int W, int m0, int ct,
                                          const float4 (&v)[MAXU][8]) {
#pragma unroll
    for (int i = 0; i < MAXU; ++i) {
        const Unit x = red_unit(W, ct, i);
        if (!x.ok) continue;
        const int m = m0 + 4 * x.fq;
        store_col8(tile, lo_off, m + 0, x.j, v[i][0].x, v[i][1].x, v[i][2].x, v[i][3].x,
                   v[i][4].x, v[i][5].x, v[i][6].x, v[i][7].x);
        store_col8(tile, lo_off, m + 1, x.j, v[i][0].y, v[i][1].y, v[i][2].y, v[i][3].y,
                   v[i][4].y, v[i][5].y, v[i][6].y, v[i][7].y);
        store_col8(tile, lo_off, m + 2, x.j, v[i][0].z, v[i][1].z, v[i][2].z, v[i][3].z,
                   v[i][4].z, v[i][5].z, v[i][6].z, v[i][7].z);
        store_col8(tile, lo_off, m + 3, x.j, v[i][0].w, v[i][1].w, v[i][2].w, v[i][3].w,
                   v[i][4].w, v[i][5].w, v[i][6].w, v[i][7].w);
    }
}

// converters: one stage -> A'_g (per group) and B' operands; db unit sums in colsum
__device__ __forceinline__ void red_convert(const RdArgs &a, uint8_t *st, int valid, int ct,
                                            float (&colsum)[2][4], int bar) {
    const uint8_t *mk = st + a.off_mask;
    int ci = 0;
    for (int g = 0; g < a.G; ++g) {
        uint8_t *tile = st + (size_t)g * kStage;
        float4 v[2][8];
        int wd = 0, wtot = 0;
        const RdSeg *dseg = nullptr;
        for (int q = 0; q < a.nseg[g]; ++q) {
            wtot += a.seg[g][q].w;
            if (a.seg[g][q].Z) { dseg = &a.seg[g][q]; wd = dseg->w; }
        }
        if (dseg) red_read<2>(reinterpret_cast<const float *>(tile), wd, valid, ct, mk, 0,
                              kMask2None, v, nullptr);
        // CBSR entries of this group: thread -> graph row ct/2, half ct&1 of its k pairs
        float cv[16];
        uint32_t cid[16];
        int cm0 = 0, ck = 0;
        bool has_cbsr = false;
        for (int q = 0; q < a.nseg[g]; ++q) {
            const RdSeg &s = a.seg[g][q];
            if (s.Z) continue;
            has_cbsr = true;
            cm0 = s.m0;
            ck = s.k;
            const uint8_t *cb = st + a.off_cbsr + (size_t)ci * a.cbsr_seg_bytes;
            const int r = ct >> 1, h = ct & 1;
            const float *vals = reinterpret_cast<const float *>(cb) + r * s.k;
            const uint8_t *ids = cb + (size_t)kRRows * s.k * 4 + r * s.k;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const int tt = 2 * t + h;
                const bool ok = tt < s.k && r < valid;
                cv[t] = ok ? vals[tt] : 0.f;
                cid[t] = ok ? (uint32_t)ids[tt] : 0xffffffffu;
            }
            ++ci;
        }
        tc::named_bar(bar, 128);                      // raw reads done before writes
        if (dseg) red_write<2>(tile, kHalf, wd, dseg->m0, ct, v);
        {   // zero the CBSR rows and the unused rows [wtot, 128)
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < a.nseg[g]; ++q) {
                const RdSeg &s = a.seg[g][q];
                if (s.Z) continue;
                for (int e = ct; e < s.w * 8; e += 128) {
                    const int m = s.m0 + e / 8, c = e % 8;
                    *reinterpret_cast<float4 *>(tile + m * 128 + c * 16) = z;
                    *reinterpret_cast<float4 *>(tile + kHalf + m * 128 + c * 16) = z;
                }
            }
            for (int e = wtot * 8 + ct; e < kTile * 8; e += 128) {
                const int m = e / 8, c = e % 8;
                *reinterpret_cast<float4 *>(tile + m * 128 + c * 16) = z;
                *reinterpret_cast<float4 *>(tile + kHalf + m * 128 + c * 16) = z;
            }
        }
        if (has_cbsr) {
            tc::named_bar(bar, 128);                  // zeros before the scatter
            const int r = ct >> 1;
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (2 * t + (ct & 1) < ck && cid[t] != 0xffffffffu) {
                    uint32_t h, l;
                    tc::split_bf16x2(cv[t], 0.f, h, l);
                    const uint32_t off = tc::sw128_off_h((uint32_t)(cm0 + (int)cid[t]), (uint32_t)r);
                    *reinterpret_cast<uint16_t *>(tile + off) = (uint16_t)(h & 0xffffu);
                    *reinterpret_cast<uint16_t *>(tile + kHalf + off) = (uint16_t)(l & 0xffffu);
                }
        }
    }
    {   // B' = mask(dY)^T
        uint8_t *tile = st + a.off_b;
        float4 v[2][8];
        red_read<2>(reinterpret_cast<const float *>(tile), a.N, valid, ct, mk, a.mw, a.mask_mode, v,
                    colsum);
        tc::named_bar(bar, 128);
        red_write<2>(tile, (uint32_t)a.N * 128u, a.N, 0, ct, v);
    }
}

// ---- specialised converter: compile-time layout (G groups, dense width WD, CBSR
// width WC, N output columns), for the square-layer shapes of the workloads:
//   G = 1: group 0 = [Z (WD) | densify(H) (WC)], G = 2: group 0 = Z, group 1 = H.
template <int W>
__device__ __forceinline__ Unit red_unit_t(int ct, int it) {
    constexpr int W4 = W / 4, fh = (W4 + 7) / 8;
    const int u = ct + 128 * it;
    const int i = u & 7, gq = (u >> 3) & 3, rest = u >> 5;
    Unit x;
    x.fq = i + 8 * (rest % fh);
    x.j = gq + 4 * (rest / fh);
    x.ok = x.fq < W4 && x.j < 8;
    return x;
}
template <int W>
__device__ __forceinline__ void red_read_t(const float *raw, int valid, int ct, const uint8_t *mkraw,
                                           int mw, int mask_mode, float4 (&v)[2][8],
                                           float (*colsum)[4]) {
    const float4 *raw4 = reinterpret_cast<const float4 *>(raw);
    constexpr int W4 = W / 4;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const Unit x = red_unit_t<W>(ct, i);
        if (!x.ok) continue;
        const int col = 4 * x.fq;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int rr = 8 * x.j + r;
            float4 q = raw4[rr * W4 + x.fq];
            if (rr >= valid) q = make_float4(0.f, 0.f, 0.f, 0.f);
            if (mask_mode != kMask2None) {
                const uint32_t w = *reinterpret_cast<const uint32_t *>(mkraw + (rr * mw + (col >> 5)) * 4);
                uint32_t b = (w >> (col & 31)) & 0xfu;
                if (mask_mode == kMask2NotM) b = ~b & 0xfu;
                if (!(b & 1u)) q.x = 0.f;
                if (!(b & 2u)) q.y = 0.f;
                if (!(b & 4u)) q.z = 0.f;
                if (!(b & 8u)) q.w = 0.f;
            }
            v[i][r] = q;
            if (colsum) {
                colsum[i][0] += q.x;
                colsum[i][1] += q.y;
                colsum[i][2] += q.z;
                colsum[i][3] += q.w;
            }
        }
    }
}
template <int W>
__device__ __forceinline__ void red_write_t(uint8_t *tile, uint32_t lo_off, int m0, int ct,
                                            const float4 (&v)[2][8]) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const Unit x = red_unit_t<W>(ct, i);
        if (!x.ok) continue;
        const int m = m0 + 4 * x.fq;
        store_col8(tile, lo_off, m + 0, x.j, v[i][0].x, v[i][1].x, v[i][2].x, v[i][3].x,
                   v[i][4].x, v[i][5].x, v[i][6].x, v[i][7].x);
        store_col8(tile, lo_off, m + 1, x.j, v[i][0].y, v[i][1].y, v[i][2].y, v[i][3].y,
                   v[i][4].y, v[i][5].y, v[i][6].y, v[i][7].y);
        store_col8(tile, lo_off, m + 2, x.j, v[i][0].z, v[i][1].z, v[i][2].z, v[i][3].z,
                   v[i][4].z, v[i][5].z, v[i][6].z, v[i][7].z);
        store_col8(tile, lo_off, m + 3, x.j, v[i][0].w, v[i][1].w, v[i][2].w, v[i][3].w,
                   v[i][4].w, v[i][5].w, v[i][6].w, v[i][7].w);
    }
}
template <int G, int WD, int WC, int N>
__device__ __forceinline__ void red_convert_t(const RdArgs &a, uint8_t *st, int valid, int ct,
                                              float (&colsum)[2][4], int bar) {
    const uint8_t *mk = st + a.off_mask;
    uint8_t *tz = st;                                   // group 0: dense rows [0, WD)
    uint8_t *th = G == 2 ? st + kStage : st;            // CBSR rows [hm0, hm0 + WC)
    constexpr int hm0 = G == 2 ? 0 : WD;
    float4 v[2][8];
    red_read_t<WD>(reinterpret_cast<const float *>(tz), valid, ct, mk, 0, kMask2None, v, nullptr);
    // CBSR: thread -> graph row r = ct & 63, contiguous half h = ct >> 6 of its k pairs
    const int kc = a.seg[G == 2 ? 1 : 0][G == 2 ? 0 : 1].k;
    const int r = ct & 63, h = ct >> 6, kh = kc >> 1;
    float cv[16];
    uint32_t cw[4];
    if constexpr (WC > 0) {
        const uint8_t *cb = st + a.off_cbsr;
        const float *vals = reinterpret_cast<const float *>(cb) + r * kc + h * kh;
        const uint8_t *ids = cb + (size_t)kRRows * kc * 4 + r * kc + h * kh;
        const bool okr = r < valid;
#pragma unroll
        for (int t = 0; t < 16; ++t) cv[t] = (t < kh && okr) ? vals[t] : 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            uint32_t w = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (4 * t + b < kh) w |= (uint32_t)ids[4 * t + b] << (8 * b);
            cw[t] = okr ? w : 0u;
        }
    }
    tc::named_bar(bar, 128);                              // raw reads done before writes
    red_write_t<WD>(tz, kHalf, 0, ct, v);
    {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (WC > 0) {
#pragma unroll
            for (int e0 = 0; e0 < WC * 8; e0 += 128) {
                const int e = e0 + ct, m = hm0 + e / 8, c = e % 8;
                *reinterpret_cast<float4 *>(th + m * 128 + c * 16) = z;
                *reinterpret_cast<float4 *>(th + kHalf + m * 128 + c * 16) = z;
            }
        }
        if constexpr (G == 1 && WD + WC < kTile) {
            for (int e = (WD + WC) * 8 + ct; e < kTile * 8; e += 128) {
                const int m = e / 8, c = e % 8;
                *reinterpret_cast<float4 *>(tz + m * 128 + c * 16) = z;
                *reinterpret_cast<float4 *>(tz + kHalf + m * 128 + c * 16) = z;
            }
        }
    }
    if constexpr (WC > 0) {
        tc::named_bar(bar, 128);                          // zeros before the scatter
        if (r < valid) {
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t < kh) {
                    const int id = (int)((cw[t >> 2] >> (8 * (t & 3))) & 0xffu);
                    uint32_t hh, ll;
                    tc::split_bf16x2(cv[t], 0.f, hh, ll);
                    const uint32_t off = tc::sw128_off_h((uint32_t)(hm0 + id), (uint32_t)r);
                    *reinterpret_cast<uint16_t *>(th + off) = (uint16_t)(hh & 0xffffu);
                    *reinterpret_cast<uint16_t *>(th + kHalf + off) = (uint16_t)(ll & 0xffffu);
                }
        }
    }
    {   // B' = mask(dY)^T
        uint8_t *tile = st + a.off_b;
        red_read_t<N>(reinterpret_cast<const float *>(tile), valid, ct, mk, a.mw, a.mask_mode, v, colsum);
        tc::named_bar(bar, 128);
        red_write_t<N>(tile, (uint32_t)N * 128u, 0, ct, v);
    }
}

// ---- MN-major converters (the specialised shapes): no transposes. dW = A^T B
// with A = [Z | densify(H)] as [rows][features] and B = mask(dY) as [rows][N]:
// both operands stay row-major ([K = graph rows][MN]), split in place into bf16
// hi / lo 128-B-swizzled 64-wide atoms (8 KB each for 64 rows) and are read by
// the MMA as MN-major operands (cute Layout_MN_SW128: LBO = 8 KB between the
// 64-wide MN atoms, SBO = 1 KB between 8-row groups, 2 KB per K=16 step).
// A [64 rows][W] fp32 block: thread ct owns column quad q = ct % (W/4) of rows
// rg + RG j (RG = 128 / (W/4)); reads and 64-bit swizzled writes are
// conflict-free.
template <int W>
struct MnMap {
    static constexpr int W4 = W / 4, RG = 128 / W4, NJ = 64 / RG;
};
template <int W>
__device__ __forceinline__ void mn_read(const float *raw, int valid, int ct, const uint8_t *mkraw,
                                        int mw, int mask_mode, float4 (&v)[MnMap<W>::NJ],
                                        float *colsum) {
    using M = MnMap<W>;
    const int q = ct % M::W4, rg = ct / M::W4, col = 4 * q;
    const float4 *raw4 = reinterpret_cast<const float4 *>(raw);
#pragma unroll
    for (int j = 0; j < M::NJ; ++j) {
        const int r = rg + M::RG * j;
        float4 x = raw4[r * M::W4 + q];
        if (r >= valid) x = make_float4(0.f, 0.f, 0.f, 0.f);
        if (mask_mode != kMask2None) {
            const uint32_t w = *reinterpret_cast<const uint32_t *>(mkraw + (r * mw + (col >> 5)) * 4);
            uint32_t b = (w >> (col & 31)) & 0xfu;
            if (mask_mode == kMask2NotM) b = ~b & 0xfu;
            if (!(b & 1u)) x.x = 0.f;
            if (!(b & 2u)) x.y = 0.f;
            if (!(b & 4u)) x.z = 0.f;
            if (!(b & 8u)) x.w = 0.f;
        }
        v[j] = x;
        if (colsum) {
            colsum[0] += x.x;
            colsum[1] += x.y;
            colsum[2] += x.z;
            colsum[3] += x.w;
        }
    }
}
// dual B: one read of the raw dY block, both masked versions (mask modes m0 / m1)
template <int W>
__device__ __forceinline__ void mn_read2(const float *raw, int valid, int ct, const uint8_t *mkraw,
                                         int mw, int m0, int m1, float4 (&v0)[MnMap<W>::NJ],
                                         float4 (&v1)[MnMap<W>::NJ], float *cs0, float *cs1) {
    using M = MnMap<W>;
    const int q = ct % M::W4, rg = ct / M::W4, col = 4 * q;
    const float4 *raw4 = reinterpret_cast<const float4 *>(raw);
#pragma unroll
    for (int j = 0; j < M::NJ; ++j) {
        const int r = rg + M::RG * j;
        float4 x = raw4[r * M::W4 + q];
        if (r >= valid) x = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t w = *reinterpret_cast<const uint32_t *>(mkraw + (r * mw + (col >> 5)) * 4);
        const uint32_t bm = (w >> (col & 31)) & 0xfu;
        const uint32_t b0 = m0 == kMask2NotM ? (~bm & 0xfu) : m0 == kMask2M ? bm : 0xfu;
        const uint32_t b1 = m1 == kMask2NotM ? (~bm & 0xfu) : m1 == kMask2M ? bm : 0xfu;
        float4 y0 = x, y1 = x;
        if (!(b0 & 1u)) y0.x = 0.f;
        if (!(b0 & 2u)) y0.y = 0.f;
        if (!(b0 & 4u)) y0.z = 0.f;
        if (!(b0 & 8u)) y0.w = 0.f;
        if (!(b1 & 1u)) y1.x = 0.f;
        if (!(b1 & 2u)) y1.y = 0.f;
        if (!(b1 & 4u)) y1.z = 0.f;
        if (!(b1 & 8u)) y1.w = 0.f;
        v0[j] = y0;
        v1[j] = y1;
        cs0[0] += y0.x; cs0[1] += y0.y; cs0[2] += y0.z; cs0[3] += y0.w;
        cs1[0] += y1.x; cs1[1] += y1.y; cs1[2] += y1.z; cs1[3] += y1.w;
    }
}
// hi atoms at tile + 8 KB a, lo atoms at tile + lo_off + 8 KB a
template <int W>
__device__ __forceinline__ void mn_write(uint8_t *tile, uint32_t lo_off, int ct,
                                         const float4 (&v)[MnMap<W>::NJ]) {
    using M = MnMap<W>;
    const int q = ct % M::W4, rg = ct / M::W4, c = 4 * q;
    const uint32_t atom = (uint32_t)(c >> 6) * 8192u;
#pragma unroll
    for (int j = 0; j < M::NJ; ++j) {
        const int r = rg + M::RG * j;
        uint2 h, l;
        tc::split_bf16x2(v[j].x, v[j].y, h.x, l.x);
        tc::split_bf16x2(v[j].z, v[j].w, h.y, l.y);
        const uint32_t off = atom + tc::sw128_off_h((uint32_t)r, (uint32_t)(c & 63));
        *reinterpret_cast<uint2 *>(tile + off) = h;
        *reinterpret_cast<uint2 *>(tile + lo_off + off) = l;
    }
}
// G = 3: dual B (variant 5): group 0 = [Z | H] as for G = 1, group 1 = a second
// split Z (TMA-landed atoms, its unused feature atom zeroed once per slot), and
// two B operands, B0 = mask_mode(dY) at off_b and B1 = mask_mode1(dY) at off_b1
template <int G, int WD, int WC, int N>
__device__ __forceinline__ void red_convert_mn(const RdArgs &a, uint8_t *st, int valid, int ct,
                                               float (&colsum)[2][4], int bar) {
    const uint8_t *mk = st + a.off_mask;
    uint8_t *tz = st;                                   // group 0: Z atoms from 0
    uint8_t *th = G == 2 ? st + kStage : st + WD * 128; // H atoms (G = 1, 3: right after Z's)
    float4 vz[MnMap<WD>::NJ];
    const bool zsplit = a.seg[0][0].split != 0;         // Z landed as operand atoms (TMA)
    if (!zsplit) mn_read<WD>(reinterpret_cast<const float *>(tz), valid, ct, mk, 0, kMask2None, vz, nullptr);
    // CBSR: thread -> graph row r = ct & 63, contiguous half h = ct >> 6 of its k pairs
    const int kc = WC > 0 ? a.seg[G == 2 ? 1 : 0][G == 2 ? 0 : 1].k : 0;
    const int r = ct & 63, h = ct >> 6, kh = kc >> 1;
    float cv[16];
    uint32_t cw[4];
    if constexpr (WC > 0) {
        const uint8_t *cb = st + a.off_cbsr;
        const float *vals = reinterpret_cast<const float *>(cb) + r * kc + h * kh;
        const uint8_t *ids = cb + (size_t)kRRows * kc * 4 + r * kc + h * kh;
        const bool okr = r < valid;
#pragma unroll
        for (int t = 0; t < 16; ++t) cv[t] = (t < kh && okr) ? vals[t] : 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            uint32_t w = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (4 * t + b < kh) w |= (uint32_t)ids[4 * t + b] << (8 * b);
            cw[t] = okr ? w : 0u;
        }
    }
    tc::named_bar(bar, 128);                              // raw reads done before writes
    if (!zsplit) mn_write<WD>(tz, kHalf, ct, vz);
    {   // zero the H atoms (scattered into below) and, for a lone 64-wide Z, the
        // unused second feature atom (M = 128 rows of the accumulator)
        constexpr int ZB = WC > 0 ? WC * 128 : (G == 1 && WD < kTile ? (kTile - WD) * 128 : 0);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int e0 = 0; e0 < ZB / 16; e0 += 128) {
            const int e = e0 + ct;
            if (e < ZB / 16) {
                *reinterpret_cast<float4 *>(th + 16 * e) = z;
                *reinterpret_cast<float4 *>(th + kHalf + 16 * e) = z;
            }
        }
    }
    if constexpr (WC > 0) {
        tc::named_bar(bar, 128);                          // zeros before the scatter
        if (r < valid) {
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t < kh) {
                    const int id = (int)((cw[t >> 2] >> (8 * (t & 3))) & 0xffu);
                    uint32_t hh, ll;
                    tc::split_bf16x2(cv[t], 0.f, hh, ll);
                    const uint32_t off = (uint32_t)(id >> 6) * 8192u +
                                         tc::sw128_off_h((uint32_t)r, (uint32_t)(id & 63));
                    *reinterpret_cast<uint16_t *>(th + off) = (uint16_t)(hh & 0xffffu);
                    *reinterpret_cast<uint16_t *>(th + kHalf + off) = (uint16_t)(ll & 0xffffu);
                }
        }
    }
    if constexpr (G == 3) {   // B0 = mask_mode(dY) in place, B1 = mask_mode1(dY) at off_b1
        uint8_t *tile = st + a.off_b;
        float4 v0[MnMap<N>::NJ], v1[MnMap<N>::NJ];
        mn_read2<N>(reinterpret_cast<const float *>(tile), valid, ct, mk, a.mw, a.mask_mode, a.mask_mode1,
                    v0, v1, colsum[0], colsum[1]);
        tc::named_bar(bar, 128);
        mn_write<N>(tile, (uint32_t)N * 128u, ct, v0);
        mn_write<N>(st + a.off_b1, (uint32_t)N * 128u, ct, v1);
    } else {   // B = mask(dY), [rows][N], hi atoms then lo atoms (N * 128 bytes each)
        uint8_t *tile = st + a.off_b;
        float4 v[MnMap<N>::NJ];
        mn_read<N>(reinterpret_cast<const float *>(tile), valid, ct, mk, a.mw, a.mask_mode, v, colsum[0]);
        tc::named_bar(bar, 128);
        mn_write<N>(tile, (uint32_t)N * 128u, ct, v);
    }
}

template <int G_, int WD_, int WC_, int N_>
__global__ void __launch_bounds__(kRedThreads, 1) tc2_reduce_kernel(const __grid_constant__ RdArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t full[kMaxSA], conv[kMaxSA], empty[kMaxSA], accf;
    __shared__ uint32_t tmem_slot;
    __shared__ float dbs[2][8][128];
    const long long kt0 = clock64();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int SA = a.SA, G = a.G, N = a.N;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(G * N)) ncols <<= 1;
    if (tid == 0) {
        for (int i = 0; i < SA; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&conv[i], 4);
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(&accf, 1);
        tc::fence_mbar_init();
    }
    if (warp == 1) {
        tc::tmem_alloc(&tmem_slot, ncols);
        tc::tmem_relinquish();
    }
    if constexpr (G_ == 3) {
        // dual B: group 1 holds one 64-wide Z; its second feature atom (hi and lo)
        // is never written by TMA or the converters -- zero it once per stage slot
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int e = tid; e < SA * 1024; e += kRedThreads) {
            uint8_t *t1 = sm + (size_t)(e >> 10) * a.stage_bytes + kStage + 8192;
            const int u = e & 1023;                       // 512 x 16 B hi, 512 x 16 B lo
            *reinterpret_cast<float4 *>(t1 + (u < 512 ? 0 : kHalf) + 16 * (u & 511)) = z;
        }
        tc::fence_async_smem();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    const int64_t rbeg = (int64_t)blockIdx.x * a.rows_per_cta;
    const int64_t rend = a.n < rbeg + a.rows_per_cta ? a.n : rbeg + a.rows_per_cta;
    const int64_t total = rend > rbeg ? (rend - rbeg + kRRows - 1) / kRRows : 0;
    float *out = a.part + (int64_t)blockIdx.x * ((int64_t)G * kTile * N + (int64_t)a.ndb * N);

    if (warp == 0) {
        for (int64_t it = 0; it < total; ++it) {
            const int slot = (int)(it % SA);
            const uint32_t u = (uint32_t)(it / SA);
            if (u > 0) {
                RDBG_T0;
                tc::mbar_wait_sleep(&empty[slot], (u - 1) & 1u);
                if (lane == 0) RDBG_ADD(0);
            }
            red_produce(a, rbeg + it * kRRows, rend, sm + (size_t)slot * a.stage_bytes, &full[slot], lane);
            __syncwarp();
        }
    } else if (warp == 1) {
        if (lane == 0 && total > 0) {
            // the specialised shapes read both operands MN-major (bits 15, 16)
            const uint32_t idesc = tc::idesc_bf16(kTile, N) | (G_ > 0 ? (3u << 15) : 0u);
            for (int64_t it = 0; it < total; ++it) {
                const int slot = (int)(it % SA);
                {
                    RDBG_T0;
                    tc::mbar_wait_sleep(&conv[slot], (uint32_t)((it / SA) & 1));
                    RDBG_ADD(1);
                }
                tc::fence_after();
                uint8_t *st = sm + (size_t)slot * a.stage_bytes;
                const uint32_t sb0 = tc::smem_u32(st + a.off_b), blo = (uint32_t)N * 128u;
                for (int g = 0; g < G; ++g) {
                    const uint32_t sa = tc::smem_u32(st + (size_t)g * kStage);
                    const uint32_t sb = (G_ == 3 && g == 1) ? tc::smem_u32(st + a.off_b1) : sb0;
                    const uint32_t d = tmem + (uint32_t)(g * N);
#pragma unroll
                    for (int ks = 0; ks < kRRows / 16; ++ks) {
                        uint64_t ah, al, bh, bl;
                        if constexpr (G_ > 0) {            // K = 16 graph rows = 2 KB
                            const uint32_t ko = ks * 2048u;
                            ah = tc::desc_mn_sw128(sa + ko, 8192u, 1024u);
                            al = tc::desc_mn_sw128(sa + kHalf + ko, 8192u, 1024u);
                            bh = tc::desc_mn_sw128(sb + ko, 8192u, 1024u);
                            bl = tc::desc_mn_sw128(sb + blo + ko, 8192u, 1024u);
                        } else {
                            const uint32_t ko = ks * 32;
                            ah = tc::desc_sw128(sa + ko);
                            al = tc::desc_sw128(sa + kHalf + ko);
                            bh = tc::desc_sw128(sb + ko);
                            bl = tc::desc_sw128(sb + blo + ko);
                        }
                        tc::mma_bf16(d, ah, bh, idesc, (it == 0 && ks == 0) ? 0u : 1u);
                        tc::mma_bf16(d, ah, bl, idesc, 1u);
                        tc::mma_bf16(d, al, bh, idesc, 1u);
                    }
                }
                tc::mma_commit(&empty[slot]);
            }
            tc::mma_commit(&accf);
        }
        __syncwarp();
    } else {
        // two converter groups of 4 warps take alternate stages (their barrier
        // waits and latencies overlap); group 0 also reads the accumulator out
        const int grp = (warp - 2) >> 2, bar = 1 + grp;
        const int ct = tid - 64 - 128 * grp;
        float colsum[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        for (int64_t it = grp; it < total; it += 2) {
            const int slot = (int)(it % SA);
            {
                RDBG_T0;
                tc::mbar_wait(&full[slot], (uint32_t)((it / SA) & 1));
                if (ct == 0) RDBG_ADD(2);
            }
            const int64_t rb = rbeg + it * kRRows;
            const int valid = (int)(rend - rb < kRRows ? rend - rb : kRRows);
            {
                RDBG_T0;
                if constexpr (G_ > 0)
                    red_convert_mn<G_, WD_, WC_, N_>(a, sm + (size_t)slot * a.stage_bytes, valid, ct, colsum, bar);
                else
                    red_convert(a, sm + (size_t)slot * a.stage_bytes, valid, ct, colsum, bar);
                if (ct == 0) RDBG_ADD(3);
            }
            tc::fence_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&conv[slot]);
        }
        // db partials: per thread unit, then summed over the units of a column in a
        // fixed order (dual B: the same for group 1's B, a second round)
        for (int d2 = 0; d2 < (G_ == 3 ? 2 : 1); ++d2) {
            for (int e = ct; e < 8 * 128; e += 128) dbs[grp][e >> 7][e & 127] = 0.f;
            tc::named_bar(3, 256);
            if constexpr (G_ > 0) {
                const int q = ct % MnMap<N_>::W4, rg = ct / MnMap<N_>::W4;
                for (int e = 0; e < 4; ++e) dbs[grp][rg][4 * q + e] = colsum[d2][e];
            } else {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const Unit x = red_unit(N, ct, i);
                    if (x.ok)
                        for (int e = 0; e < 4; ++e) dbs[grp][x.j][4 * x.fq + e] = colsum[i][e];
                }
            }
            tc::named_bar(3, 256);
            if (grp == 0)
                for (int c = ct; c < N; c += 128) {
                    float s = 0.f;
                    for (int q = 0; q < 2; ++q)
                        for (int j = 0; j < 8; ++j) s += dbs[q][j][c];
                    out[(int64_t)G * kTile * N + (int64_t)d2 * N + c] = s;
                }
            tc::named_bar(3, 256);                        // dbs reused by the next round
        }
        // accumulator -> per-CTA partial (lane = feature row), group 0
        const int qd = warp & 3;
        if (total > 0 && grp == 0) {
            tc::mbar_wait_sleep(&accf, 0u);
            tc::fence_after();
        }
        const int m = qd * 32 + lane;
        const uint32_t lb = tmem + ((uint32_t)(qd * 32) << 16);
        for (int g = 0; g < (grp == 0 ? G : 0); ++g)
            for (int j = 0; j < N; j += 16) {
                float v[16];
                if (total > 0) tc::tmem_ld16(lb + (uint32_t)(g * N + j), v);
                else
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = 0.f;
                float4 *o = reinterpret_cast<float4 *>(out + ((int64_t)g * kTile + m) * N + j);
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            }
    }
    tc::fence_before();
    __syncthreads();
    if (a.dbg && tid == 0) atomicAdd(a.dbg + blockIdx.x * 16 + 8, (unsigned long long)(clock64() - kt0));
    if (warp == 1) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, ncols);
    }
}

// Sum per-CTA partials in a fixed order and scatter to the segment outputs; one
// job per blockIdx.y (several weight gradients in one launch).
struct PartsJobs {
    Tc2PartsJob job[Tc2Deferred::kMax];
};
__global__ void tc2_reduce_parts_kernel(const __grid_constant__ PartsJobs jobs) {
    const Tc2PartsJob &o = jobs.job[blockIdx.y];
    const int G = o.G, N = o.N, nparts = o.nparts;
    const float *__restrict__ part = o.part;
    __shared__ float red[8][33];
    const int64_t len = (int64_t)G * kTile * N + (int64_t)o.ndb * N;
    const int64_t e = (int64_t)blockIdx.x * 32 + threadIdx.x;
    if ((int64_t)blockIdx.x * 32 >= len) return;          // this job is shorter (block-uniform)
    float acc = 0.f;
    if (e < len)
#pragma unroll 8
        for (int c = threadIdx.y; c < nparts; c += 8) acc += __ldg(part + (int64_t)c * len + e);
    red[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y != 0 || e >= len) return;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x];
    if (e >= (int64_t)G * kTile * N) {
        const int64_t c = e - (int64_t)G * kTile * N;
        float *db = c < N ? o.db : o.db1;
        if (db) db[c < N ? c : c - N] = s;
        return;
    }
    const int g = (int)(e / ((int64_t)kTile * N));
    const int m = (int)((e / N) % kTile), c = (int)(e % N);
    for (int i = 0; i < o.nout; ++i)
        if (o.g[i] == g && m >= o.m0[i] && m < o.m0[i] + o.w[i])
            o.dst[i][(int64_t)(m - o.m0[i]) * N + c] = s;
}

}  // namespace

// ================================================================= host side
size_t tc2_bimg_bytes(int K, int Ntot) {
    return (size_t)((K + kChunk - 1) / kChunk) * 2 * (size_t)Ntot * 128;
}

void launch_tc2_pack_b(const float *W, int ldw, int K, int NB, int n0, int Ntot, bool transpose,
                       uint8_t *img, cudaStream_t s) {
    const int64_t total = (int64_t)((K + kChunk - 1) / kChunk) * NB * (kChunk / 2);
    int64_t blocks = (total + 255) / 256;
    if (blocks > 592) blocks = 592;
    if (blocks < 1) blocks = 1;
    tc2_pack_b_kernel<<<(unsigned)blocks, 256, 0, s>>>(W, ldw, K, NB, n0, Ntot, transpose ? 1 : 0, img);
    note_launch("tc2_pack_b");
}

void launch_tc2_pack_b_multi(const Tc2PackJob *jobs, int n, cudaStream_t s) {
    if (n <= 0) return;
    DR_CHECK(n <= kMaxPackJobs, DR_ERR_INVALID_ARGUMENT, "tc2_pack_b_multi: too many jobs");
    PackJobs j{};
    int64_t most = 1;
    for (int i = 0; i < n; ++i) {
        j.job[i] = jobs[i];
        const int64_t total = (int64_t)((jobs[i].K + kChunk - 1) / kChunk) * jobs[i].NB * (kChunk / 2);
        most = std::max(most, total);
    }
    int64_t bx = (most + 255) / 256;
    if (bx > 148) bx = 148;
    tc2_pack_b_multi_kernel<<<dim3((unsigned)bx, (unsigned)n), 256, 0, s>>>(j);
    note_launch("tc2_pack_b");
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    DR_CHECK(fn != nullptr, DR_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// output map: [n x W] fp32 row-major, box = 16 columns x 32 rows, SWIZZLE_64B
// [n x 2K] bf16 split rows ([hi | lo]), box = 64 columns x 128 rows, 128-B swizzle
// (= the K-major SW128 operand tile layout)
static void make_tmap_split(CUtensorMap *m, const float *A, int64_t n, int K, int box_rows = kTile) {
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * K), (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    const cuuint32_t box[2] = {(cuuint32_t)kChunk, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void *)A, dims, strides,
                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DR_CHECK(r == CUDA_SUCCESS, DR_ERR_CUDA, "cuTensorMapEncodeTiled (split) failed");
}

// [n x K] fp32 row-major, box = 64 columns x 128 rows, no swizzle (row-major
// [128][64] landing tile), zero fill out of range
static void make_tmap(CUtensorMap *m, const float *A, int64_t n, int K) {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 4};
    const cuuint32_t box[2] = {(cuuint32_t)kChunk, (cuuint32_t)kTile};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void *)A, dims, strides, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DR_CHECK(r == CUDA_SUCCESS, DR_ERR_CUDA, "cuTensorMapEncodeTiled failed");
}

static bool seg_ok(const Tc2Seg &s) {
    if (s.K < 4 || s.K > 256 || s.K % 4) return false;
    if (s.A && s.split && (s.K % kChunk || s.mask_mode != kMask2None)) return false;
    if (!s.A && (s.k < 1 || s.k > 32 || s.k > s.K)) return false;
    return true;
}

bool tc2_next_drelu_supported(int epi, int N, int k) {
    return epi == kEpi2Fwd && (N == 32 || N == 64) && k >= 1 && k <= 32 && (k & (k - 1)) == 0 && k <= N;
}

bool tc2_rows_supported(const Tc2RowsDesc &d) {
    if (knobs().dense_simt) return false;         // A/B switch for tests and profiling
    if (d.N < 16 || d.N > 256 || d.N % 16) return false;
    if (d.G < 1 || d.G > 2 || 2 * d.G * d.N > 512) return false;
    int steps = 0;
    for (int g = 0; g < d.G; ++g) {
        if (d.nseg[g] < 1 || d.nseg[g] > 2) return false;
        for (int q = 0; q < d.nseg[g]; ++q) {
            if (!seg_ok(d.seg[g][q])) return false;
            if (d.seg[g][q].mask_mode != kMask2None && (d.mask_width + 31) / 32 > 8) return false;
            steps += (d.seg[g][q].K + kChunk - 1) / kChunk;
        }
    }
    if (steps > kMaxSteps) return false;
    if (d.epi == kEpi2Dz && d.root && (d.root_k < 1 || d.root_k > 32 || (d.N - d.n_dz) % 16)) return false;
    if (d.epi == kEpi2Dz && d.n_dz % 16) return false;
    if (d.next_k && !tc2_next_drelu_supported(d.epi, d.N, d.next_k)) return false;
    const size_t bchunk = (size_t)256 * d.N;
    const size_t budget = (size_t)(kSmemBase - 4 * epi_warp_bytes(d.next_k > 0 || d.head_w) -
                                   (d.head_w ? 10 * 1024 : 0));
    return 2 * kStage + 2 * kMaskStage + 2 * bchunk <= budget;
}

int launch_tc2_rows(const Tc2RowsDesc &d, cudaStream_t s) {
    if (d.n <= 0) return 0;
    DR_CHECK(tc2_rows_supported(d), DR_ERR_UNSUPPORTED, "tc2_rows: unsupported shape");
    R2Args a{};
    a.n = d.n;
    a.N = d.N;
    a.G = d.G;
    a.S = 0;
    for (int g = 0; g < d.G; ++g) {
        a.bimg[g] = d.bimg[g];
        a.bias[g] = d.bias[g];
        int bc = 0;
        for (int q = 0; q < d.nseg[g]; ++q) {
            const Tc2Seg &sd = d.seg[g][q];
            a.seg[g][q] = R2Seg{sd.A, sd.hval, sd.hidx, sd.k, sd.K, sd.A ? sd.mask_mode : kMask2None,
                                sd.A && sd.split ? 1 : 0};
            if (sd.A && sd.split) make_tmap_split(&a.tmap[g][q], sd.A, d.n, sd.K);
            else if (sd.A) make_tmap(&a.tmap[g][q], sd.A, d.n, sd.K);
            const int chunks = (sd.K + kChunk - 1) / kChunk;
            for (int c = 0; c < chunks; ++c)
                a.step[a.S++] = R2Step{(int8_t)g, (int8_t)q, (int8_t)c, (int8_t)bc++,
                                       (int8_t)(q == 0 && c == 0)};
        }
    }
    a.mask_in = d.mask_in;
    a.mw = (d.mask_width + 31) / 32;
    a.bchunk = (uint32_t)(256 * d.N);
    a.epi = d.epi;
    a.merge = d.merge;
    a.y = d.y;
    a.mask_out = d.mask_out;
    a.tap_a = d.tap_a;
    a.tap_b = d.tap_b;
    a.n_dz = d.n_dz;
    a.crow = d.crow;
    a.dz = d.dz;
    a.root_idx = d.root_idx;
    a.root_k = d.root_k;
    a.root = d.root;
    a.head = d.head_w ? 1 : 0;
    a.head_w = d.head_w;
    a.head_b = d.head_b;
    a.labels = d.labels;
    a.head_inv_n = d.n > 0 ? 1.0f / (float)d.n : 0.f;
    a.head_dy = d.head_dy;
    a.head_part = d.head_part;
    DR_CHECK(!a.head || (d.G == 2 && d.epi == kEpi2Fwd && !d.next_k && d.head_b && d.labels &&
                         d.head_dy && d.head_part),
             DR_ERR_INVALID_ARGUMENT, "tc2_rows: bad fused-head arguments");
    a.nk = d.next_k;
    a.nk_stream = knobs().tpr_stream ? 1 : 0;
    a.nval = d.next_val;
    a.nidx = d.next_idx;
    DR_CHECK(!a.nk || (a.nval && a.nidx), DR_ERR_INVALID_ARGUMENT, "tc2_rows: null next CBSR");
    // stages: two epilogue warpgroups when B stays resident beside >= 3 A stages or
    // a ring of >= 2 B chunks fits beside 3; else one, with B resident beside >= 2
    // A stages or a ring. The fused-head variant's own static arrays (~9 KB) come
    // out of the same budget.
    const size_t st_bytes = kStage + kMaskStage;
    auto budget_for = [&](int ewg) {
        return (size_t)(kSmemBase - 4 * ewg * epi_warp_bytes(a.nk > 0 || a.head) - (a.head ? 10 * 1024 : 0));
    };
    size_t budget = budget_for(2);
    const bool res2 = (size_t)a.S * a.bchunk + 3 * st_bytes <= budget && a.S <= kMaxSB;
    const bool ring2 = 3 * st_bytes + 2 * (size_t)a.bchunk <= budget;
    // measured (C5, profiles/r03/ab_ewg.txt): two warpgroups shorten the fused head
    // (L1 cell 57.7 -> 53.6 us) and dZ' with the root-term columns, cost 1-2 us where
    // the 8 epilogue warps slow the converters on the same sub-partitions, and leave
    // the C5 step unchanged (23.37 k vs 23.45 k graphs/s): off by default (knob
    // tc2_ewg: 1 default, 0 auto = the head and dZ' with root, 2 forced)
    const bool heavy_epi = a.head || (a.epi == kEpi2Dz && a.root && a.N > a.n_dz);
    int want = knobs().tc2_ewg == 0 ? (heavy_epi ? 2 : 1) : (int)knobs().tc2_ewg;
    if (a.nk) want = 1;            // the 16-warp layout is built for the head and dZ' only
    a.ewg = (res2 || ring2) && want == 2 ? 2 : 1;
    if (a.ewg == 1) budget = budget_for(1);
    if (a.ewg == 2 && res2) {
        a.b_resident = 1;
        a.SB = a.S;
        a.SA = (int)std::min<size_t>(kMaxSA, (budget - (size_t)a.S * a.bchunk) / st_bytes);
    } else if (a.ewg == 2) {
        a.b_resident = 0;
        a.SA = 3;
        a.SB = (int)std::min<size_t>(4, (budget - 3 * st_bytes) / a.bchunk);
    } else if ((size_t)a.S * a.bchunk + 2 * st_bytes <= budget && a.S <= kMaxSB) {
        a.b_resident = 1;
        a.SB = a.S;
        a.SA = (int)std::min<size_t>(kMaxSA, (budget - (size_t)a.S * a.bchunk) / st_bytes);
    } else {
        a.b_resident = 0;
        a.SA = 3;
        if (3 * st_bytes + 2 * (size_t)a.bchunk > budget) a.SA = 2;
        a.SB = (int)std::min<size_t>(4, (budget - a.SA * st_bytes) / a.bchunk);
    }
    a.epi_off = (uint32_t)((a.SA * st_bytes + (size_t)a.SB * a.bchunk + 1023) / 1024 * 1024);
    const size_t smem = (size_t)a.epi_off + 4 * a.ewg * epi_warp_bytes(a.nk > 0 || a.head) + 1024;
    a.dz_split = d.dz_split ? 1 : 0;
    const int64_t tiles = (d.n + kTile - 1) / kTile;
    const int64_t grid = tiles < 148 ? tiles : 148;
    ProfScope ps(d.epi == kEpi2Dz ? "tc_dz" : "tc_proj", s);
    const bool w2 = a.ewg == 2;
    const void *fn = a.head ? (w2 ? (const void *)tc2_rows_kernel<-1, true>     // fused head (NK < 0)
                                  : (const void *)tc2_rows_kernel<-1, false>)
                   : a.nk == 1 ? (const void *)tc2_rows_kernel<1, false>
                   : a.nk == 2 ? (const void *)tc2_rows_kernel<2, false>
                   : a.nk == 4 ? (const void *)tc2_rows_kernel<4, false>
                   : a.nk == 8 ? (const void *)tc2_rows_kernel<8, false>
                   : a.nk == 16 ? (const void *)tc2_rows_kernel<16, false>
                   : a.nk == 32 ? (const void *)tc2_rows_kernel<32, false>
                   : w2 ? (const void *)tc2_rows_kernel<0, true>
                        : (const void *)tc2_rows_kernel<0, false>;
    ensure_smem(fn, smem);
    static unsigned long long *dbg_buf = nullptr;
    if (knobs().tc2_debug) {
        if (!dbg_buf) DR_CUDA(cudaMalloc(&dbg_buf, 148 * 16 * 8));
        DR_CUDA(cudaMemsetAsync(dbg_buf, 0, 148 * 16 * 8, s));
        a.dbg = dbg_buf;
    }
    {
        void *args[] = {(void *)&a};
        DR_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(w2 ? 512 : 320), args, smem, s));
    }
    note_launch("tc2_rows");
    if (a.dbg) {
        unsigned long long h[148 * 16];
        DR_CUDA(cudaStreamSynchronize(s));
        DR_CUDA(cudaMemcpy(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost));
        double t[16] = {0}, tmax = 0, smax = 0;
        unsigned long long g0 = ~0ull, g1 = 0, g0max = 0;
        for (int b = 0; b < grid; ++b) {
            for (int q = 0; q < 10; ++q) t[q] += (double)h[b * 16 + q] / grid;
            tmax = std::max(tmax, (double)h[b * 16 + 8]);
            smax = std::max(smax, (double)h[b * 16 + 10]);
            g0 = std::min(g0, h[b * 16 + 11]);
            g0max = std::max(g0max, h[b * 16 + 11]);
            g1 = std::max(g1, h[b * 16 + 12]);
        }
        fprintf(stderr, "[tc2_rows] max CTA kcycles %.1f, max setup kcycles %.1f, CTA start spread %.1f us, "
                "first start -> last end %.1f us\n", tmax / 1e3, smax / 1e3, (g0max - g0) / 1e3, (g1 - g0) / 1e3);
        fprintf(stderr,
                "[tc2_rows n=%lld N=%d G=%d S=%d SA=%d SB=%d res=%d ewg=%d epi=%d] kcycles/CTA: total %.1f | "
                "prod wait %.1f | mma wait conv %.1f acc %.1f | conv wait %.1f work %.1f | epi wait "
                "%.1f work %.1f\n",
                (long long)d.n, a.N, a.G, a.S, a.SA, a.SB, a.b_resident, a.ewg, a.epi, t[8] / 1e3,
                t[0] / 1e3, t[1] / 1e3, t[2] / 1e3, t[3] / 1e3, t[4] / 1e3, t[5] / 1e3, t[6] / 1e3);
    }
    return (int)grid;
}

// stage layout of the reduce kernel: [A'_g 32 KB each][B' 256 N][CBSR raw][mask words]
static void red_layout(const Tc2ReduceDesc &d, int ncb, int maxk, RdArgs &a) {
    auto r1k = [](uint32_t x) { return (x + 1023u) & ~1023u; };
    uint32_t off = (uint32_t)d.G * kStage;
    a.off_b = off;
    off += r1k((uint32_t)256 * d.N);
    a.off_b1 = off;
    if (d.mask_mode1 >= 0) off += r1k((uint32_t)256 * d.N);   // dual B: group 1's operand
    a.off_cbsr = off;
    a.cbsr_seg_bytes = (uint32_t)(kRRows * maxk * 4 + rup16((uint32_t)kRRows * maxk) + 16);
    a.cbsr_seg_bytes = (a.cbsr_seg_bytes + 127u) & ~127u;
    off += r1k(a.cbsr_seg_bytes * (uint32_t)ncb);
    a.off_mask = off;
    off += r1k(kRRows * 8 * 4 + 16);
    a.stage_bytes = off;
    a.SA = (int)std::min<size_t>(kMaxSA, (size_t)kSmemBudgetRed / a.stage_bytes);
}

// The specialised (MN-major) reduce shapes: 1 = [Z 64 | H 64] N 64, 2 = Z 128 / H 128
// in two groups N 128, 3 = Z 64 N 64, 4 = Z 128 N 128, 5 = dual B: [Z 64 | H 64] with
// B0 and split Z' 64 with B1, N 64; 0 = the generic kernel, -1 = unsupported dual.
static int red_variant(const Tc2ReduceDesc &d) {
    auto is_seg = [&](int g, int q, bool dense, int w) {
        return d.seg[g][q].w == w && (d.seg[g][q].Z != nullptr) == dense && (dense || d.seg[g][q].k <= 32);
    };
    if (d.mask_mode1 >= 0)
        return (d.G == 2 && d.nseg[0] == 2 && d.nseg[1] == 1 && d.N == 64 && is_seg(0, 0, true, 64) &&
                is_seg(0, 1, false, 64) && is_seg(1, 0, true, 64) && d.seg[0][0].split && d.seg[1][0].split &&
                d.mask && d.mask_mode != kMask2None)
                   ? 5 : -1;
    if (d.G == 1 && d.nseg[0] == 2 && d.N == 64 && is_seg(0, 0, true, 64) && is_seg(0, 1, false, 64)) return 1;
    if (d.G == 2 && d.nseg[0] == 1 && d.nseg[1] == 1 && d.N == 128 && is_seg(0, 0, true, 128) &&
        is_seg(1, 0, false, 128))
        return 2;
    if (d.G == 1 && d.nseg[0] == 1 && d.N == 64 && is_seg(0, 0, true, 64)) return 3;
    if (d.G == 1 && d.nseg[0] == 1 && d.N == 128 && is_seg(0, 0, true, 128)) return 4;
    return 0;
}

bool tc2_reduce_supported(const Tc2ReduceDesc &d) {
    if (knobs().dense_simt) return false;
    if (d.mask_mode1 >= 0 && red_variant(d) != 5) return false;
    if (d.N < 16 || d.N > 128 || d.N % 16) return false;
    if (d.G < 1 || d.G > 2) return false;
    for (int g = 0; g < d.G; ++g) {
        if (d.nseg[g] < 1 || d.nseg[g] > 2) return false;
        int w = 0, dense = 0, cb = 0;
        for (int q = 0; q < d.nseg[g]; ++q) {
            const Tc2RedSeg &s = d.seg[g][q];
            if (s.w < 4 || s.w % 4) return false;
            w += s.w;
            if (s.Z) ++dense;
            else {
                ++cb;
                if (s.k < 1 || s.k > 32 || s.k > s.w) return false;
            }
        }
        if (w > 128 || dense > 1 || cb > 1) return false;
        // split Z rows (TMA-loaded operand atoms) only on the MN-major shapes
        for (int q = 0; q < d.nseg[g]; ++q)
            if (d.seg[g][q].Z && d.seg[g][q].split && red_variant(d) == 0) return false;
    }
    if (d.mask_mode != kMask2None && (d.N + 31) / 32 > 8) return false;
    int ncb = 0, maxk = 0;
    for (int g = 0; g < d.G; ++g)
        for (int q = 0; q < d.nseg[g]; ++q)
            if (!d.seg[g][q].Z) {
                ++ncb;
                maxk = std::max(maxk, d.seg[g][q].k);
            }
    RdArgs a{};
    red_layout(d, ncb, maxk, a);
    return a.SA >= 2;
}

size_t tc2_reduce_work_floats(int G, int N) {
    return (size_t)148 * ((size_t)G * kTile * N + 2 * (size_t)N);    // up to two db vectors (dual B)
}

void launch_tc2_reduce(const Tc2ReduceDesc &d, float *work, cudaStream_t s, Tc2Deferred *defer) {
    DR_CHECK(tc2_reduce_supported(d), DR_ERR_UNSUPPORTED, "tc2_reduce: unsupported shape");
    RdArgs a{};
    a.n = d.n;
    a.N = d.N;
    a.G = d.G;
    Tc2PartsJob o{};
    int ncb = 0, maxk = 0;
    for (int g = 0; g < d.G; ++g) {
        a.nseg[g] = d.nseg[g];
        int m0 = 0;
        for (int q = 0; q < d.nseg[g]; ++q) {
            const Tc2RedSeg &sd = d.seg[g][q];
            a.seg[g][q] = RdSeg{sd.Z, sd.hval, sd.hidx, sd.k, sd.w, m0, sd.Z && sd.split ? 1 : 0};
            if (sd.Z && sd.split) make_tmap_split(&a.zmap[g][q], sd.Z, d.n, sd.w, kRRows);
            if (!sd.Z) {
                ++ncb;
                maxk = std::max(maxk, sd.k);
            }
            o.g[o.nout] = g;
            o.m0[o.nout] = m0;
            o.w[o.nout] = sd.w;
            o.dst[o.nout] = sd.grad;
            ++o.nout;
            m0 += sd.w;
        }
    }
    o.db = d.db;
    o.db1 = d.db1;
    o.ndb = d.mask_mode1 >= 0 ? 2 : 1;
    a.dy = d.dy;
    a.mask = d.mask;
    a.mask_mode = d.mask_mode;
    a.mask_mode1 = d.mask_mode1;
    a.ndb = o.ndb;
    a.mw = (d.N + 31) / 32;
    red_layout(d, ncb, maxk, a);
    DR_CHECK(a.SA >= 2, DR_ERR_UNSUPPORTED, "tc2_reduce: shared memory budget");
    const size_t smem = (size_t)a.SA * a.stage_bytes + 1024;
    int64_t grid = (d.n + 4 * kRRows - 1) / (4 * kRRows);
    if (grid > 148) grid = 148;
    if (grid < 1) grid = 1;
    a.rows_per_cta = ((d.n + grid - 1) / grid + kRRows - 1) / kRRows * kRRows;
    a.part = work;
    ProfScope ps("tc_dw", s);
    static unsigned long long *dbg_buf = nullptr;
    if (knobs().tc2_debug) {
        if (!dbg_buf) DR_CUDA(cudaMalloc(&dbg_buf, 148 * 16 * 8));
        DR_CUDA(cudaMemsetAsync(dbg_buf, 0, 148 * 16 * 8, s));
        a.dbg = dbg_buf;
    }
    // specialised converters for the square-layer shapes; generic otherwise
    const int var = red_variant(d);
    const void *fn = var == 1 ? (const void *)tc2_reduce_kernel<1, 64, 64, 64>
                   : var == 2 ? (const void *)tc2_reduce_kernel<2, 128, 128, 128>
                   : var == 3 ? (const void *)tc2_reduce_kernel<1, 64, 0, 64>
                   : var == 4 ? (const void *)tc2_reduce_kernel<1, 128, 0, 128>
                   : var == 5 ? (const void *)tc2_reduce_kernel<3, 64, 64, 64>
                              : (const void *)tc2_reduce_kernel<0, 0, 0, 0>;
    ensure_smem(fn, smem);
    {
        void *args[] = {(void *)&a};
        DR_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kRedThreads), args, smem, s));
    }
    note_launch("tc2_reduce");
    if (a.dbg) {
        unsigned long long h[148 * 16];
        DR_CUDA(cudaStreamSynchronize(s));
        DR_CUDA(cudaMemcpy(h, dbg_buf, sizeof(h), cudaMemcpyDeviceToHost));
        double t[16] = {0};
        for (int b = 0; b < grid; ++b)
            for (int q = 0; q < 16; ++q) t[q] += (double)h[b * 16 + q] / grid;
        fprintf(stderr,
                "[tc2_reduce n=%lld N=%d G=%d SA=%d stage=%u rows/cta=%lld] kcycles/CTA: total %.1f | "
                "prod wait empty %.1f | mma wait conv %.1f | conv wait full %.1f work %.1f\n",
                (long long)d.n, a.N, a.G, a.SA, a.stage_bytes, (long long)a.rows_per_cta, t[8] / 1e3,
                t[0] / 1e3, t[1] / 1e3, t[2] / 1e3, t[3] / 1e3);
    }
    o.part = work;
    o.nparts = (int)grid;
    o.G = d.G;
    o.N = d.N;
    if (defer) {
        DR_CHECK(defer->n < Tc2Deferred::kMax, DR_ERR_INVALID_ARGUMENT, "tc2_reduce: too many deferred");
        defer->job[defer->n++] = o;
        return;
    }
    Tc2Deferred one;
    one.job[one.n++] = o;
    launch_tc2_reduce_parts(one, s);
}

void launch_tc2_reduce_parts(Tc2Deferred &defer, cudaStream_t s) {
    if (defer.n == 0) return;
    PartsJobs j{};
    int64_t most = 1;
    for (int i = 0; i < defer.n; ++i) {
        j.job[i] = defer.job[i];
        most = std::max<int64_t>(most, (int64_t)defer.job[i].G * kTile * defer.job[i].N +
                                           (int64_t)defer.job[i].ndb * defer.job[i].N);
    }
    ProfScope ps("tc_dw_sum", s);
    tc2_reduce_parts_kernel<<<dim3((unsigned)((most + 31) / 32), (unsigned)defer.n), dim3(32, 8), 0, s>>>(j);
    note_launch("tc2_reduce_parts");
    defer.n = 0;
}

}  // namespace dr

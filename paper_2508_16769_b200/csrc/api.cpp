// api.cpp — the C ABI of include/dr.h: validation, the HeteroConv layer
// orchestration over three CUDA streams (§3.4), the training step
// and the NCCL bootstrap. Every compute step runs in this library's kernels.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_map>

#include <nvtx3/nvToolsExt.h>

#include "nccl_api.h"
#include "proj.h"
#include "tc2.h"

namespace dr {

// ------------------------------------------------------------------ errors & bookkeeping
static thread_local std::string t_err;
static thread_local int64_t t_launches = 0;

void set_error(dr_status s, const std::string &msg) {
    t_err = std::string(dr_status_str(s)) + ": " + msg;
}
void clear_error() { t_err.clear(); }
void fail(dr_status s, const std::string &msg) { throw Error{s, msg}; }

void note_launch(const char *name) {
    ++t_launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(DR_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ profiling
struct ProfRec {
    std::string name;
    cudaEvent_t a, b;
};
static thread_local bool t_prof = false;
static thread_local std::vector<ProfRec> t_recs;
static thread_local std::vector<cudaEvent_t> t_pool;
static thread_local std::string t_tag;

static cudaEvent_t pool_get() {
    if (!t_pool.empty()) {
        cudaEvent_t e = t_pool.back();
        t_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    DR_CUDA(cudaEventCreate(&e));
    return e;
}

// DR_NVTX=1: every launch is wrapped in an NVTX range named "<base>.<tag>", so
// `ncu --nvtx --print-nvtx-rename kernel` reports per-tag kernel metrics (the
// DRAM traffic of profiles/ncu_traffic.json). Off by default (no overhead).
static bool nvtx_on() { return knobs().nvtx != 0; }

ProfScope::ProfScope(const char *b, cudaStream_t st) {
    if (nvtx_on()) {
        const std::string name = t_tag.empty() ? std::string(b) : std::string(b) + "." + t_tag;
        nvtxRangePushA(name.c_str());
        nvtx = true;
    }
    if (!t_prof) return;
    s = st;
    base = b;
    a = pool_get();
    DR_CUDA(cudaEventRecord(a, s));
}

ProfScope::~ProfScope() {
    if (nvtx) nvtxRangePop();
    if (!a) return;
    cudaEvent_t e = nullptr;
    try {
        e = pool_get();
    } catch (...) {
        return;
    }
    cudaEventRecord(e, s);
    t_recs.push_back({t_tag.empty() ? std::string(base) : std::string(base) + "." + t_tag, a, e});
}

TagScope::TagScope(const char *tag) : prev(t_tag) {
    t_tag = prev.empty() ? std::string(tag) : prev + "." + tag;
}
TagScope::~TagScope() { t_tag = prev; }

// cudaFuncSetAttribute applies to the current device's context only: the cache
// is keyed on (device, kernel) so a process driving several GPUs sets it per device
void ensure_smem(const void *fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> set;
    if (bytes <= 48 * 1024) return;
    int dev = 0;
    DR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    size_t &cur = set[{dev, fn}];
    if (bytes > cur) {
        DR_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        cur = bytes;
    }
}

// Per-host-thread helper streams/events for the 3-stream fork/join.
struct StreamCtx {
    int device = -1;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};
    cudaStream_t cap = nullptr;                  // private capture stream (CUDA graphs)
    cudaEvent_t fork = nullptr, ev[6] = {};
};
static thread_local StreamCtx t_ctx;

static StreamCtx &ctx() {
    int dev = 0;
    DR_CUDA(cudaGetDevice(&dev));
    if (t_ctx.device != dev) {
        if (t_ctx.device >= 0) {
            // previous device's objects: leave them (rare; device switches per thread)
        }
        for (int q = 0; q < 3; ++q) DR_CUDA(cudaStreamCreateWithFlags(&t_ctx.s[q], cudaStreamNonBlocking));
        DR_CUDA(cudaStreamCreateWithFlags(&t_ctx.cap, cudaStreamNonBlocking));
        DR_CUDA(cudaEventCreateWithFlags(&t_ctx.fork, cudaEventDisableTiming));
        for (int q = 0; q < 6; ++q) DR_CUDA(cudaEventCreateWithFlags(&t_ctx.ev[q], cudaEventDisableTiming));
        t_ctx.device = dev;
    }
    return t_ctx;
}

static void wait_on(cudaStream_t waiter, cudaStream_t producer, cudaEvent_t ev) {
    if (waiter == producer) return;
    DR_CUDA(cudaEventRecord(ev, producer));
    DR_CUDA(cudaStreamWaitEvent(waiter, ev, 0));
}

// Between dr_profile_begin and dr_profile_end every layer runs on the caller's
// stream, so the per-launch events time isolated kernels (results are
// bit-identical either way).
static bool force_sequential() { return t_prof || knobs().seq_streams; }

static bool is_pow2(int k) { return k > 0 && (k & (k - 1)) == 0; }

static void check_k(int k, int dim, const char *what) {
    DR_CHECK(dim >= 1 && dim <= 256 && dim % 4 == 0, DR_ERR_SHAPE_MISMATCH,
             std::string(what) + ": dim must be a multiple of 4 in [4, 256]");
    DR_CHECK(k >= 1 && k <= dim && k <= 128 && is_pow2(k), DR_ERR_BAD_K,
             std::string(what) + ": k must be a power of two with 1 <= k <= min(dim, 128)");
}

static void check_cbsr(const dr_cbsr *h, const char *what) {
    DR_CHECK(h != nullptr, DR_ERR_INVALID_ARGUMENT, std::string(what) + ": null cbsr");
    DR_CHECK(h->idx_bytes == 1, DR_ERR_UNSUPPORTED, std::string(what) + ": idx_bytes must be 1");
    DR_CHECK(h->n >= 0, DR_ERR_INVALID_ARGUMENT, std::string(what) + ": negative n");
    DR_CHECK(h->n == 0 || (h->idx && h->val), DR_ERR_INVALID_ARGUMENT,
             std::string(what) + ": null cbsr buffers");
    check_k(h->k, h->dim, what);
}

static void check_out_width(int n, const char *what) {
    DR_CHECK(n >= 4 && n <= 256 && n % 4 == 0 && (n % 32 == 0 || n == 4 || n == 8 || n == 16),
             DR_ERR_SHAPE_MISMATCH,
             std::string(what) + ": width must be 4, 8, 16 or a multiple of 32 up to 256");
}

// ------------------------------------------------------------------ tape layout
// per-edge-type k (Q27): pins' source CBSR width; == k_cell shares H_c
static int k_pins_of(const dr_layer *L) { return L->k_pins ? L->k_pins : L->k_cell; }
static bool pins_own(const dr_layer *L) { return k_pins_of(L) != L->k_cell; }

struct TapeLayout {
    size_t hc_val, hc_idx, hn_val, hn_idx, hp_val, hp_idx, z[3], mask, tap_a, tap_b;
    size_t dz[3], root_c, root_n, work[3];
    size_t img_fa, img_fb, img_fn, img_dz[3];     // packed tcgen05 B operands
    size_t total;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static TapeLayout tape_layout(const dr_graph *g, const dr_layer *L, uint32_t flags) {
    TapeLayout t{};
    const size_t nc = (size_t)g->n_cell, nn = (size_t)g->n_net;
    const size_t dc = L->d_cell, dn = L->d_net, D = L->d_out, kc = L->k_cell, kn = L->k_net;
    size_t off = 0;
    auto put = [&](size_t bytes) { size_t o = off; off += al(bytes); return o; };
    t.hc_val = put(nc * kc * 4);
    t.hc_idx = put(nc * kc);
    t.hn_val = put(nn * kn * 4);
    t.hn_idx = put(nn * kn);
    const size_t kp = (size_t)k_pins_of(L);
    t.hp_val = pins_own(L) ? put(nc * kp * 4) : t.hc_val;
    t.hp_idx = pins_own(L) ? put(nc * kp) : t.hc_idx;
    t.z[DR_NEAR] = put(nc * dc * 4);
    t.z[DR_PINS] = put(nn * dc * 4);
    t.z[DR_PINNED] = put(nc * dn * 4);
    t.mask = put(nc * ((D + 31) / 32) * 4);
    t.tap_a = (flags & DR_FWD_TAPS) ? put(nc * D * 4) : (size_t)-1;
    t.tap_b = (flags & DR_FWD_TAPS) ? put(nc * D * 4) : (size_t)-1;
    t.dz[DR_NEAR] = put(nc * dc * 4);
    t.dz[DR_PINS] = put(nn * dc * 4);
    t.dz[DR_PINNED] = put(nc * dn * 4);
    t.root_c = put(nc * kc * 4);
    t.root_n = put(nn * kn * 4);
    auto mx = [](size_t a, size_t b) { return a > b ? a : b; };
    const size_t red = tc2_reduce_work_floats(2, (int)D);
    t.work[0] = put(mx(dw_part_floats(nc, (int)dc, (int)D), red) * 4);
    t.work[1] = put(mx(mx(dw_part_floats(nn, (int)dc, (int)D), dw_part_floats(nn, (int)dn, (int)D)), red) * 4);
    t.work[2] = put(mx(dw_part_floats(nc, (int)dn, (int)D), red) * 4);
    // packed B operands of the tensor-core GEMMs (tc2.h)
    t.img_fa = put(tc2_bimg_bytes((int)dc, (int)D) * 2);
    t.img_fb = put(tc2_bimg_bytes((int)dn, (int)D));
    t.img_fn = put(tc2_bimg_bytes((int)dc, (int)D) + tc2_bimg_bytes((int)dn, (int)D));
    t.img_dz[DR_NEAR] = put(tc2_bimg_bytes((int)D, (int)(2 * dc)));
    t.img_dz[DR_PINS] = put(tc2_bimg_bytes((int)D, (int)(dc + dn)));
    t.img_dz[DR_PINNED] = put(tc2_bimg_bytes((int)D, (int)dn));
    t.total = off;
    return t;
}

static void check_layer(const dr_graph *g, const dr_layer *L) {
    DR_CHECK(g && L, DR_ERR_INVALID_ARGUMENT, "null graph/layer");
    check_k(L->k_cell, L->d_cell, "layer k_cell/d_cell");
    check_k(L->k_net, L->d_net, "layer k_net/d_net");
    DR_CHECK(L->k_pins >= 0, DR_ERR_BAD_K, "layer: negative k_pins");
    check_k(k_pins_of(L), L->d_cell, "layer k_pins/d_cell");
    check_out_width(L->d_out, "layer d_out");
    check_out_width(L->d_cell, "layer d_cell");
    check_out_width(L->d_net, "layer d_net");
    for (int r = 0; r < 3; ++r)
        DR_CHECK(L->wn[r] && L->b[r], DR_ERR_INVALID_ARGUMENT, "layer: null wn/b");
    DR_CHECK(L->wr[DR_PINNED] == nullptr, DR_ERR_UNSUPPORTED, "layer: wr[PINNED] must be NULL");
    DR_CHECK(L->merge == DR_MERGE_MAX || L->merge == DR_MERGE_SUM, DR_ERR_INVALID_ARGUMENT,
             "layer: bad merge");
}

// Z of relation r in the tape as split bf16 rows ([hi | lo], x = hi + lo with the
// same rounding as the converters'): the SpMM epilogues write them, and both
// consumers TMA-load them as ready operand tiles -- the projection (K-major
// SW128) and the dW reduce GEMM (MN-major atoms) -- with no conversion. On for
// the square layers whose consumers take that path (every width 64 or 128,
// k <= 32 CBSR roots); bit-identical to converting fp32 Z.
static bool z_split_ok(const dr_layer *L, int) {
    if (knobs().dense_simt || !knobs().z_split) return false;
    const int D = L->d_out;
    return (D == 64 || D == 128) && L->d_cell == D && L->d_net == D && L->k_cell <= 32 &&
           L->k_net <= 32;
}

// f4, a layer over dr_shards (dr_shard_layer_*): this rank's destination rows,
// every source row read in place from its owner (peer memory), every per-source
// backward contribution written in place into its owner's inbox
struct ShardCtx {
    PeerSrc cell, net;                 // all ranks' local CBSR (pv / pi)
    PeerSrc near_g, pins_g, pinned_g;  // + the inbox slots each relation writes (pg)
    int rank;
};

// ------------------------------------------------------------------ layer forward / backward
// Ln / tape_next (row a5): the next layer and its tape; when given, the
// projection epilogues also write the next layer's input CBSR (Eq. 2-3 on Y_cell
// after the merge and on Y_net) into tape_next (flags_next = that tape's flags).
// DR_FWD_INPUT_IN_TAPE: this layer's H_c / H_n are already in `tape` (written so
// by the previous layer); its own D-ReLU launches are skipped.
// DR_FWD_Y_SCRATCH: y_cell / y_net need not be written when the fused epilogue
// covers the shape (they are still written, and D-ReLU'd standalone, otherwise).
static void heteroconv_fwd(const dr_graph *g, const dr_layer *L, const float *xc, const float *xn,
                           float *yc, float *yn, void *tape, uint32_t flags, cudaStream_t st,
                           const dr_layer *Ln = nullptr, void *tape_next = nullptr,
                           uint32_t flags_next = 0, const HeadArgs *head = nullptr,
                           int *head_parts = nullptr, const ShardCtx *sh = nullptr) {
    if (head_parts) *head_parts = 0;
    const TapeLayout T = tape_layout(g, L, flags);
    const bool in_tape = (flags & DR_FWD_INPUT_IN_TAPE) != 0 || sh != nullptr;
    DR_CHECK(!sh || (!Ln && !head && !pins_own(L)), DR_ERR_UNSUPPORTED,
             "sharded layer: no chaining, fused head or k_pins");
    TapeLayout TN{};
    char *tn = (char *)tape_next;
    if (Ln) TN = tape_layout(g, Ln, flags_next);
    // fused next-layer D-ReLU per output type, or the standalone fallback
    const bool fuse_c = Ln && tc2_next_drelu_supported(kEpi2Fwd, L->d_out, Ln->k_cell);
    const bool fuse_n = Ln && tc2_next_drelu_supported(kEpi2Fwd, L->d_out, Ln->k_net);
    const bool y_scratch = (flags & DR_FWD_Y_SCRATCH) != 0;
    // DR_FWD_NO_NET_OUT: Y_net feeds nothing (the last layer: the head reads
    // cells only, Q14) -- the pins SpMM and the net projection are not run
    const bool no_net = (flags & DR_FWD_NO_NET_OUT) != 0;
    DR_CHECK(!no_net || !Ln, DR_ERR_INVALID_ARGUMENT, "DR_FWD_NO_NET_OUT with a next layer");
    DR_CHECK(!in_tape || !pins_own(L), DR_ERR_UNSUPPORTED,
             "DR_FWD_INPUT_IN_TAPE with k_pins: pins' own CBSR needs the dense input");
    DR_CHECK(!Ln || !pins_own(Ln), DR_ERR_UNSUPPORTED,
             "chained forward into a layer with k_pins: its pins CBSR needs the dense input");
    char *tp = (char *)tape;
    float *hcv = (float *)(tp + T.hc_val), *hnv = (float *)(tp + T.hn_val);
    uint8_t *hci = (uint8_t *)(tp + T.hc_idx), *hni = (uint8_t *)(tp + T.hn_idx);
    if (sh) {          // this rank's own CBSR (its rows are the local rows)
        hcv = const_cast<float *>(sh->cell.pv[sh->rank]);
        hci = const_cast<uint8_t *>(sh->cell.pi[sh->rank]);
        hnv = const_cast<float *>(sh->net.pv[sh->rank]);
        hni = const_cast<uint8_t *>(sh->net.pi[sh->rank]);
    }
    float *hpv = sh ? hcv : (float *)(tp + T.hp_val);
    uint8_t *hpi = sh ? hci : (uint8_t *)(tp + T.hp_idx);
    const int kp = k_pins_of(L);
    float *z[3];
    for (int r = 0; r < 3; ++r) z[r] = (float *)(tp + T.z[r]);
    const int nc = g->n_cell, nn = g->n_net;
    bool zs[3];
    for (int r = 0; r < 3; ++r) zs[r] = !sh && z_split_ok(L, r);
    const PeerSrc *pc = sh ? &sh->cell : nullptr, *pn = sh ? &sh->net : nullptr;
    // ---- the two projections (tensor-core row GEMMs when the shapes allow) and
    // their packed weight images, packed by ONE launch before the streams fork
    Tc2RowsDesc dnet, dcell;
    {   // net: Y_net = Z_pins Wn_pins + densify(H_n) Wr_pins + b_pins   (Eq. 7, 9)
        Tc2RowsDesc &d = dnet;
        d.n = nn; d.N = L->d_out; d.G = 1; d.epi = kEpi2Fwd;
        d.nseg[0] = L->wr[DR_PINS] ? 2 : 1;
        d.seg[0][0].A = z[DR_PINS]; d.seg[0][0].K = L->d_cell; d.seg[0][0].split = zs[DR_PINS];
        d.seg[0][1].hval = hnv; d.seg[0][1].hidx = hni; d.seg[0][1].k = L->k_net;
        d.seg[0][1].K = L->d_net;
        d.bimg[0] = (uint8_t *)(tp + T.img_fn); d.bias[0] = L->b[DR_PINS];
        d.y = yn;
        if (fuse_n) {
            d.next_k = Ln->k_net;
            d.next_val = (float *)(tn + TN.hn_val);
            d.next_idx = (uint8_t *)(tn + TN.hn_idx);
            if (y_scratch) d.y = nullptr;
        }
        if (!tc2_rows_supported(d)) {          // dense y + standalone D-ReLU
            d.next_k = 0;
            d.y = yn;
        }
    }
    {   // cell: Y_cell = max(Y_near, Y_pinned), M   (Eq. 6, 8, 14)
        Tc2RowsDesc &d = dcell;
        d.n = nc; d.N = L->d_out; d.G = 2; d.epi = kEpi2Fwd;
        d.nseg[0] = L->wr[DR_NEAR] ? 2 : 1;
        d.seg[0][0].A = z[DR_NEAR]; d.seg[0][0].K = L->d_cell; d.seg[0][0].split = zs[DR_NEAR];
        d.seg[0][1].hval = hcv; d.seg[0][1].hidx = hci; d.seg[0][1].k = L->k_cell;
        d.seg[0][1].K = L->d_cell;
        d.nseg[1] = 1;
        d.seg[1][0].A = z[DR_PINNED]; d.seg[1][0].K = L->d_net; d.seg[1][0].split = zs[DR_PINNED];
        d.bimg[0] = (uint8_t *)(tp + T.img_fa); d.bimg[1] = (uint8_t *)(tp + T.img_fb);
        d.bias[0] = L->b[DR_NEAR]; d.bias[1] = L->b[DR_PINNED];
        d.merge = L->merge;
        d.y = yc; d.mask_out = (uint32_t *)(tp + T.mask);
        d.tap_a = (flags & DR_FWD_TAPS) ? (float *)(tp + T.tap_a) : nullptr;
        d.tap_b = (flags & DR_FWD_TAPS) ? (float *)(tp + T.tap_b) : nullptr;
        if (fuse_c) {
            d.next_k = Ln->k_cell;
            d.next_val = (float *)(tn + TN.hc_val);
            d.next_idx = (uint8_t *)(tn + TN.hc_idx);
            if (y_scratch) d.y = nullptr;
        }
        if (head && !Ln) {     // the last layer: linear head + MSE in the epilogue, Y not stored
            d.head_w = head->w; d.head_b = head->b; d.labels = head->labels;
            d.head_dy = head->dy; d.head_part = head->work;
            d.y = nullptr;
        }
        if (!tc2_rows_supported(d)) {
            d.next_k = 0;
            d.y = yc;
            d.head_w = nullptr;
        }
    }
    const bool net_tc = !no_net && nn > 0 && tc2_rows_supported(dnet);
    const bool cell_tc = nc > 0 && tc2_rows_supported(dcell);
    {
        Tc2PackJob jobs[kMaxPackJobs];
        int nj = 0;
        auto job = [&](const float *W, int K, uint8_t *img) {   // B_op[n][kk] = W[kk][n]
            Tc2PackJob &j = jobs[nj++];
            j.W = W; j.ldw = L->d_out; j.K = K; j.NB = L->d_out; j.n0 = 0; j.Ntot = L->d_out;
            j.transpose = 1; j.img = img;
        };
        if (net_tc) {
            job(L->wn[DR_PINS], L->d_cell, (uint8_t *)dnet.bimg[0]);
            if (L->wr[DR_PINS])
                job(L->wr[DR_PINS], L->d_net, (uint8_t *)dnet.bimg[0] + tc2_bimg_bytes(L->d_cell, L->d_out));
        }
        if (cell_tc) {
            job(L->wn[DR_NEAR], L->d_cell, (uint8_t *)dcell.bimg[0]);
            if (L->wr[DR_NEAR])
                job(L->wr[DR_NEAR], L->d_cell, (uint8_t *)dcell.bimg[0] + tc2_bimg_bytes(L->d_cell, L->d_out));
            job(L->wn[DR_PINNED], L->d_net, (uint8_t *)dcell.bimg[1]);
        }
        launch_tc2_pack_b_multi(jobs, nj, st);
    }
    const bool seq = (flags & DR_FWD_SEQUENTIAL) != 0 || force_sequential();
    StreamCtx &C = ctx();
    cudaStream_t s0 = seq ? st : C.s[0], s1 = seq ? st : C.s[1], s2 = seq ? st : C.s[2];
    if (!seq) {
        DR_CUDA(cudaEventRecord(C.fork, st));
        for (int q = 0; q < 3; ++q) DR_CUDA(cudaStreamWaitEvent(C.s[q], C.fork, 0));
    }
    if (!in_tape) { TagScope t("cell"); launch_drelu(xc, nc, L->d_cell, L->d_cell, L->k_cell, hcv, hci, s0); }  // Eq. 2-3
    if (!seq) DR_CUDA(cudaEventRecord(C.ev[0], s0));                               // H_c ready
    if (!in_tape) { TagScope t("net"); launch_drelu(xn, nn, L->d_net, L->d_net, L->k_net, hnv, hni, s2); }
    if (!seq) DR_CUDA(cudaEventRecord(C.ev[1], s2));                               // H_n ready
    { TagScope t("near"); launch_spmm_fwd(g->rel[DR_NEAR], hcv, hci, L->k_cell, L->d_cell, z[DR_NEAR], s0, zs[DR_NEAR], NgSched{}, pc); }  // Eq. 5-7
    if (pins_own(L)) {          // Q27: pins' own cell CBSR, on its own stream
        TagScope t("pins");
        launch_drelu(xc, nc, L->d_cell, L->d_cell, kp, hpv, hpi, s1);
    } else if (!seq) {
        DR_CUDA(cudaStreamWaitEvent(s1, C.ev[0], 0));
    }
    if (!no_net) { TagScope t("pins"); launch_spmm_fwd(g->rel[DR_PINS], hpv, hpi, kp, L->d_cell, z[DR_PINS], s1, zs[DR_PINS], NgSched{}, pc); }
    { TagScope t("pinned"); launch_spmm_fwd(g->rel[DR_PINNED], hnv, hni, L->k_net, L->d_net, z[DR_PINNED], s2, zs[DR_PINNED], NgSched{}, pn); }
    if (!seq) DR_CUDA(cudaEventRecord(C.ev[2], s2));                               // Z_pinned ready
    if (!seq) DR_CUDA(cudaStreamWaitEvent(s1, C.ev[1], 0));
    if (!no_net) {   // net: Y_net = Z_pins Wn_pins + densify(H_n) Wr_pins + b_pins   (Eq. 7, 9)
        TagScope t("net");
        if (net_tc) {
            launch_tc2_rows(dnet, s1);
        } else {
            ProjFwdArgs a;
            a.n = nn; a.Ka = L->d_cell; a.N = L->d_out;
            a.Za = z[DR_PINS]; a.Wa = L->wn[DR_PINS]; a.ba = L->b[DR_PINS];
            a.Wr = L->wr[DR_PINS]; a.hval = hnv; a.hidx = hni; a.k = L->k_net;
            a.y = yn;
            DR_CHECK(!zs[DR_PINS], DR_ERR_UNSUPPORTED, "projection: split Z needs tc2");
            launch_proj_fwd(a, s1);
        }
        if (Ln && !dnet.next_k)                 // next layer's H_n from the dense Y_net
            launch_drelu(yn, nn, L->d_out, L->d_out, Ln->k_net, (float *)(tn + TN.hn_val),
                         (uint8_t *)(tn + TN.hn_idx), s1);
    }
    if (!seq) DR_CUDA(cudaStreamWaitEvent(s0, C.ev[2], 0));
    {   // cell: Y_cell = max(Y_near, Y_pinned), M   (Eq. 6, 8, 14)
        TagScope t("cell");
        if (cell_tc) {
            const int grid = launch_tc2_rows(dcell, s0);
            if (dcell.head_w && head_parts) *head_parts = grid;
        } else {
            ProjFwdArgs a;
            a.n = nc; a.Ka = L->d_cell; a.Kb = L->d_net; a.N = L->d_out;
            a.Za = z[DR_NEAR]; a.Wa = L->wn[DR_NEAR]; a.ba = L->b[DR_NEAR];
            a.Wr = L->wr[DR_NEAR]; a.hval = hcv; a.hidx = hci; a.k = L->k_cell;
            a.Zb = z[DR_PINNED]; a.Wb = L->wn[DR_PINNED]; a.bb = L->b[DR_PINNED];
            a.merge = L->merge;
            a.y = yc;
            a.mask = (uint32_t *)(tp + T.mask);
            a.tap_a = dcell.tap_a;
            a.tap_b = dcell.tap_b;
            DR_CHECK(!zs[DR_NEAR] && !zs[DR_PINNED], DR_ERR_UNSUPPORTED, "projection: split Z needs tc2");
            launch_proj_fwd(a, s0);
        }
        if (Ln && !dcell.next_k)                // next layer's H_c from the dense Y_cell
            launch_drelu(yc, nc, L->d_out, L->d_out, Ln->k_cell, (float *)(tn + TN.hc_val),
                         (uint8_t *)(tn + TN.hc_idx), s0);
    }
    if (!seq) {
        wait_on(st, s0, C.ev[3]);
        wait_on(st, s1, C.ev[4]);
        wait_on(st, s2, C.ev[5]);
    }
}

// defer: queue the weight gradients' fixed-order partial sums there (the caller
// launches them once for several layers); nullptr: one launch at the end here
static void heteroconv_bwd(const dr_graph *g, const dr_layer *L, void *tape, const float *dyc,
                           const float *dyn, float *dxc, float *dxn, dr_layer_grad *G,
                           uint32_t flags, cudaStream_t st, Tc2Deferred *defer = nullptr,
                           const ShardCtx *sh = nullptr) {
    Tc2Deferred own_parts;
    Tc2Deferred *pq = defer ? defer : &own_parts;
    const TapeLayout T = tape_layout(g, L, flags);
    char *tp = (char *)tape;
    const float *hcv = (float *)(tp + T.hc_val), *hnv = (float *)(tp + T.hn_val);
    const uint8_t *hci = (uint8_t *)(tp + T.hc_idx), *hni = (uint8_t *)(tp + T.hn_idx);
    if (sh) {
        hcv = sh->cell.pv[sh->rank];
        hci = sh->cell.pi[sh->rank];
        hnv = sh->net.pv[sh->rank];
        hni = sh->net.pi[sh->rank];
    }
    const uint8_t *hpi = (uint8_t *)(tp + T.hp_idx);
    const int kp = k_pins_of(L);
    const bool own = pins_own(L);
    const uint32_t *mask = (uint32_t *)(tp + T.mask);
    float *z[3], *dz[3];
    for (int r = 0; r < 3; ++r) {
        z[r] = (float *)(tp + T.z[r]);
        dz[r] = (float *)(tp + T.dz[r]);
    }
    float *root_c = (float *)(tp + T.root_c), *root_n = (float *)(tp + T.root_n);
    float *work[3];
    for (int q = 0; q < 3; ++q) work[q] = (float *)(tp + T.work[q]);
    const int mode_near = L->merge == DR_MERGE_MAX ? kMaskM : kMaskNone;        // Eq. 12
    const int mode_pinned = L->merge == DR_MERGE_MAX ? kMaskNotM : kMaskNone;   // Eq. 13
    const int nc = g->n_cell, nn = g->n_net, D = L->d_out;
    // ---- dZ' row GEMMs: descriptors and their packed weights (B_op[n][kk] = W[n][kk],
    // Wn in columns [0, Kd), the Sage root weight Wr in [Kd, N)), one packing launch
    const RelDev &rn = g->rel[DR_NEAR];
    const bool near_tiled = !sh && dxc && !rn.ewT && rn.n_src == nc &&
                            tspmm_supported(rn.tilesT, L->d_cell, L->k_cell);
    Tc2RowsDesc dzd[3];
    bool dz_tc[3] = {false, false, false};
    if (dxc || dxn) {
        Tc2PackJob jobs[kMaxPackJobs];
        int nj = 0;
        auto prep = [&](int r, int64_t n, int Kd, const float *dy, int mode, const float *W,
                        const float *Wr, int Kr, const uint8_t *ridx, int rk, float *root,
                        const float *c, bool split) {
            Tc2RowsDesc &d = dzd[r];
            d.n = n; d.N = Kd + (Wr ? Kr : 0); d.G = 1; d.epi = kEpi2Dz;
            d.nseg[0] = 1;
            d.seg[0][0].A = dy; d.seg[0][0].K = D; d.seg[0][0].mask_mode = mode;
            d.mask_in = mask; d.mask_width = D;
            d.bimg[0] = (uint8_t *)(tp + T.img_dz[r]); d.n_dz = Kd; d.crow = c; d.dz = dz[r];
            d.dz_split = split;   // [hi | lo] bf16 rows for the tensor-core tiled SSpMM
            if (Wr) { d.root_idx = ridx; d.root_k = rk; d.root = root; }
            dz_tc[r] = n > 0 && tc2_rows_supported(d);
            if (!dz_tc[r]) return;
            jobs[nj++] = Tc2PackJob{W, D, D, Kd, 0, d.N, 0, (uint8_t *)d.bimg[0]};
            if (Wr) jobs[nj++] = Tc2PackJob{Wr, D, D, Kr, Kd, d.N, 0, (uint8_t *)d.bimg[0]};
        };
        prep(DR_NEAR, nc, L->d_cell, dyc, mode_near, L->wn[DR_NEAR], L->wr[DR_NEAR], L->d_cell, hci,
             L->k_cell, root_c, g->rel[DR_NEAR].c, near_tiled);
        if (dyn)
            prep(DR_PINS, nn, L->d_cell, dyn, kMaskNone, L->wn[DR_PINS], L->wr[DR_PINS], L->d_net,
                 hni, L->k_net, root_n, g->rel[DR_PINS].c, false);
        prep(DR_PINNED, nc, L->d_net, dyc, mode_pinned, L->wn[DR_PINNED], nullptr, 0, nullptr, 0,
             nullptr, g->rel[DR_PINNED].c, false);
        launch_tc2_pack_b_multi(jobs, nj, st);
    }
    const bool seq = (flags & DR_FWD_SEQUENTIAL) != 0 || force_sequential();
    StreamCtx &C = ctx();
    cudaStream_t s0 = seq ? st : C.s[0], s1 = seq ? st : C.s[1], s2 = seq ? st : C.s[2];
    if (!seq) {
        DR_CUDA(cudaEventRecord(C.fork, st));
        for (int q = 0; q < 3; ++q) DR_CUDA(cudaStreamWaitEvent(C.s[q], C.fork, 0));
    }
    auto dw = [&](int64_t n, int K, const float *Zd, const float *hv, const uint8_t *hi, int k,
                  const float *dy, int mode, float *gw, float *gb, float *wk, cudaStream_t s) {
        DwArgs a;
        a.n = n; a.K = K; a.N = D; a.Z = Zd; a.hval = hv; a.hidx = hi; a.k = k;
        a.dy = dy; a.mask = mask; a.mask_mode = mode;
        launch_dw(a, gw, gb, wk, s);
    };
    if (dxc || dxn) {
        // dZ'_psi = c_psi (dY_psi Wn_psi^T) (row-scaled by the destination normaliser),
        // with the Sage root term (dY_psi Wr_psi^T) at the kept indices as extra columns
        // (descriptors and packed weights prepared before the fork, dz_prep)
        auto dzk = [&](int r, int64_t n, int Kd, const float *dy, int mode, const float *W,
                       const float *Wr, const uint8_t *ridx, int rk, float *root,
                       const float *c, float *out, cudaStream_t s) {
            if (dz_tc[r]) {
                launch_tc2_rows(dzd[r], s);
                return;
            }
            ProjBwdArgs a;
            a.n = n; a.N = D; a.K = Kd; a.dy = dy; a.mask = mask; a.mask_mode = mode;
            a.W = W; a.c = c; a.dz = out;
            launch_proj_bwd_dz(a, s);
            if (Wr) {
                RootArgs q;
                q.n = n; q.N = D; q.k = rk; q.dy = dy; q.mask = mask; q.mask_mode = mode;
                q.Wr = Wr; q.hidx = ridx; q.out = root;
                launch_root_dots(q, s);
            }
        };
        const bool near_split = near_tiled && dz_tc[DR_NEAR];
        {
            TagScope t("near");
            dzk(DR_NEAR, nc, L->d_cell, dyc, mode_near, L->wn[DR_NEAR], L->wr[DR_NEAR], hci,
                L->k_cell, root_c, g->rel[DR_NEAR].c, dz[DR_NEAR], s0);
        }
        if (dyn) {
            TagScope t("pins");
            dzk(DR_PINS, nn, L->d_cell, dyn, kMaskNone, L->wn[DR_PINS], L->wr[DR_PINS], hni,
                L->k_net, root_n, g->rel[DR_PINS].c, dz[DR_PINS], s1);
        }
        if (!seq) DR_CUDA(cudaEventRecord(C.ev[0], s1));                           // dZ_pins, root_n
        {
            TagScope t("pinned");
            dzk(DR_PINNED, nc, L->d_net, dyc, mode_pinned, L->wn[DR_PINNED], nullptr, nullptr, 0,
                nullptr, g->rel[DR_PINNED].c, dz[DR_PINNED], s2);
        }
        // SSpMM per source node type (Alg. 2 stage 2-3, ownership instead of atomics)
        // dY_net == 0 (dyn == NULL): no pins term (dZ'_pins = 0) and no pins root term
        const float *rootc = L->wr[DR_NEAR] ? root_c : nullptr;
        if (sh) {
            // sharded: every relation's per-source sums go straight into the source
            // owners' inbox slots (the owners add them up, dr_shard_layer_dx)
            if (dxc) {
                if (!seq) DR_CUDA(cudaStreamWaitEvent(s0, C.ev[0], 0));
                TagScope t("cell");
                const RelDev &rp = g->rel[DR_PINS];
                launch_spmm_bwd(rn.bwd, rn.n_src, BwdTerm{&rn, dz[DR_NEAR], false}, BwdTerm{}, nullptr,
                                nullptr, L->k_cell, L->d_cell, nullptr, nullptr, false, s0, NgSched{},
                                &sh->near_g);
                if (dyn)
                    launch_spmm_bwd(rp.bwd, rp.n_src, BwdTerm{&rp, dz[DR_PINS], false}, BwdTerm{},
                                    nullptr, nullptr, L->k_cell, L->d_cell, nullptr, nullptr, false, s0,
                                    NgSched{}, &sh->pins_g);
            }
            if (dxn) {
                if (!seq) DR_CUDA(cudaStreamWaitEvent(s2, C.ev[0], 0));
                TagScope t("net");
                const RelDev &rq = g->rel[DR_PINNED];
                launch_spmm_bwd(rq.bwd, rq.n_src, BwdTerm{&rq, dz[DR_PINNED], false}, BwdTerm{},
                                nullptr, nullptr, L->k_net, L->d_net, nullptr, nullptr, false, s2,
                                NgSched{}, &sh->pinned_g);
            }
        } else if (dxc) {
            if (!seq) DR_CUDA(cudaStreamWaitEvent(s0, C.ev[0], 0));
            BwdTerm t0{&g->rel[DR_NEAR], dz[DR_NEAR], false}, t1{&g->rel[DR_PINS], dz[DR_PINS], false};
            if (!dyn) t1 = BwdTerm{};
            TagScope t("cell");
            if (own) {
                // Q27: near (+ root) writes the dense dX_c row at idx_c, then the pins
                // term adds its mask gradient at pins' own kept indices idx_p
                const float *rootp = L->wr[DR_NEAR] ? root_c : nullptr;
                if (near_tiled)
                    launch_tspmm_bwd(rn, dz[DR_NEAR], near_split, false, rootp, hci, L->k_cell,
                                     L->d_cell, nullptr, dxc, s0);
                else
                    launch_spmm_bwd(rn.bwd, nc, t0, BwdTerm{}, rootp, hci, L->k_cell, L->d_cell,
                                    nullptr, dxc, false, s0);
                TagScope t2("pins");
                if (dyn)
                    launch_spmm_bwd(g->rel[DR_PINS].bwd, nc, t1, BwdTerm{}, nullptr, hpi, kp,
                                    L->d_cell, nullptr, dxc, true, s0);
            } else if (near_tiled && !dyn) {
                launch_tspmm_bwd(rn, dz[DR_NEAR], near_split, false, rootc, hci, L->k_cell,
                                 L->d_cell, nullptr, dxc, s0);
            } else if (near_tiled) {
                // tensor-core tiled near term; the low-degree pins term (+ the root
                // term) first goes to root_c in place with the SIMT kernel, and the
                // tiled kernel adds it in its epilogue as it would the root term
                {
                    TagScope t2("pins");
                    launch_spmm_bwd(g->rel[DR_PINS].bwd, nc, t1, BwdTerm{},
                                    L->wr[DR_NEAR] ? root_c : nullptr, hci, L->k_cell, L->d_cell,
                                    root_c, nullptr, false, s0);
                }
                launch_tspmm_bwd(rn, dz[DR_NEAR], near_split, false, root_c, hci, L->k_cell,
                                 L->d_cell, nullptr, dxc, s0);
            } else {
                launch_spmm_bwd(g->src_cell, nc, t0, t1, L->wr[DR_NEAR] ? root_c : nullptr, hci,
                                L->k_cell, L->d_cell, nullptr, dxc, false, s0);
            }
        }
        if (dxn && !sh) {
            if (!seq) DR_CUDA(cudaStreamWaitEvent(s2, C.ev[0], 0));
            BwdTerm t0{&g->rel[DR_PINNED], dz[DR_PINNED], false}, t1{};
            TagScope t("net");
            launch_spmm_bwd(g->src_net, nn, t0, t1, (L->wr[DR_PINS] && dyn) ? root_n : nullptr, hni,
                            L->k_net, L->d_net, nullptr, dxn, false, s2);
        }
    }
    // weight gradients: dW = Z^T dY_psi, dWr = H^T dY_psi, db = colsum(dY_psi), on the
    // tensor cores when the shapes allow (tc2 reduce GEMM), else the SIMT kernels
    auto dwt = [&](int64_t n, const float *Za, int wa, float *ga, const float *hv,
                   const uint8_t *hi, int k, int wb, float *gb, const float *dy, int mode,
                   float *db, float *wk, cudaStream_t s, bool zsplit) -> bool {
        Tc2ReduceDesc d;
        d.n = n; d.N = D; d.dy = dy; d.mask = mask; d.mask_mode = mode; d.db = db;
        Tc2RedSeg sa, sb;
        sa.Z = Za; sa.w = wa; sa.grad = ga; sa.split = zsplit;
        sb.hval = hv; sb.hidx = hi; sb.k = k; sb.w = wb; sb.grad = gb;
        d.G = 1; d.nseg[0] = 1; d.seg[0][0] = sa;
        if (gb && wa + wb <= 128) {
            d.nseg[0] = 2; d.seg[0][1] = sb;
        } else if (gb) {                           // two groups of 128 feature rows
            d.G = 2; d.nseg[1] = 1; d.seg[1][0] = sb;
        }
        if (!tc2_reduce_supported(d)) {
            DR_CHECK(!zsplit, DR_ERR_UNSUPPORTED, "dW: split Z needs the tensor-core reduce");
            return false;
        }
        launch_tc2_reduce(d, wk, s, pq);
        return true;
    };
    // near + pinned weight gradients in ONE reduce launch when the layer is a max
    // merge of the square D = 64 shapes: both read dY_cell, with complementary masks
    // (Eq. 12-13), so one pass over dY and the mask feeds both B operands (dual B)
    bool dw_dual = false;
    if (knobs().dw_dual && !sh && mode_near == kMaskM && mode_pinned == kMaskNotM && L->wr[DR_NEAR] &&
        D == 64 && L->d_cell == 64 && L->d_net == 64 && L->k_cell <= 32 && z_split_ok(L, DR_NEAR) &&
        z_split_ok(L, DR_PINNED)) {
        Tc2ReduceDesc d;
        d.n = nc; d.N = D; d.dy = dyc; d.mask = mask; d.mask_mode = mode_near; d.db = G->b[DR_NEAR];
        d.mask_mode1 = mode_pinned; d.db1 = G->b[DR_PINNED];
        d.G = 2; d.nseg[0] = 2; d.nseg[1] = 1;
        Tc2RedSeg sz, sh2, sp;
        sz.Z = z[DR_NEAR]; sz.w = L->d_cell; sz.grad = G->wn[DR_NEAR]; sz.split = true;
        sh2.hval = hcv; sh2.hidx = hci; sh2.k = L->k_cell; sh2.w = L->d_cell; sh2.grad = G->wr[DR_NEAR];
        sp.Z = z[DR_PINNED]; sp.w = L->d_net; sp.grad = G->wn[DR_PINNED]; sp.split = true;
        d.seg[0][0] = sz; d.seg[0][1] = sh2; d.seg[1][0] = sp;
        if (tc2_reduce_supported(d)) {
            TagScope t("near_pinned");
            launch_tc2_reduce(d, work[0], s0, pq);
            dw_dual = true;
        }
    }
    if (!dw_dual) {
        TagScope t("near");
        if (!dwt(nc, z[DR_NEAR], L->d_cell, G->wn[DR_NEAR], hcv, hci, L->k_cell, L->d_cell,
                 L->wr[DR_NEAR] ? G->wr[DR_NEAR] : nullptr, dyc, mode_near, G->b[DR_NEAR],
                 work[0], s0, !sh && z_split_ok(L, DR_NEAR))) {
            dw(nc, L->d_cell, z[DR_NEAR], nullptr, nullptr, 0, dyc, mode_near, G->wn[DR_NEAR],
               G->b[DR_NEAR], work[0], s0);
            TagScope t2("root");
            if (L->wr[DR_NEAR])
                dw(nc, L->d_cell, nullptr, hcv, hci, L->k_cell, dyc, mode_near, G->wr[DR_NEAR],
                   nullptr, work[0], s0);
        }
    }
    if (!dw_dual) {
        TagScope t("pinned");
        if (!dwt(nc, z[DR_PINNED], L->d_net, G->wn[DR_PINNED], nullptr, nullptr, 0, 0, nullptr,
                 dyc, mode_pinned, G->b[DR_PINNED], work[2], s2, !sh && z_split_ok(L, DR_PINNED)))
            dw(nc, L->d_net, z[DR_PINNED], nullptr, nullptr, 0, dyc, mode_pinned,
               G->wn[DR_PINNED], G->b[DR_PINNED], work[2], s2);
    }
    if (!dyn) {                  // dY_net == 0: the pins gradients are exactly zero
        DR_CUDA(cudaMemsetAsync(G->wn[DR_PINS], 0, (size_t)L->d_cell * D * 4, s1));
        if (L->wr[DR_PINS]) DR_CUDA(cudaMemsetAsync(G->wr[DR_PINS], 0, (size_t)L->d_net * D * 4, s1));
        DR_CUDA(cudaMemsetAsync(G->b[DR_PINS], 0, (size_t)D * 4, s1));
    } else {
        TagScope t("pins");
        if (!dwt(nn, z[DR_PINS], L->d_cell, G->wn[DR_PINS], hnv, hni, L->k_net, L->d_net,
                 L->wr[DR_PINS] ? G->wr[DR_PINS] : nullptr, dyn, kMaskNone, G->b[DR_PINS],
                 work[1], s1, !sh && z_split_ok(L, DR_PINS))) {
            dw(nn, L->d_cell, z[DR_PINS], nullptr, nullptr, 0, dyn, kMaskNone, G->wn[DR_PINS],
               G->b[DR_PINS], work[1], s1);
            TagScope t2("root");
            if (L->wr[DR_PINS])
                dw(nn, L->d_net, nullptr, hnv, hni, L->k_net, dyn, kMaskNone, G->wr[DR_PINS],
                   nullptr, work[1], s1);
        }
    }
    if (!seq) {
        wait_on(st, s0, C.ev[3]);
        wait_on(st, s1, C.ev[4]);
        wait_on(st, s2, C.ev[5]);
    }
    if (!defer) launch_tc2_reduce_parts(own_parts, st);   // after the join: every reduce done
}

// ------------------------------------------------------------------ NCCL (loaded at run time)
NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = dlerror();
            return;
        }
        api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
        api.commCount = (decltype(api.commCount))dlsym(h, "ncclCommCount");
        api.commUserRank = (decltype(api.commUserRank))dlsym(h, "ncclCommUserRank");
        api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
        api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
        api.reduceScatter = (decltype(api.reduceScatter))dlsym(h, "ncclReduceScatter");
        api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
        api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
        api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
        api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.commCount &&
                 api.commUserRank && api.allReduce && api.allGather && api.reduceScatter &&
                 api.groupStart && api.groupEnd && api.getErrorString && api.commGetAsyncError;
        if (!api.ok) api.err = "missing NCCL symbols";
    });
    if (!api.ok) fail(DR_ERR_NCCL, "cannot load NCCL: " + api.err);
    return api;
}

}  // namespace dr

using namespace dr;

// ------------------------------------------------------------------ trainer
struct dr_trainer {
    dr_train_cfg cfg{};
    float *params = nullptr;
    int64_t n_params = 0;
    ncclComm_t comm = nullptr;
    int world = 1;
    Alloc alloc;
    float *grad = nullptr, *m = nullptr, *v = nullptr, *scalars = nullptr;  // scalars: loss
    int64_t step = 0;
    char *ws = nullptr;
    size_t ws_cap = 0;
    std::vector<dr_layer> L;
    std::vector<dr_layer_grad> G;
    float *head_w = nullptr, *head_b = nullptr, *ghead_w = nullptr, *ghead_b = nullptr;
    int64_t *step_dev = nullptr;             // Adam step counter (device, inside scalars)
    // CUDA graphs of the whole step (§3.2 "CUDA-graph captured per batch shape"),
    // keyed by the call's graph and buffers; a key runs eagerly once, then is captured
    struct GraphEntry {
        uint64_t graph_uid = 0;
        const void *xc = nullptr, *xn = nullptr, *lab = nullptr, *loss = nullptr, *gout = nullptr;
        int runs = 0;
        int64_t kernels = 0;                 // kernel nodes (counted as launches per replay)
        uint64_t last_use = 0;
        cudaGraphExec_t exec = nullptr;
    };
    // LRU-bounded: training over many designs (one dr_graph each) or fresh input
    // buffers every step must not grow the cache (or keep execs of dead graphs)
    static constexpr size_t kMaxGraphs = 128;
    std::vector<GraphEntry> graphs;
    uint64_t use_clock = 0;
};

namespace {

int64_t layer_params(int dc, int dn, int D) {
    return (int64_t)dc * D * 3 + (int64_t)dn * D * 2 + 3 * (int64_t)D;
}

// Carve per-layer weight pointers out of a flat buffer (layout documented in dr.h).
template <typename LayerT, typename P>
void carve(const dr_train_cfg &c, P *base, std::vector<LayerT> &out, P **hw, P **hb) {
    out.clear();
    P *p = base;
    int dc = c.d_in_cell, dn = c.d_in_net;
    const int D = c.d_hidden;
    for (int l = 0; l < c.n_layers; ++l) {
        LayerT x{};
        x.wn[DR_NEAR] = p; p += (int64_t)dc * D;
        x.wr[DR_NEAR] = p; p += (int64_t)dc * D;
        x.b[DR_NEAR] = p; p += D;
        x.wn[DR_PINNED] = p; p += (int64_t)dn * D;
        x.b[DR_PINNED] = p; p += D;
        x.wn[DR_PINS] = p; p += (int64_t)dc * D;
        x.wr[DR_PINS] = p; p += (int64_t)dn * D;
        x.b[DR_PINS] = p; p += D;
        x.wr[DR_PINNED] = nullptr;
        out.push_back(x);
        dc = dn = D;
    }
    *hw = p; p += D;
    *hb = p;
}

}  // namespace

#define DR_API_BEGIN                                                                         \
    clear_error();                                                                           \
    try {
#define DR_API_END                                                                           \
    }                                                                                        \
    catch (const Error &e) {                                                                 \
        set_error(e.status, e.msg);                                                          \
        return e.status;                                                                     \
    }                                                                                        \
    catch (const std::bad_alloc &) {                                                         \
        set_error(DR_ERR_OUT_OF_MEMORY, "host allocation failed");                           \
        return DR_ERR_OUT_OF_MEMORY;                                                         \
    }                                                                                        \
    return DR_OK;

extern "C" {

const char *dr_status_str(dr_status s) {
    switch (s) {
        case DR_OK: return "DR_OK";
        case DR_ERR_INVALID_ARGUMENT: return "DR_ERR_INVALID_ARGUMENT";
        case DR_ERR_BAD_K: return "DR_ERR_BAD_K";
        case DR_ERR_SHAPE_MISMATCH: return "DR_ERR_SHAPE_MISMATCH";
        case DR_ERR_OUT_OF_RANGE: return "DR_ERR_OUT_OF_RANGE";
        case DR_ERR_DUPLICATE_EDGE: return "DR_ERR_DUPLICATE_EDGE";
        case DR_ERR_TRANSPOSE_MISMATCH: return "DR_ERR_TRANSPOSE_MISMATCH";
        case DR_ERR_NONFINITE: return "DR_ERR_NONFINITE";
        case DR_ERR_TAPE_MISMATCH: return "DR_ERR_TAPE_MISMATCH";
        case DR_ERR_OUT_OF_MEMORY: return "DR_ERR_OUT_OF_MEMORY";
        case DR_ERR_CUDA: return "DR_ERR_CUDA";
        case DR_ERR_NCCL: return "DR_ERR_NCCL";
        case DR_ERR_UNSUPPORTED: return "DR_ERR_UNSUPPORTED";
    }
    return "DR_ERR_UNKNOWN";
}

const char *dr_last_error(void) { return t_err.c_str(); }

const char *dr_version(void) { return "libdr 0.1 sm_100a (DR-CircuitGNN hot path, arXiv 2508.16769)"; }

dr_status dr_profile_begin(void) {
    DR_API_BEGIN
    for (auto &r : t_recs) {
        t_pool.push_back(r.a);
        t_pool.push_back(r.b);
    }
    t_recs.clear();
    t_prof = true;
    DR_API_END
}

dr_status dr_profile_end(dr_profile_entry *out, int32_t cap, int32_t *n_out) {
    DR_API_BEGIN
    t_prof = false;
    std::vector<dr_profile_entry> agg;
    for (auto &r : t_recs) {
        DR_CUDA(cudaEventSynchronize(r.b));
        float ms = 0.f;
        DR_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        dr_profile_entry *e = nullptr;
        for (auto &x : agg)
            if (r.name == x.name) e = &x;
        if (!e) {
            agg.emplace_back();
            e = &agg.back();
            std::memset(e, 0, sizeof(*e));
            std::strncpy(e->name, r.name.c_str(), sizeof(e->name) - 1);
        }
        e->launches += 1;
        e->total_ms += ms;
        if (ms > e->max_ms) e->max_ms = ms;
    }
    for (auto &r : t_recs) {
        t_pool.push_back(r.a);
        t_pool.push_back(r.b);
    }
    t_recs.clear();
    if (n_out) *n_out = (int32_t)agg.size();
    for (int32_t i = 0; out && i < cap && i < (int32_t)agg.size(); ++i) out[i] = agg[i];
    DR_API_END
}

int64_t dr_launch_count(void) { return t_launches; }
void dr_launch_count_reset(void) { t_launches = 0; }


dr_status dr_drelu_topk(const float *x, int64_t n, int32_t dim, int64_t ldx, dr_cbsr *out,
                        void *stream) {
    DR_API_BEGIN
    check_cbsr(out, "drelu out");
    DR_CHECK(n >= 0 && out->n == n && out->dim == dim, DR_ERR_SHAPE_MISMATCH,
             "drelu: out->n/dim must equal n/dim");
    DR_CHECK(ldx >= dim, DR_ERR_SHAPE_MISMATCH, "drelu: ldx < dim");
    DR_CHECK(n == 0 || x, DR_ERR_INVALID_ARGUMENT, "drelu: null x");
    launch_drelu(x, n, dim, ldx, out->k, out->val, (uint8_t *)out->idx, (cudaStream_t)stream);
    DR_API_END
}

dr_status dr_spmm_fwd(const dr_graph *g, dr_rel r, const dr_cbsr *h, float *z, void *stream) {
    DR_API_BEGIN
    DR_CHECK(g != nullptr, DR_ERR_INVALID_ARGUMENT, "spmm_fwd: null graph");
    DR_CHECK(r >= 0 && r < 3, DR_ERR_INVALID_ARGUMENT, "spmm_fwd: bad relation");
    check_cbsr(h, "spmm_fwd h_src");
    const RelDev &R = g->rel[r];
    DR_CHECK(h->n == R.n_src, DR_ERR_SHAPE_MISMATCH, "spmm_fwd: h_src->n != relation n_src");
    DR_CHECK(R.n_dst == 0 || z, DR_ERR_INVALID_ARGUMENT, "spmm_fwd: null z");
    launch_spmm_fwd(R, h->val, (const uint8_t *)h->idx, h->k, h->dim, z, (cudaStream_t)stream);
    DR_API_END
}

dr_status dr_spmm_bwd(const dr_graph *g, dr_rel r, const float *dz, const dr_cbsr *h,
                      float *g_kept, float *dx, int32_t accumulate, void *stream) {
    DR_API_BEGIN
    DR_CHECK(g != nullptr, DR_ERR_INVALID_ARGUMENT, "spmm_bwd: null graph");
    DR_CHECK(r >= 0 && r < 3, DR_ERR_INVALID_ARGUMENT, "spmm_bwd: bad relation");
    check_cbsr(h, "spmm_bwd h_src");
    const RelDev &R = g->rel[r];
    DR_CHECK(h->n == R.n_src, DR_ERR_SHAPE_MISMATCH, "spmm_bwd: h_src->n != relation n_src");
    DR_CHECK(g_kept || dx, DR_ERR_INVALID_ARGUMENT, "spmm_bwd: both outputs NULL");
    DR_CHECK(R.n_dst == 0 || dz, DR_ERR_INVALID_ARGUMENT, "spmm_bwd: null dz");
    BwdTerm t0{&R, dz, true}, t1{};
    launch_spmm_bwd(R.bwd, R.n_src, t0, t1, nullptr, (const uint8_t *)h->idx, h->k, h->dim,
                    g_kept, dx, accumulate != 0, (cudaStream_t)stream);
    DR_API_END
}

// ------------------------------------------------------------------ NEXT-2 (per-neighbour-group K)
dr_status dr_drelu_topk_sorted(const float *x, int64_t n, int32_t dim, int64_t ldx, dr_cbsr *out,
                               void *stream) {
    DR_API_BEGIN
    check_cbsr(out, "drelu_sorted out");
    DR_CHECK(n >= 0 && out->n == n && out->dim == dim, DR_ERR_SHAPE_MISMATCH,
             "drelu_sorted: out->n/dim must equal n/dim");
    DR_CHECK(ldx >= dim, DR_ERR_SHAPE_MISMATCH, "drelu_sorted: ldx < dim");
    DR_CHECK(n == 0 || x, DR_ERR_INVALID_ARGUMENT, "drelu_sorted: null x");
    DR_CHECK(out->k <= 32, DR_ERR_BAD_K, "drelu_sorted: k must be <= 32");
    launch_drelu(x, n, dim, ldx, out->k, out->val, (uint8_t *)out->idx, (cudaStream_t)stream, true);
    DR_API_END
}

}  // extern "C"

struct dr_ng_plan {
    const dr_graph *g = nullptr;
    int r = 0;
    NgSched ng;                          // ng.kT: device [nnz], K(deg row[e]) per CSC edge
    Alloc alloc;
    cudaStream_t stream = nullptr;
};

extern "C" {

dr_status dr_ng_plan_create(const dr_graph *g, dr_rel r, const dr_ng_sched *s, void *stream,
                            dr_ng_plan **out) {
    DR_API_BEGIN
    DR_CHECK(g != nullptr && out != nullptr, DR_ERR_INVALID_ARGUMENT, "ng_plan: null graph/out");
    DR_CHECK(r >= 0 && r < 3, DR_ERR_INVALID_ARGUMENT, "ng_plan: bad relation");
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "ng_plan: null schedule");
    DR_CHECK(s->kb[0] >= s->kb[1] && s->kb[1] >= s->kb[2] && s->kb[2] >= 1 && s->kb[0] <= 32,
             DR_ERR_BAD_K, "ng_plan: need 32 >= kb[0] >= kb[1] >= kb[2] >= 1");
    DR_CHECK(s->thr[0] <= s->thr[1], DR_ERR_INVALID_ARGUMENT, "ng_plan: need thr[0] <= thr[1]");
    *out = nullptr;
    auto *p = new dr_ng_plan;
    p->g = g;
    p->r = r;
    p->alloc = g->alloc;
    p->stream = (cudaStream_t)stream;
    p->ng.on = 1;
    p->ng.thr0 = s->thr[0];
    p->ng.thr1 = s->thr[1];
    p->ng.kb0 = s->kb[0];
    p->ng.kb1 = s->kb[1];
    p->ng.kb2 = s->kb[2];
    const RelDev &R = g->rel[r];
    if (R.nnz > 0) {
        uint8_t *kT = nullptr;
        try {
            kT = (uint8_t *)p->alloc.get((size_t)R.nnz, p->stream);
            launch_ng_edge_k(R, p->ng, kT, p->stream);
        } catch (...) {
            if (kT) p->alloc.put(kT, p->stream);
            delete p;
            throw;
        }
        p->ng.kT = kT;
    }
    *out = p;
    DR_API_END
}

dr_status dr_ng_plan_destroy(dr_ng_plan *p) {
    if (!p) return DR_OK;
    if (p->ng.kT) {
        cudaStreamSynchronize(p->stream);
        p->alloc.put((void *)p->ng.kT, p->stream);
    }
    delete p;
    return DR_OK;
}

dr_status dr_spmm_fwd_ng(const dr_ng_plan *p, const dr_cbsr *h, float *z, void *stream) {
    DR_API_BEGIN
    DR_CHECK(p != nullptr, DR_ERR_INVALID_ARGUMENT, "spmm_fwd_ng: null plan");
    check_cbsr(h, "spmm_fwd_ng h_src");
    const RelDev &R = p->g->rel[p->r];
    DR_CHECK(h->n == R.n_src, DR_ERR_SHAPE_MISMATCH, "spmm_fwd_ng: h_src->n != relation n_src");
    DR_CHECK(h->k >= p->ng.kb0, DR_ERR_BAD_K, "spmm_fwd_ng: h_src->k < kb[0]");
    DR_CHECK(R.n_dst == 0 || z, DR_ERR_INVALID_ARGUMENT, "spmm_fwd_ng: null z");
    launch_spmm_fwd(R, h->val, (const uint8_t *)h->idx, h->k, h->dim, z, (cudaStream_t)stream,
                    false, p->ng);
    DR_API_END
}

dr_status dr_spmm_bwd_ng(const dr_ng_plan *p, const float *dz, const dr_cbsr *h, float *g_kept,
                         float *dx, void *stream) {
    DR_API_BEGIN
    DR_CHECK(p != nullptr, DR_ERR_INVALID_ARGUMENT, "spmm_bwd_ng: null plan");
    check_cbsr(h, "spmm_bwd_ng h_src");
    const RelDev &R = p->g->rel[p->r];
    DR_CHECK(h->n == R.n_src, DR_ERR_SHAPE_MISMATCH, "spmm_bwd_ng: h_src->n != relation n_src");
    DR_CHECK(h->k >= p->ng.kb0, DR_ERR_BAD_K, "spmm_bwd_ng: h_src->k < kb[0]");
    DR_CHECK(g_kept || dx, DR_ERR_INVALID_ARGUMENT, "spmm_bwd_ng: both outputs NULL");
    DR_CHECK(R.n_dst == 0 || dz, DR_ERR_INVALID_ARGUMENT, "spmm_bwd_ng: null dz");
    BwdTerm t0{&R, dz, true}, t1{};
    launch_spmm_bwd(R.bwd, R.n_src, t0, t1, nullptr, (const uint8_t *)h->idx, h->k, h->dim,
                    g_kept, dx, false, (cudaStream_t)stream, p->ng);
    DR_API_END
}

dr_status dr_heteroconv_tape_bytes(const dr_graph *g, const dr_layer *L, uint32_t flags,
                                   size_t *bytes) {
    DR_API_BEGIN
    check_layer(g, L);
    DR_CHECK(bytes != nullptr, DR_ERR_INVALID_ARGUMENT, "null bytes");
    *bytes = tape_layout(g, L, flags).total;
    DR_API_END
}

dr_status dr_heteroconv_fwd(const dr_graph *g, const dr_layer *L, const float *x_cell,
                            const float *x_net, float *y_cell, float *y_net, void *tape,
                            uint32_t flags, void *stream) {
    DR_API_BEGIN
    check_layer(g, L);
    DR_CHECK(tape != nullptr, DR_ERR_TAPE_MISMATCH, "null tape");
    DR_CHECK((g->n_cell == 0 || (x_cell && y_cell)) && (g->n_net == 0 || (x_net && y_net)),
             DR_ERR_INVALID_ARGUMENT, "heteroconv_fwd: null input/output");
    DR_CHECK(!(flags & DR_FWD_INPUT_IN_TAPE), DR_ERR_INVALID_ARGUMENT,
             "heteroconv_fwd: DR_FWD_INPUT_IN_TAPE needs dr_heteroconv_fwd_chain");
    heteroconv_fwd(g, L, x_cell, x_net, y_cell, y_net, tape, flags, (cudaStream_t)stream);
    DR_API_END
}

dr_status dr_heteroconv_fwd_chain(const dr_graph *g, const dr_layer *L, const float *x_cell,
                                  const float *x_net, float *y_cell, float *y_net, void *tape,
                                  uint32_t flags, const dr_layer *next_L, void *next_tape,
                                  uint32_t next_flags, void *stream) {
    DR_API_BEGIN
    check_layer(g, L);
    DR_CHECK(tape != nullptr, DR_ERR_TAPE_MISMATCH, "null tape");
    const bool in_tape = (flags & DR_FWD_INPUT_IN_TAPE) != 0;
    DR_CHECK((g->n_cell == 0 || ((x_cell || in_tape) && y_cell)) &&
                 (g->n_net == 0 || ((x_net || in_tape) && y_net)),
             DR_ERR_INVALID_ARGUMENT, "heteroconv_fwd_chain: null input/output");
    DR_CHECK(!next_L == !next_tape, DR_ERR_INVALID_ARGUMENT,
             "heteroconv_fwd_chain: next_L and next_tape go together");
    if (next_L) {
        check_layer(g, next_L);
        DR_CHECK(next_L->d_cell == L->d_out && next_L->d_net == L->d_out, DR_ERR_SHAPE_MISMATCH,
                 "heteroconv_fwd_chain: next layer input widths != d_out");
        DR_CHECK(next_tape != tape, DR_ERR_INVALID_ARGUMENT, "heteroconv_fwd_chain: same tape");
    }
    heteroconv_fwd(g, L, x_cell, x_net, y_cell, y_net, tape, flags, (cudaStream_t)stream, next_L,
                   next_tape, next_flags);
    DR_API_END
}

dr_status dr_heteroconv_bwd(const dr_graph *g, const dr_layer *L, void *tape,
                            const float *dy_cell, const float *dy_net, float *dx_cell,
                            float *dx_net, dr_layer_grad *grads, uint32_t flags, void *stream) {
    DR_API_BEGIN
    check_layer(g, L);
    DR_CHECK(tape != nullptr, DR_ERR_TAPE_MISMATCH, "null tape");
    DR_CHECK(grads != nullptr, DR_ERR_INVALID_ARGUMENT, "null grads");
    for (int r = 0; r < 3; ++r) {
        DR_CHECK(grads->wn[r] && grads->b[r], DR_ERR_INVALID_ARGUMENT, "null grad wn/b");
        DR_CHECK(!L->wr[r] || grads->wr[r], DR_ERR_INVALID_ARGUMENT, "null grad wr");
    }
    DR_CHECK(dy_cell, DR_ERR_INVALID_ARGUMENT, "null dy_cell");
    heteroconv_bwd(g, L, tape, dy_cell, dy_net, dx_cell, dx_net, grads, flags,
                   (cudaStream_t)stream);
    DR_API_END
}

// ------------------------------------------------------------------ f4: a sharded layer
}  // extern "C"

struct dr_shard_layer {
    dr_graph g;                        // local rows; rel[r] = the shard blocks (not owned)
    int32_t world = 1, rank = 0, m_cell = 0, m_net = 0;
};

namespace {
ShardCtx shard_ctx(const dr_shard_layer *sl, const dr_layer *L, const dr_peer_cbsr *hc,
                   const dr_peer_cbsr *hn, float *const *inbox_c, float *const *inbox_n) {
    DR_CHECK(hc && hn && hc->world == sl->world && hn->world == sl->world, DR_ERR_INVALID_ARGUMENT,
             "shard_layer: peer tables missing or of another world size");
    ShardCtx c{};
    c.rank = sl->rank;
    c.cell.m = sl->m_cell;
    c.net.m = sl->m_net;
    c.cell.rank = c.net.rank = sl->rank;
    for (int q = 0; q < sl->world; ++q) {
        DR_CHECK(hc->val[q] && hc->idx[q] && hn->val[q] && hn->idx[q], DR_ERR_INVALID_ARGUMENT,
                 "shard_layer: null CBSR pointer in a peer table");
        c.cell.pv[q] = hc->val[q];
        c.cell.pi[q] = (const uint8_t *)hc->idx[q];
        c.net.pv[q] = hn->val[q];
        c.net.pi[q] = (const uint8_t *)hn->idx[q];
    }
    c.near_g = c.pins_g = c.cell;
    c.pinned_g = c.net;
    if (inbox_c && inbox_n) {
        const int64_t slot_c = (int64_t)sl->world * sl->m_cell * L->k_cell;
        for (int q = 0; q < sl->world; ++q) {
            DR_CHECK(inbox_c[q] && inbox_n[q], DR_ERR_INVALID_ARGUMENT, "shard_layer: null inbox");
            c.near_g.pg[q] = inbox_c[q];               // slots [0][rank]
            c.pins_g.pg[q] = inbox_c[q] + slot_c;      // slots [1][rank]
            c.pinned_g.pg[q] = inbox_n[q];
        }
    }
    return c;
}
void check_shard_layer(const dr_shard_layer *sl, const dr_layer *L) {
    DR_CHECK(sl != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_layer: null layer set");
    check_layer(&sl->g, L);
    DR_CHECK(!pins_own(L), DR_ERR_UNSUPPORTED, "shard_layer: k_pins is not supported");
}
}  // namespace

extern "C" {

dr_status dr_shard_layer_create(const dr_shard *near, const dr_shard *pins, const dr_shard *pinned,
                                dr_shard_layer **out) {
    DR_API_BEGIN
    DR_CHECK(near && pins && pinned && out, DR_ERR_INVALID_ARGUMENT, "shard_layer: null argument");
    *out = nullptr;
    const int W = near->world;
    DR_CHECK(pins->world == W && pinned->world == W && pins->rank == near->rank &&
                 pinned->rank == near->rank && W <= kMaxPeers,
             DR_ERR_INVALID_ARGUMENT, "shard_layer: shards of different worlds / ranks (or > 8)");
    // cells: near dst == near src == pinned dst == pins src ranges; nets: pins dst == pinned src
    DR_CHECK(near->dst_begin == near->src_begin && near->dst_end == near->src_end &&
                 pinned->dst_begin == near->dst_begin && pinned->dst_end == near->dst_end &&
                 pins->src_begin == near->src_begin && pins->src_end == near->src_end &&
                 pins->max_src == near->max_src && pinned->src_begin == pins->dst_begin &&
                 pinned->src_end == pins->dst_end,
             DR_ERR_SHAPE_MISMATCH,
             "shard_layer: the three shards must share one cell and one net partition "
             "(near: cells -> cells, pins: cells -> nets, pinned: nets -> cells)");
    std::unique_ptr<dr_shard_layer> sl(new dr_shard_layer());
    sl->world = W;
    sl->rank = near->rank;
    sl->m_cell = near->max_src;
    sl->m_net = pinned->max_src;
    sl->g.n_cell = (int32_t)(near->dst_end - near->dst_begin);
    sl->g.n_net = (int32_t)(pins->dst_end - pins->dst_begin);
    sl->g.rel[DR_NEAR] = near->rel;
    sl->g.rel[DR_PINS] = pins->rel;
    sl->g.rel[DR_PINNED] = pinned->rel;
    *out = sl.release();
    DR_API_END
}

dr_status dr_shard_layer_destroy(dr_shard_layer *sl) {
    delete sl;
    return DR_OK;
}

dr_status dr_shard_layer_tape_bytes(const dr_shard_layer *sl, const dr_layer *L, uint32_t flags,
                                    size_t *bytes) {
    DR_API_BEGIN
    check_shard_layer(sl, L);
    DR_CHECK(bytes != nullptr, DR_ERR_INVALID_ARGUMENT, "null bytes");
    *bytes = tape_layout(&sl->g, L, flags).total;
    DR_API_END
}

dr_status dr_shard_layer_fwd(const dr_shard_layer *sl, const dr_layer *L, const dr_peer_cbsr *h_cell,
                             const dr_peer_cbsr *h_net, float *y_cell, float *y_net, void *tape,
                             uint32_t flags, void *stream) {
    DR_API_BEGIN
    check_shard_layer(sl, L);
    DR_CHECK(tape && (sl->g.n_cell == 0 || y_cell) && (sl->g.n_net == 0 || y_net),
             DR_ERR_INVALID_ARGUMENT, "shard_layer_fwd: null tape / output");
    const ShardCtx c = shard_ctx(sl, L, h_cell, h_net, nullptr, nullptr);
    heteroconv_fwd(&sl->g, L, nullptr, nullptr, y_cell, y_net, tape, flags & ~DR_FWD_NO_NET_OUT,
                   (cudaStream_t)stream, nullptr, nullptr, 0, nullptr, nullptr, &c);
    DR_API_END
}

dr_status dr_shard_layer_bwd(const dr_shard_layer *sl, const dr_layer *L, void *tape,
                             const float *dy_cell, const float *dy_net, const dr_peer_cbsr *h_cell,
                             const dr_peer_cbsr *h_net, float *const *inbox_cell,
                             float *const *inbox_net, dr_layer_grad *grads, uint32_t flags,
                             void *stream) {
    DR_API_BEGIN
    check_shard_layer(sl, L);
    DR_CHECK(tape && grads && dy_cell && dy_net && inbox_cell && inbox_net, DR_ERR_INVALID_ARGUMENT,
             "shard_layer_bwd: null argument");
    for (int r = 0; r < 3; ++r) {
        DR_CHECK(grads->wn[r] && grads->b[r], DR_ERR_INVALID_ARGUMENT, "null grad wn/b");
        DR_CHECK(!L->wr[r] || grads->wr[r], DR_ERR_INVALID_ARGUMENT, "null grad wr");
    }
    const ShardCtx c = shard_ctx(sl, L, h_cell, h_net, inbox_cell, inbox_net);
    // dx pointers only switch the SSpMM on: the sharded path writes the inboxes
    float *on = reinterpret_cast<float *>(tape);
    heteroconv_bwd(&sl->g, L, tape, dy_cell, dy_net, on, on, grads, flags, (cudaStream_t)stream,
                   nullptr, &c);
    DR_API_END
}

dr_status dr_shard_layer_dx(const dr_shard_layer *sl, const dr_layer *L, void *tape,
                            const dr_peer_cbsr *h_cell, const dr_peer_cbsr *h_net,
                            const float *inbox_cell, const float *inbox_net, float *dx_cell,
                            float *dx_net, void *stream) {
    DR_API_BEGIN
    check_shard_layer(sl, L);
    DR_CHECK(tape && inbox_cell && inbox_net && dx_cell && dx_net, DR_ERR_INVALID_ARGUMENT,
             "shard_layer_dx: null argument");
    const ShardCtx c = shard_ctx(sl, L, h_cell, h_net, nullptr, nullptr);
    const TapeLayout T = tape_layout(&sl->g, L, 0);
    char *tp = (char *)tape;
    float *root_c = (float *)(tp + T.root_c), *root_n = (float *)(tp + T.root_n);
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nc = sl->g.n_cell, nn = sl->g.n_net;
    // cells: near and pins slots of every rank (+ the Sage root term), then the mask scatter
    launch_inbox_root(inbox_cell, 2 * sl->world, (int64_t)sl->m_cell * L->k_cell,
                      L->wr[DR_NEAR] ? root_c : nullptr, nc * L->k_cell, root_c, st);
    launch_cbsr_scatter(root_c, c.cell.pi[sl->rank], nc, L->k_cell, L->d_cell, dx_cell, st);
    launch_inbox_root(inbox_net, sl->world, (int64_t)sl->m_net * L->k_net,
                      L->wr[DR_PINS] ? root_n : nullptr, nn * L->k_net, root_n, st);
    launch_cbsr_scatter(root_n, c.net.pi[sl->rank], nn, L->k_net, L->d_net, dx_net, st);
    DR_API_END
}

dr_status dr_heteroconv_tape_view(const dr_graph *g, const dr_layer *L, void *tape,
                                  uint32_t flags, dr_tape_view *v) {
    DR_API_BEGIN
    check_layer(g, L);
    DR_CHECK(tape && v, DR_ERR_INVALID_ARGUMENT, "null tape/view");
    const TapeLayout T = tape_layout(g, L, flags);
    char *tp = (char *)tape;
    std::memset(v, 0, sizeof(*v));
    v->h_cell = dr_cbsr{g->n_cell, L->d_cell, L->k_cell, 1, tp + T.hc_idx, (float *)(tp + T.hc_val)};
    v->h_net = dr_cbsr{g->n_net, L->d_net, L->k_net, 1, tp + T.hn_idx, (float *)(tp + T.hn_val)};
    v->h_pins = dr_cbsr{g->n_cell, L->d_cell, k_pins_of(L), 1, tp + T.hp_idx, (float *)(tp + T.hp_val)};
    for (int r = 0; r < 3; ++r) {
        v->z[r] = (float *)(tp + T.z[r]);
        v->z_split[r] = z_split_ok(L, r) ? 1 : 0;
    }
    if (flags & DR_FWD_TAPS) {
        v->y_near = (float *)(tp + T.tap_a);
        v->y_pinned = (float *)(tp + T.tap_b);
    }
    v->mask = (uint32_t *)(tp + T.mask);
    DR_API_END
}

int64_t dr_train_param_count(const dr_train_cfg *c) {
    if (!c || c->n_layers < 1) return -1;
    int64_t n = 0;
    int dc = c->d_in_cell, dn = c->d_in_net;
    for (int l = 0; l < c->n_layers; ++l) {
        n += layer_params(dc, dn, c->d_hidden);
        dc = dn = c->d_hidden;
    }
    return n + c->d_hidden + 1;
}

dr_status dr_trainer_create(const dr_train_cfg *c, float *params, int64_t n_params,
                            void *nccl_comm, const dr_allocator *a, dr_trainer **out) {
    DR_API_BEGIN
    DR_CHECK(c && params && out, DR_ERR_INVALID_ARGUMENT, "null cfg/params/out");
    *out = nullptr;
    DR_CHECK(c->n_layers >= 1 && c->n_layers <= 8, DR_ERR_INVALID_ARGUMENT, "n_layers in [1,8]");
    DR_CHECK(dr_train_param_count(c) == n_params, DR_ERR_SHAPE_MISMATCH,
             "n_params != dr_train_param_count(cfg)");
    check_k(c->k_cell, c->d_in_cell, "cfg k_cell/d_in_cell");
    check_k(c->k_net, c->d_in_net, "cfg k_net/d_in_net");
    check_k(c->k_cell, c->d_hidden, "cfg k_cell/d_hidden");
    check_k(c->k_net, c->d_hidden, "cfg k_net/d_hidden");
    DR_CHECK(c->k_pins >= 0, DR_ERR_BAD_K, "cfg: negative k_pins");
    if (c->k_pins) {
        check_k(c->k_pins, c->d_in_cell, "cfg k_pins/d_in_cell");
        check_k(c->k_pins, c->d_hidden, "cfg k_pins/d_hidden");
    }
    check_out_width(c->d_hidden, "cfg d_hidden");
    check_out_width(c->d_in_cell, "cfg d_in_cell");
    check_out_width(c->d_in_net, "cfg d_in_net");
    // owned until every step below succeeded (a throw frees it: nothing leaks)
    std::unique_ptr<dr_trainer, dr_status (*)(dr_trainer *)> t(new dr_trainer(), dr_trainer_destroy);
    t->cfg = *c;
    t->params = params;
    t->n_params = n_params;
    if (a && a->alloc && a->free) {
        t->alloc.a = *a;
        t->alloc.custom = true;
    }
    if (nccl_comm) {
        t->comm = (ncclComm_t)nccl_comm;
        DR_NCCL(nccl().commCount(t->comm, &t->world));
    }
    const size_t pb = (size_t)n_params * 4;
    char *blk = (char *)t->alloc.get(al(pb) * 3 + 256, nullptr);
    t->grad = (float *)blk;
    t->m = (float *)(blk + al(pb));
    t->v = (float *)(blk + 2 * al(pb));
    t->scalars = (float *)(blk + 3 * al(pb));
    t->step_dev = (int64_t *)(blk + 3 * al(pb) + 64);
    DR_CUDA(cudaMemset(blk, 0, al(pb) * 3 + 256));
    DR_CUDA(cudaDeviceSynchronize());
    carve(t->cfg, (const float *)t->params, t->L, (const float **)&t->head_w, (const float **)&t->head_b);
    carve(t->cfg, t->grad, t->G, &t->ghead_w, &t->ghead_b);
    for (auto &l : t->L) {
        l.d_out = c->d_hidden;
        l.k_cell = c->k_cell;
        l.k_net = c->k_net;
        l.k_pins = c->k_pins;
        l.merge = DR_MERGE_MAX;
    }
    int dc = c->d_in_cell, dn = c->d_in_net;
    for (auto &l : t->L) {
        l.d_cell = dc;
        l.d_net = dn;
        dc = dn = c->d_hidden;
    }
    *out = t.release();
    DR_API_END
}

// One training step (forward, head/MSE, backward, allreduce, Adam), enqueued on st.
static void train_step_body(dr_trainer *t, const dr_graph *g, const float *x_cell,
                            const float *x_net, const float *labels, float *loss_host,
                            float *grad_out, char *ws, cudaStream_t st) {
    const dr_train_cfg &c = t->cfg;
    const int nl = c.n_layers, D = c.d_hidden;
    const size_t nc = (size_t)g->n_cell, nn = (size_t)g->n_net;
    std::vector<size_t> tape_off(nl);
    size_t off = 0;
    for (int l = 0; l < nl; ++l) {
        tape_off[l] = off;
        off += al(tape_layout(g, &t->L[l], 0).total);
    }
    const size_t y_off = off;
    off += nl * (al(nc * D * 4) + al(nn * D * 4));
    const size_t dy_off = off;
    off += 2 * (al(nc * D * 4) + al(nn * D * 4));
    const size_t head_off = off;
    auto yc = [&](int l) { return (float *)(ws + y_off + l * (al(nc * D * 4) + al(nn * D * 4))); };
    auto yn = [&](int l) { return (float *)(ws + y_off + l * (al(nc * D * 4) + al(nn * D * 4)) + al(nc * D * 4)); };
    auto dyc = [&](int q) { return (float *)(ws + dy_off + q * (al(nc * D * 4) + al(nn * D * 4))); };
    auto dyn = [&](int q) { return (float *)(ws + dy_off + q * (al(nc * D * 4) + al(nn * D * 4)) + al(nc * D * 4)); };
    // ---- forward
    const float *xc = x_cell, *xn = x_net;
    static const char *ltag[8] = {"L0", "L1", "L2", "L3", "L4", "L5", "L6", "L7"};
    // row a5: layer l's projection epilogues write layer l+1's input CBSR into its
    // tape (DR_FWD_INPUT_IN_TAPE there), and Y_l itself is never stored; the last
    // layer's Y_net reaches nothing (the head reads cells, Q14): not computed
    bool chain = knobs().chain != 0;
    for (int l = 0; l < nl; ++l) chain = chain && !pins_own(&t->L[l]);
    const bool no_net = knobs().skip_dead_net != 0;
    // the linear head + MSE (Q14) runs in the last cell projection's epilogue when
    // the shapes allow (its per-CTA sums finished by one small launch), else as
    // its own kernels on the stored Y_cell
    HeadArgs h;
    h.n = (int64_t)nc; h.N = D; h.y = yc(nl - 1); h.w = t->head_w; h.b = t->head_b;
    h.labels = labels; h.dy = dyc(0); h.grad_w = t->ghead_w; h.grad_b = t->ghead_b;
    h.loss = t->scalars; h.work = (float *)(ws + head_off);
    int head_parts = 0;
    for (int l = 0; l < nl; ++l) {
        TagScope tg(ltag[l]);
        const bool last = l == nl - 1;
        uint32_t fl = (chain && l > 0) ? DR_FWD_INPUT_IN_TAPE : 0u;
        if (last && no_net) fl |= DR_FWD_NO_NET_OUT;
        if (chain && !last)
            heteroconv_fwd(g, &t->L[l], xc, xn, yc(l), yn(l), ws + tape_off[l], fl | DR_FWD_Y_SCRATCH,
                           st, &t->L[l + 1], ws + tape_off[l + 1], 0);
        else
            heteroconv_fwd(g, &t->L[l], xc, xn, yc(l), yn(l), ws + tape_off[l], fl, st, nullptr,
                           nullptr, 0, (last && knobs().head_fuse) ? &h : nullptr, &head_parts);
        xc = yc(l);
        xn = yn(l);
    }
    // ---- head + MSE
    if (head_parts > 0) launch_head_reduce(h, head_parts, st);
    else launch_head_mse(h, st);
    if (!no_net)                                 // last layer's Y_net feeds nothing: dY_net = 0
        DR_CUDA(cudaMemsetAsync(dyn(0), 0, nn * D * 4, st));
    // ---- backward
    Tc2Deferred parts;
    int cur = 0;
    for (int l = nl - 1; l >= 0; --l) {
        float *dxc = l > 0 ? dyc(cur ^ 1) : nullptr;
        float *dxn = l > 0 ? dyn(cur ^ 1) : nullptr;
        TagScope tg(ltag[l]);
        const float *dyn_l = (l == nl - 1 && no_net) ? nullptr : dyn(cur);
        heteroconv_bwd(g, &t->L[l], ws + tape_off[l], dyc(cur), dyn_l, dxc, dxn, &t->G[l], 0, st,
                       &parts);
        cur ^= 1;
    }
    launch_tc2_reduce_parts(parts, st);          // every layer's weight-gradient sums, one launch
    // ---- data-parallel gradient exchange: one allreduce (sum) of the flat gradient
    // (issued whenever a communicator is given, also at world size 1)
    if (t->comm)
        DR_NCCL(nccl().allReduce(t->grad, t->grad, (size_t)t->n_params, ncclFloat32, ncclSum,
                                 t->comm, st));
    const float inv_world = 1.0f / (float)t->world;
    if (grad_out) {
        DR_CUDA(cudaMemcpyAsync(grad_out, t->grad, (size_t)t->n_params * 4,
                                cudaMemcpyDeviceToDevice, st));
        if (t->world > 1) launch_scale(grad_out, t->n_params, inv_world, st);
    }
    // ---- Adam (1/W mean folded in; step counter and bias corrections on the device)
    launch_adam(t->params, t->grad, t->m, t->v, t->n_params, c.lr, c.weight_decay, c.beta1,
                c.beta2, c.eps, t->step_dev, inv_world, st);
    if (loss_host)
        DR_CUDA(cudaMemcpyAsync(loss_host, t->scalars, 4, cudaMemcpyDeviceToHost, st));
}

dr_status dr_train_step(dr_trainer *t, const dr_graph *g, const float *x_cell, const float *x_net,
                        const float *labels, float *loss_host, float *grad_out, void *stream) {
    DR_API_BEGIN
    DR_CHECK(t && g, DR_ERR_INVALID_ARGUMENT, "null trainer/graph");
    DR_CHECK((g->n_cell == 0 || (x_cell && labels)) && (g->n_net == 0 || x_net),
             DR_ERR_INVALID_ARGUMENT, "null inputs");
    cudaStream_t st = (cudaStream_t)stream;
    if (t->comm) {       // a peer failure of an earlier step's allreduce surfaces here
        ncclResult_t ae = ncclSuccess;
        DR_NCCL(nccl().commGetAsyncError(t->comm, &ae));
        DR_CHECK(ae == ncclSuccess || ae == ncclInProgress, DR_ERR_NCCL,
                 std::string("communicator async error: ") + nccl().getErrorString(ae));
    }
    const dr_train_cfg &c = t->cfg;
    const int nl = c.n_layers, D = c.d_hidden;
    const size_t nc = (size_t)g->n_cell, nn = (size_t)g->n_net;
    // ---- workspace (grow-only): tapes, layer outputs, gradient ping-pong, head partials
    size_t off = 0;
    for (int l = 0; l < nl; ++l) off += al(tape_layout(g, &t->L[l], 0).total);
    off += nl * (al(nc * D * 4) + al(nn * D * 4));
    off += 2 * (al(nc * D * 4) + al(nn * D * 4));
    off += al(head_work_floats(D) * 4);
    if (off > t->ws_cap) {
        DR_CUDA(cudaStreamSynchronize(st));
        for (auto &e : t->graphs)
            if (e.exec) cudaGraphExecDestroy(e.exec);
        t->graphs.clear();                     // captured graphs point at the old workspace
        if (t->ws) t->alloc.put(t->ws, st);
        t->ws = (char *)t->alloc.get(off, st);
        t->ws_cap = off;
    }
    t->step += 1;
    if (t_prof || knobs().no_graph) {          // per-kernel profiling runs eagerly
        train_step_body(t, g, x_cell, x_net, labels, loss_host, grad_out, t->ws, st);
    } else {
        dr_trainer::GraphEntry *ge = nullptr;
        for (auto &e : t->graphs)
            if (e.graph_uid == g->uid && e.xc == x_cell && e.xn == x_net && e.lab == labels &&
                e.loss == loss_host && e.gout == grad_out)
                ge = &e;
        if (!ge && t->graphs.size() >= dr_trainer::kMaxGraphs) {   // evict the least recently used
            size_t lru = 0;
            for (size_t i = 1; i < t->graphs.size(); ++i)
                if (t->graphs[i].last_use < t->graphs[lru].last_use) lru = i;
            if (t->graphs[lru].exec) {
                DR_CUDA(cudaStreamSynchronize(st));          // a replay may still be in flight
                cudaGraphExecDestroy(t->graphs[lru].exec);
            }
            t->graphs.erase(t->graphs.begin() + lru);
        }
        if (!ge) {
            t->graphs.push_back({});
            ge = &t->graphs.back();
            ge->graph_uid = g->uid; ge->xc = x_cell; ge->xn = x_net; ge->lab = labels;
            ge->loss = loss_host; ge->gout = grad_out;
        }
        ge->last_use = ++t->use_clock;
        if (ge->exec) {
            DR_CUDA(cudaGraphLaunch(ge->exec, st));
            t_launches += ge->kernels;
        } else if (ge->runs++ == 0) {          // first use: eager (attributes, caches)
            train_step_body(t, g, x_cell, x_net, labels, loss_host, grad_out, t->ws, st);
        } else {                               // capture on a private stream, replay on st
            StreamCtx &C = ctx();
            cudaGraph_t graph = nullptr;
            DR_CUDA(cudaStreamBeginCapture(C.cap, cudaStreamCaptureModeThreadLocal));
            try {
                train_step_body(t, g, x_cell, x_net, labels, loss_host, grad_out, t->ws, C.cap);
            } catch (...) {
                cudaStreamEndCapture(C.cap, &graph);
                if (graph) cudaGraphDestroy(graph);
                cudaGetLastError();
                throw;
            }
            DR_CUDA(cudaStreamEndCapture(C.cap, &graph));
            size_t nn_nodes = 0;
            cudaGraphGetNodes(graph, nullptr, &nn_nodes);
            std::vector<cudaGraphNode_t> nodes(nn_nodes);
            cudaGraphGetNodes(graph, nodes.data(), &nn_nodes);
            ge->kernels = 0;
            for (auto nd : nodes) {
                cudaGraphNodeType ty;
                if (cudaGraphNodeGetType(nd, &ty) == cudaSuccess && ty == cudaGraphNodeTypeKernel)
                    ++ge->kernels;
            }
            t_launches -= ge->kernels;         // the capture counted them; the replay below counts
            const cudaError_t ie = cudaGraphInstantiate(&ge->exec, graph, 0);
            cudaGraphDestroy(graph);
            DR_CUDA(ie);
            DR_CUDA(cudaGraphLaunch(ge->exec, st));
            t_launches += ge->kernels;
        }
    }
    DR_API_END
}

dr_status dr_trainer_destroy(dr_trainer *t) {
    if (!t) return DR_OK;
    cudaDeviceSynchronize();
    for (auto &e : t->graphs)
        if (e.exec) cudaGraphExecDestroy(e.exec);
    if (t->ws) t->alloc.put(t->ws, nullptr);
    if (t->grad) t->alloc.put(t->grad, nullptr);
    delete t;
    return DR_OK;
}

dr_status dr_nccl_unique_id(void *id128) {
    DR_API_BEGIN
    DR_CHECK(id128 != nullptr, DR_ERR_INVALID_ARGUMENT, "null id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    DR_NCCL(nccl().getUniqueId(&id));
    std::memcpy(id128, &id, sizeof(id));
    DR_API_END
}

dr_status dr_nccl_comm_init(const void *id128, int32_t nranks, int32_t rank, void **comm) {
    DR_API_BEGIN
    DR_CHECK(id128 && comm && nranks >= 1 && rank >= 0 && rank < nranks,
             DR_ERR_INVALID_ARGUMENT, "bad nccl init args");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t c = nullptr;
    DR_NCCL(nccl().commInitRank(&c, nranks, id, rank));
    *comm = (void *)c;
    DR_API_END
}

dr_status dr_nccl_comm_destroy(void *comm) {
    DR_API_BEGIN
    if (comm) DR_NCCL(nccl().commDestroy((ncclComm_t)comm));
    DR_API_END
}

}  // extern "C"

// Single-graph multi-GPU DR-SpMM (beyond the paper; include/dr.h
// "single-graph multi-GPU"). A relation is split by contiguous destination-row
// ranges; each rank keeps its row block of the CSR with columns renumbered into
// the padded global source space (rank block q = rows [q*max_src, (q+1)*max_src)),
// so the allgathered CBSR is addressed directly and the SpMM / SSpMM are the
// ordinary SIMT kernels of spmm.cu on a rectangular block. The exchanges are
// NCCL collectives on the caller's communicator: allgather of the compact CBSR
// (k*5 B per source row) and reduce-scatter of the partial g (k*4 B per row).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "dr_internal.h"
#include "nccl_api.h"


using namespace dr;

namespace {

#define SH_BEGIN  \
    clear_error(); \
    try {
#define SH_END                                                         \
    }                                                                  \
    catch (const Error &e) {                                           \
        set_error(e.status, e.msg);                                    \
        return e.status;                                               \
    }                                                                  \
    catch (const std::bad_alloc &) {                                   \
        set_error(DR_ERR_OUT_OF_MEMORY, "host allocation failed");     \
        return DR_ERR_OUT_OF_MEMORY;                                   \
    }                                                                  \
    return DR_OK;

void check_rel(const dr_rel_desc *r) {
    DR_CHECK(r != nullptr, DR_ERR_INVALID_ARGUMENT, "shard: null relation");
    DR_CHECK(r->n_dst >= 0 && r->n_src >= 0 && r->nnz >= 0, DR_ERR_INVALID_ARGUMENT,
             "shard: negative size");
    DR_CHECK(r->nnz < (int64_t)INT32_MAX, DR_ERR_UNSUPPORTED, "shard: nnz must be < 2^31");
    DR_CHECK(r->row_ptr && (r->nnz == 0 || r->col_idx), DR_ERR_INVALID_ARGUMENT,
             "shard: null CSR pointer");
    DR_CHECK(r->module == DR_SAGE_MEAN || r->module == DR_GRAPHCONV_SYM, DR_ERR_INVALID_ARGUMENT,
             "shard: bad module");
    DR_CHECK(!r->col_ptr && !r->row_idx && !r->tval && !r->deg_dst && !r->deg_src &&
                 !r->norm_dst && !r->norm_src,
             DR_ERR_UNSUPPORTED, "shard: the optional CSC / degree / normaliser inputs are not "
                                 "supported (the shard computes the global ones)");
}

void default_plan(const dr_rel_desc &r, int world, int64_t *dp, int64_t *sp) {
    dp[0] = 0;
    for (int q = 1; q < world; ++q) {
        const int64_t target = r.nnz * q / world;
        const int64_t *it = std::lower_bound(r.row_ptr, r.row_ptr + r.n_dst + 1, target);
        dp[q] = std::max<int64_t>(dp[q - 1], (int64_t)(it - r.row_ptr));
    }
    dp[world] = r.n_dst;
    for (int q = 1; q < world; ++q) dp[q] = std::min<int64_t>(dp[q], r.n_dst);
    if (r.n_dst == r.n_src) {
        for (int q = 0; q <= world; ++q) sp[q] = dp[q];
    } else {
        for (int q = 0; q <= world; ++q) sp[q] = (int64_t)r.n_src * q / world;
    }
}

void check_part(const int64_t *p, int world, int64_t n, const char *what) {
    DR_CHECK(p[0] == 0 && p[world] == n, DR_ERR_INVALID_ARGUMENT,
             std::string("shard: ") + what + " must run from 0 to n");
    for (int q = 0; q < world; ++q)
        DR_CHECK(p[q] <= p[q + 1], DR_ERR_INVALID_ARGUMENT,
                 std::string("shard: ") + what + " not non-decreasing");
}

void check_cbsr_rows(const dr_cbsr *h, int64_t n, const char *what) {
    DR_CHECK(h != nullptr, DR_ERR_INVALID_ARGUMENT, std::string(what) + ": null cbsr");
    DR_CHECK(h->idx_bytes == 1, DR_ERR_UNSUPPORTED, std::string(what) + ": idx_bytes must be 1");
    DR_CHECK(h->n == n, DR_ERR_SHAPE_MISMATCH, std::string(what) + ": wrong row count");
    DR_CHECK(h->dim >= 4 && h->dim <= 256 && h->dim % 4 == 0, DR_ERR_SHAPE_MISMATCH,
             std::string(what) + ": dim must be a multiple of 4 in [4, 256]");
    DR_CHECK(h->k >= 1 && h->k <= h->dim && h->k <= 128 && (h->k & (h->k - 1)) == 0,
             DR_ERR_BAD_K, std::string(what) + ": k must be a power of two <= min(dim, 128)");
    DR_CHECK(n == 0 || (h->idx && h->val), DR_ERR_INVALID_ARGUMENT,
             std::string(what) + ": null buffers");
}

ncclComm_t comm_for(const dr_shard *s, void *c) {
    if (!c) {
        DR_CHECK(s->world == 1, DR_ERR_INVALID_ARGUMENT, "shard: world > 1 needs a communicator");
        return nullptr;
    }
    int n = 0, r = -1;
    DR_NCCL(nccl().commCount((ncclComm_t)c, &n));
    DR_NCCL(nccl().commUserRank((ncclComm_t)c, &r));
    DR_CHECK(n == s->world && r == s->rank, DR_ERR_INVALID_ARGUMENT,
             "shard: communicator size/rank differ from the shard's world/rank");
    return (ncclComm_t)c;
}

}  // namespace

extern "C" {

dr_status dr_shard_plan(const dr_rel_desc *rel, int32_t world, int64_t *dst_part,
                        int64_t *src_part) {
    SH_BEGIN
    check_rel(rel);
    DR_CHECK(world >= 1 && dst_part && src_part, DR_ERR_INVALID_ARGUMENT,
             "shard_plan: world >= 1 and outputs required");
    default_plan(*rel, world, dst_part, src_part);
    SH_END
}

dr_status dr_shard_create(const dr_rel_desc *rel, int32_t world, int32_t rank,
                          const int64_t *dst_part, const int64_t *src_part, const dr_allocator *a,
                          void *stream, dr_shard **out) {
    SH_BEGIN
    check_rel(rel);
    DR_CHECK(out != nullptr, DR_ERR_INVALID_ARGUMENT, "shard: null out");
    *out = nullptr;
    DR_CHECK(world >= 1 && rank >= 0 && rank < world, DR_ERR_INVALID_ARGUMENT,
             "shard: need 0 <= rank < world");
    std::vector<int64_t> dp(world + 1), sp(world + 1);
    default_plan(*rel, world, dp.data(), sp.data());
    if (dst_part) std::copy(dst_part, dst_part + world + 1, dp.begin());
    if (src_part) std::copy(src_part, src_part + world + 1, sp.begin());
    check_part(dp.data(), world, rel->n_dst, "dst_part");
    check_part(sp.data(), world, rel->n_src, "src_part");
    int64_t max_src = 0;
    for (int q = 0; q < world; ++q) max_src = std::max(max_src, sp[q + 1] - sp[q]);
    DR_CHECK(max_src * world < (int64_t)INT32_MAX, DR_ERR_UNSUPPORTED, "shard: too many sources");
    const int64_t *rp = rel->row_ptr;
    const int32_t *ci = rel->col_idx;
    DR_CHECK(rp[0] == 0 && rp[rel->n_dst] == rel->nnz, DR_ERR_OUT_OF_RANGE,
             "shard: row_ptr[0] != 0 or row_ptr[n_dst] != nnz");
    // global source out-degree -> global s (reading Q12); owner map
    std::vector<int32_t> deg_out((size_t)rel->n_src, 0);
    for (int64_t e = 0; e < rel->nnz; ++e) {
        DR_CHECK(ci[e] >= 0 && ci[e] < rel->n_src, DR_ERR_OUT_OF_RANGE, "shard: col out of range");
        deg_out[ci[e]]++;
    }
    std::vector<int32_t> owner((size_t)rel->n_src);
    for (int q = 0; q < world; ++q)
        for (int64_t j = sp[q]; j < sp[q + 1]; ++j) owner[j] = q;
    auto pad = [&](int32_t j) -> int32_t {
        const int q = owner[j];
        return (int32_t)(q * max_src + (j - sp[q]));
    };
    const int64_t n_pad = max_src * world;
    std::vector<float> s_pad((size_t)n_pad, 1.0f);
    for (int32_t j = 0; j < rel->n_src; ++j) {
        const double dg = std::max(deg_out[j], 1);
        s_pad[pad(j)] = (float)(rel->module == DR_SAGE_MEAN ? 1.0 : 1.0 / std::sqrt(dg));
    }
    // this rank's row block, columns in the padded space (a monotone renumbering,
    // so rows stay strictly increasing)
    const int64_t r0 = dp[rank], r1 = dp[rank + 1];
    const int64_t e0 = rp[r0], e1 = rp[r1];
    std::vector<int64_t> lrp((size_t)(r1 - r0) + 1);
    for (int64_t i = r0; i <= r1; ++i) lrp[i - r0] = rp[i] - e0;
    std::vector<int32_t> lci((size_t)(e1 - e0));
    for (int64_t e = e0; e < e1; ++e) lci[e - e0] = pad(ci[e]);
    dr_rel_desc ld{};
    ld.n_dst = (int32_t)(r1 - r0);
    ld.n_src = (int32_t)n_pad;
    ld.nnz = e1 - e0;
    ld.row_ptr = lrp.data();
    ld.col_idx = lci.empty() ? nullptr : lci.data();
    ld.val = rel->val ? rel->val + e0 : nullptr;
    ld.module = rel->module;
    struct Del {
        void operator()(dr_shard *p) const { dr_shard_destroy(p); }
    };
    std::unique_ptr<dr_shard, Del> s(new dr_shard());
    s->world = world;
    s->rank = rank;
    s->max_src = (int32_t)max_src;
    s->dst_begin = r0;
    s->dst_end = r1;
    s->src_begin = sp[rank];
    s->src_end = sp[rank + 1];
    s->n_src_glob = rel->n_src;
    s->stream = (cudaStream_t)stream;
    if (a && a->alloc && a->free) {
        s->alloc.a = *a;
        s->alloc.custom = true;
    }
    // square relation with the same source and destination ranges: the local
    // rows are the padded columns [rank * max_src, rank * max_src + rows)
    const bool own = rel->n_dst == rel->n_src && dp == sp;
    build_rel_block(ld, s_pad, own ? (int64_t)rank * max_src : -1, s->alloc, s->stream, s->rel,
                    s->blocks, s->bytes);
    *out = s.release();
    SH_END
}

dr_status dr_shard_destroy(dr_shard *s) {
    if (!s) return DR_OK;
    cudaStreamSynchronize(s->stream);
    for (void *p : s->blocks) s->alloc.put(p, s->stream);
    delete s;
    return DR_OK;
}

dr_status dr_shard_info(const dr_shard *s, dr_shard_info_t *info) {
    SH_BEGIN
    DR_CHECK(s && info, DR_ERR_INVALID_ARGUMENT, "shard_info: null argument");
    std::memset(info, 0, sizeof(*info));
    info->world = s->world;
    info->rank = s->rank;
    info->max_src = s->max_src;
    info->dst_begin = s->dst_begin;
    info->dst_end = s->dst_end;
    info->src_begin = s->src_begin;
    info->src_end = s->src_end;
    info->nnz_local = s->rel.nnz;
    info->device_bytes = s->bytes;
    info->tiles = s->rel.tiles.n_tiles;
    info->tiles_T = s->rel.tilesT.n_tiles;
    SH_END
}

dr_status dr_shard_allgather_cbsr(const dr_shard *s, const dr_cbsr *hl, dr_cbsr *ha,
                                  void *nccl_comm, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_allgather: null shard");
    check_cbsr_rows(hl, s->max_src, "shard_allgather h_local");
    check_cbsr_rows(ha, (int64_t)s->max_src * s->world, "shard_allgather h_all");
    DR_CHECK(hl->k == ha->k && hl->dim == ha->dim, DR_ERR_SHAPE_MISMATCH,
             "shard_allgather: k/dim differ");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cnt = (size_t)s->max_src * hl->k;
    ncclComm_t c = comm_for(s, nccl_comm);
    if (!c) {                              // world == 1: the gather is a copy
        if (cnt == 0) return DR_OK;
        DR_CUDA(cudaMemcpyAsync(ha->val, hl->val, cnt * 4, cudaMemcpyDeviceToDevice, st));
        DR_CUDA(cudaMemcpyAsync(ha->idx, hl->idx, cnt, cudaMemcpyDeviceToDevice, st));
        return DR_OK;
    }
    DR_NCCL(nccl().groupStart());
    DR_NCCL(nccl().allGather(hl->val, ha->val, cnt, ncclFloat32, c, st));
    DR_NCCL(nccl().allGather(hl->idx, ha->idx, cnt, ncclUint8, c, st));
    DR_NCCL(nccl().groupEnd());
    SH_END
}

dr_status dr_shard_spmm_fwd(const dr_shard *s, const dr_cbsr *ha, float *z, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_spmm_fwd: null shard");
    check_cbsr_rows(ha, (int64_t)s->max_src * s->world, "shard_spmm_fwd h_all");
    DR_CHECK(s->rel.n_dst == 0 || z, DR_ERR_INVALID_ARGUMENT, "shard_spmm_fwd: null z");
    launch_spmm_fwd(s->rel, ha->val, (const uint8_t *)ha->idx, ha->k, ha->dim, z,
                    (cudaStream_t)stream);
    SH_END
}

dr_status dr_shard_spmm_bwd(const dr_shard *s, const float *dz, const dr_cbsr *ha, float *g_part,
                            void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_spmm_bwd: null shard");
    check_cbsr_rows(ha, (int64_t)s->max_src * s->world, "shard_spmm_bwd h_all");
    DR_CHECK(g_part != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_spmm_bwd: null g_part");
    DR_CHECK(s->rel.n_dst == 0 || dz, DR_ERR_INVALID_ARGUMENT, "shard_spmm_bwd: null dz");
    BwdTerm t0{&s->rel, dz, true}, t1{};
    launch_spmm_bwd(s->rel.bwd, s->rel.n_src, t0, t1, nullptr, (const uint8_t *)ha->idx, ha->k,
                    ha->dim, g_part, nullptr, false, (cudaStream_t)stream);
    SH_END
}

dr_status dr_shard_reduce_scatter_g(const dr_shard *s, const float *g_part, const dr_cbsr *hl,
                                    float *g_local, float *dx, void *nccl_comm, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_reduce_scatter: null shard");
    check_cbsr_rows(hl, s->max_src, "shard_reduce_scatter h_local");
    DR_CHECK(g_part && g_local, DR_ERR_INVALID_ARGUMENT, "shard_reduce_scatter: null g");
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cnt = (size_t)s->max_src * hl->k;
    ncclComm_t c = comm_for(s, nccl_comm);
    if (!c) {
        if (cnt) DR_CUDA(cudaMemcpyAsync(g_local, g_part, cnt * 4, cudaMemcpyDeviceToDevice, st));
    } else {
        DR_NCCL(nccl().reduceScatter(g_part, g_local, cnt, ncclFloat32, ncclSum, c, st));
    }
    if (dx) launch_cbsr_scatter(g_local, (const uint8_t *)hl->idx, s->max_src, hl->k, hl->dim, dx, st);
    SH_END
}

// ---- f4, the exchange fused into the SpMM kernels over peer memory (NVLink P2P)
static PeerSrc peer_src(const dr_shard *s, const dr_peer_cbsr *h, int dim, int k, float *const *inbox) {
    DR_CHECK(h != nullptr, DR_ERR_INVALID_ARGUMENT, "shard peer: null dr_peer_cbsr");
    DR_CHECK(h->world == s->world && s->world <= kMaxPeers, DR_ERR_INVALID_ARGUMENT,
             "shard peer: world differs from the shard's (or > 8)");
    DR_CHECK(dim >= 4 && dim <= 256 && dim % 4 == 0, DR_ERR_SHAPE_MISMATCH,
             "shard peer: dim must be a multiple of 4 in [4, 256]");
    DR_CHECK(k >= 1 && k <= dim && k <= 128 && (k & (k - 1)) == 0, DR_ERR_BAD_K,
             "shard peer: k must be a power of two <= min(dim, 128)");
    PeerSrc p{};
    p.m = s->max_src;
    p.rank = s->rank;
    for (int q = 0; q < s->world; ++q) {
        DR_CHECK(s->max_src == 0 || (h->val[q] && h->idx[q]), DR_ERR_INVALID_ARGUMENT,
                 "shard peer: null CBSR pointer");
        p.pv[q] = h->val[q];
        p.pi[q] = (const uint8_t *)h->idx[q];
        if (inbox) {
            DR_CHECK(s->max_src == 0 || inbox[q], DR_ERR_INVALID_ARGUMENT, "shard peer: null inbox");
            p.pg[q] = inbox[q];
        }
    }
    return p;
}

dr_status dr_shard_spmm_fwd_peer(const dr_shard *s, const dr_peer_cbsr *h, int32_t dim, int32_t k,
                                 float *z, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_spmm_fwd_peer: null shard");
    const PeerSrc p = peer_src(s, h, dim, k, nullptr);
    DR_CHECK(s->rel.n_dst == 0 || z, DR_ERR_INVALID_ARGUMENT, "shard_spmm_fwd_peer: null z");
    launch_spmm_fwd(s->rel, nullptr, nullptr, k, dim, z, (cudaStream_t)stream, false, NgSched{}, &p);
    SH_END
}

dr_status dr_shard_spmm_bwd_peer(const dr_shard *s, const float *dz, const dr_peer_cbsr *h,
                                 int32_t dim, int32_t k, float *const *inbox, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr && inbox != nullptr, DR_ERR_INVALID_ARGUMENT,
             "shard_spmm_bwd_peer: null shard/inbox");
    const PeerSrc p = peer_src(s, h, dim, k, inbox);
    DR_CHECK(s->rel.n_dst == 0 || dz, DR_ERR_INVALID_ARGUMENT, "shard_spmm_bwd_peer: null dz");
    BwdTerm t0{&s->rel, dz, true}, t1{};
    launch_spmm_bwd(s->rel.bwd, s->rel.n_src, t0, t1, nullptr, nullptr, k, dim, nullptr, nullptr,
                    false, (cudaStream_t)stream, NgSched{}, &p);
    SH_END
}

dr_status dr_shard_inbox_reduce(const dr_shard *s, const float *inbox, const dr_cbsr *hl,
                                float *g_local, float *dx, void *stream) {
    SH_BEGIN
    DR_CHECK(s != nullptr, DR_ERR_INVALID_ARGUMENT, "shard_inbox_reduce: null shard");
    check_cbsr_rows(hl, s->max_src, "shard_inbox_reduce h_local");
    DR_CHECK((s->max_src == 0 || (inbox && g_local)), DR_ERR_INVALID_ARGUMENT,
             "shard_inbox_reduce: null inbox/g");
    cudaStream_t st = (cudaStream_t)stream;
    launch_inbox_sum(inbox, s->world, (int64_t)s->max_src * hl->k, g_local, st);
    if (dx) launch_cbsr_scatter(g_local, (const uint8_t *)hl->idx, s->max_src, hl->k, hl->dim, dx, st);
    SH_END
}

}  // extern "C"

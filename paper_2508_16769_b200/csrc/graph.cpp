// graph.cpp — dr_graph_create / destroy: host preprocessing of the three
// relation subgraphs and their device upload.
//
// Alg. 1 stage 1: encode each adjacency as CSR (rows =
// destinations, Eq. 4); Alg. 2 stage 1: transpose to CSC for the
// backward; Alg. 1 stage 2: classify rows by degree (hub rows ->
// CTA-per-row kernel, others packed by descending degree). §3.4:
// the three subgraphs are initialised concurrently on worker threads, each
// uploading on its own CUDA stream.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <thread>

#include "dr_internal.h"

namespace dr {
namespace {

struct HostRel {
    int32_t n_dst = 0, n_src = 0;
    int64_t nnz = 0;
    dr_module module = DR_SAGE_MEAN;
    std::vector<int32_t> rowptr, col, order, colptr, row, orderT;
    std::vector<float> ew, c, s, ewT;
    std::vector<int32_t> deg_in, deg_out;
    int32_t n_hub = 0, n_hubT = 0, n_warp = 0, n_warpT = 0, max_in = 0, max_out = 0;
    bool weighted = false;
    dr_status st = DR_OK;
    std::string err;
};

// Processing order (see Sched in dr_internal.h): hubs by descending degree,
// then the warp and sub-warp classes, each grouped by power-of-two degree bucket
// (descending) and ordered by `loc` inside a bucket (by id when `loc` is empty).
// `identity` keeps plain id order with no classes (pure-DRAM measurement flag).
void make_order(const std::vector<int32_t> &deg, bool identity, const std::vector<int64_t> &loc,
                int warp_deg, std::vector<int32_t> &order, int32_t &n_hub, int32_t &n_warp) {
    const int32_t n = (int32_t)deg.size();
    order.resize(n);
    std::iota(order.begin(), order.end(), 0);
    n_hub = n_warp = 0;
    if (identity) return;
    auto bucket = [&](int32_t i) -> int {          // 0 = hub; smaller = heavier
        const int32_t d = deg[i];
        if (d > kHubDeg) return 0;
        int lg = 0;
        while ((1 << lg) < d) ++lg;                 // ceil(log2(d)), 0 for d <= 1
        return 1 + (9 - lg);
    };
    // Locality blocks (DR_ORDER_BLOCK = log2 rows per block, default 12): inside a
    // class (hub / warp / sub-warp rows, contiguous as the kernels require) rows
    // are grouped into blocks of 2^lb consecutive locality ranks and degree-bucketed
    // inside a block, so the rows in flight at once stay spatially close (their
    // shared neighbours hit L2) while each warp still sees similar degrees. lb < 0:
    // one block (degree buckets major, the round-1 order). Default (-2): blocks of
    // 4096 from 256k rows on (C4: SIMT SpMM + SSpMM -3 %), degree-major below (the
    // working set of a C2 / C5 graph is L2-resident anyway and mixed degrees cost
    // balance: +3-6 %; profiles/r02/ab_order.txt).
    int lb = (int)knobs().order_block;
    if (lb == -2) lb = n >= (1 << 18) ? 12 : -1;
    std::vector<int64_t> key((size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        const int b = bucket(i);
        const int cls = b == 0 ? 0 : (deg[i] > warp_deg ? 1 : 2);
        const int64_t l = loc.empty() ? (int64_t)i : loc[i];
        int64_t inner;
        if (b == 0) inner = (int64_t)(INT32_MAX - deg[i]);
        else if (lb < 0) inner = ((int64_t)b << 32) | (l & 0xffffffffLL);
        else inner = ((l >> lb) << 36) | ((int64_t)b << 32) | (l & 0xffffffffLL);
        key[i] = ((int64_t)cls << 60) | inner;
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t x, int32_t y) { return key[x] < key[y]; });
    for (int32_t i = 0; i < n; ++i) {
        if (deg[i] > kHubDeg) ++n_hub;
        else if (deg[i] > warp_deg) ++n_warp;
    }
}

// Locality rank of the cells: breadth-first order over the near graph (each
// component from a pseudo-peripheral start found by a first BFS). On a
// geometric graph consecutive ranks are spatial neighbours, so rows processed
// together touch overlapping neighbour sets (L2 reuse of gathered rows).
std::vector<int64_t> bfs_rank(int32_t n, const std::vector<int32_t> &rp,
                              const std::vector<int32_t> &col) {
    std::vector<int64_t> rank((size_t)n, -1);
    std::vector<int32_t> queue((size_t)n), mark((size_t)n, -1);
    int64_t next = 0;
    for (int32_t s = 0; s < n; ++s) {
        if (rank[s] >= 0) continue;
        // first sweep: farthest node from s within its component
        size_t qh = 0, qt = 0;
        queue[qt++] = s;
        mark[s] = s;
        int32_t last = s;
        while (qh < qt) {
            const int32_t u = queue[qh++];
            last = u;
            for (int32_t e = rp[u]; e < rp[u + 1]; ++e) {
                const int32_t v = col[e];
                if (mark[v] != s && rank[v] < 0) {
                    mark[v] = s;
                    queue[qt++] = v;
                }
            }
        }
        // second sweep from the pseudo-peripheral node assigns the ranks
        qh = qt = 0;
        queue[qt++] = last;
        rank[last] = next++;
        while (qh < qt) {
            const int32_t u = queue[qh++];
            for (int32_t e = rp[u]; e < rp[u + 1]; ++e) {
                const int32_t v = col[e];
                if (rank[v] < 0) {
                    rank[v] = next++;
                    queue[qt++] = v;
                }
            }
        }
    }
    return rank;
}

// Host form of a TileSet (see dr_internal.h).
struct HostTiles {
    std::vector<int32_t> rows, chunk_beg, halo;
    std::vector<uint64_t> abits;
    std::vector<int32_t> cta_beg, cta_chunks, cta_tiles;
    int32_t tile_stride = 1;
    int32_t n_tiles = 0, grid = 0;
    int64_t n_chunks = 0;
};

struct HostTiles;
void split_ctas(HostTiles &T, int64_t tile_w);

// Tiles of <= 128 rows of a relation (rp, col over n rows), grown as BFS balls
// over the relation from the lowest-ranked unassigned row (rank = the locality
// order), so a tile is a compact neighbourhood and its halo small; then per
// tile the sorted distinct column ids (the halo, padded to 64-id chunks with
// -1) and, per chunk, its edges as (m << 6 | u). Column c is row c + row_off
// for the BFS when that is in [0, n) (square relation: row_off = 0; a
// dr_shard block: its own rank's columns), else a leaf. pack: a ball that
// stops growing is topped up with the next unassigned rows in rank order (a
// shard block's many edge-free padded rows then share tiles).
void build_tiles(int32_t n, const std::vector<int32_t> &rp, const std::vector<int32_t> &col,
                 const std::vector<int64_t> &rank, HostTiles &T, int64_t n_cols = -1,
                 int64_t row_off = 0, bool pack = false) {
    if (n_cols < 0) n_cols = n;
    auto row_of = [&](int32_t c) -> int32_t {
        const int64_t v = (int64_t)c + row_off;
        return (v >= 0 && v < n) ? (int32_t)v : -1;
    };
    std::vector<int32_t> seq((size_t)n);
    if (rank.empty()) std::iota(seq.begin(), seq.end(), 0);
    else
        for (int32_t i = 0; i < n; ++i) seq[(size_t)rank[i]] = i;
    std::vector<char> assigned((size_t)n, 0);
    std::vector<int32_t> queue;
    queue.reserve(kTsRows * 8);
    std::vector<int32_t> local((size_t)n_cols, -1);
    std::vector<int32_t> tile, hl;
    T.chunk_beg.push_back(0);
    size_t pos = 0;
    int32_t next_seed = -1;
    while (true) {
        if (next_seed < 0) {
            while (pos < (size_t)n && assigned[seq[pos]]) ++pos;
            if (pos >= (size_t)n) break;
            next_seed = seq[pos];
        }
        tile.clear();
        queue.clear();
        const int32_t s0 = next_seed;
        assigned[s0] = 1;
        tile.push_back(s0);
        queue.push_back(s0);
        for (size_t qh = 0; qh < queue.size() && (int)tile.size() < kTsRows; ++qh) {
            const int32_t u = queue[qh];
            for (int32_t e = rp[u]; e < rp[u + 1] && (int)tile.size() < kTsRows; ++e) {
                const int32_t v = row_of(col[e]);
                if (v >= 0 && !assigned[v]) {
                    assigned[v] = 1;
                    tile.push_back(v);
                    queue.push_back(v);
                }
            }
        }
        if (pack)
            while ((int)tile.size() < kTsRows) {
                while (pos < (size_t)n && assigned[seq[pos]]) ++pos;
                if (pos >= (size_t)n) break;
                assigned[seq[pos]] = 1;
                tile.push_back(seq[pos]);
            }
        // next tile grows from the lowest-ranked unassigned neighbour of this one, so
        // consecutive tiles (one CTA's run) are adjacent and share halo rows in L2
        next_seed = -1;
        int64_t best = INT64_MAX;
        for (int32_t i : tile)
            for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
                const int32_t v = row_of(col[e]);
                if (v < 0) continue;
                const int64_t r = rank.empty() ? (int64_t)v : rank[v];
                if (!assigned[v] && r < best) {
                    best = r;
                    next_seed = v;
                }
            }
        // halo: sorted distinct columns of the tile's rows
        hl.clear();
        for (int32_t i : tile)
            for (int32_t e = rp[i]; e < rp[i + 1]; ++e)
                if (local[col[e]] < 0) {
                    local[col[e]] = 0;
                    hl.push_back(col[e]);
                }
        std::sort(hl.begin(), hl.end());
        for (size_t u = 0; u < hl.size(); ++u) local[hl[u]] = (int32_t)u;
        const int64_t nch = std::max<int64_t>(1, ((int64_t)hl.size() + kTsChunk - 1) / kTsChunk);
        for (int m = 0; m < kTsRows; ++m) T.rows.push_back(m < (int)tile.size() ? tile[m] : -1);
        for (int64_t u = 0; u < nch * kTsChunk; ++u)
            T.halo.push_back(u < (int64_t)hl.size() ? hl[(size_t)u] : -1);
        // adjacency of the tile as one 64-bit row mask per (chunk, tile row):
        // bit u of abits[chunk][m] <=> edge (row m, halo slot 64 chunk + u)
        const size_t base = T.abits.size();
        T.abits.resize(base + (size_t)nch * kTsRows, 0ull);
        for (int m = 0; m < (int)tile.size(); ++m) {
            const int32_t i = tile[m];
            for (int32_t e = rp[i]; e < rp[i + 1]; ++e) {
                const int32_t u = local[col[e]];
                T.abits[base + (size_t)(u / kTsChunk) * kTsRows + m] |= 1ull << (u % kTsChunk);
            }
        }
        for (int32_t h : hl) local[h] = -1;
        T.n_chunks += nch;
        T.chunk_beg.push_back((int32_t)T.n_chunks);
        ++T.n_tiles;
    }
    split_ctas(T, -1);
}

// Persistent-kernel work split of a TileSet: CTA b takes a contiguous run of tiles
// balanced by cost = chunks + tile_w per tile (tile_w < 0: DR_TS_TILE_W, else 0)
// -- neighbouring balls share halo rows, which the CTA then re-reads from L2
// (measured better than round-robin, DR_TS_ORDER=rr); its chunks are
// cta_chunks[cta_beg[b], cta_beg[b+1]).
void split_ctas(HostTiles &T, int64_t tile_w) {
    if (tile_w < 0) {                 // forward: weight 1 once CTAs own many tiles
        tile_w = knobs().ts_tile_w >= 0 ? knobs().ts_tile_w : (T.n_tiles >= 16 * 148 ? 1 : 0);
    }
    T.grid = std::min<int32_t>(T.n_tiles, 148);
    T.cta_beg.assign((size_t)T.grid + 1, 0);
    T.cta_chunks.clear();
    T.cta_tiles.clear();
    T.cta_chunks.reserve((size_t)T.n_chunks);
    const bool rr = knobs().ts_order_rr != 0;
    int32_t t0 = 0;
    for (int32_t b = 0; b < T.grid; ++b) {
        T.cta_beg[b] = (int32_t)T.cta_chunks.size();
        if (rr) {
            int32_t cnt = 0;
            for (int32_t t = b; t < T.n_tiles; t += T.grid, ++cnt)
                for (int32_t c = T.chunk_beg[t]; c < T.chunk_beg[t + 1]; ++c) T.cta_chunks.push_back(c);
            T.cta_tiles.push_back(b);
            T.cta_tiles.push_back(cnt);
        } else {
            const int64_t c1 = (T.n_chunks + tile_w * (int64_t)T.n_tiles) * (b + 1) / T.grid;
            int32_t t1 = t0;
            while (t1 < T.n_tiles && (b == T.grid - 1 || T.chunk_beg[t1] + tile_w * (int64_t)t1 < c1)) ++t1;
            for (int32_t c = T.chunk_beg[t0]; c < T.chunk_beg[t1]; ++c) T.cta_chunks.push_back(c);
            T.cta_tiles.push_back(t0);
            T.cta_tiles.push_back(t1 - t0);
            t0 = t1;
        }
    }
    T.tile_stride = rr ? T.grid : 1;
    T.cta_beg[T.grid] = (int32_t)T.cta_chunks.size();
}

void build_rel(const dr_rel_desc &d, bool validate, HostRel &h) {
    h.n_dst = d.n_dst;
    h.n_src = d.n_src;
    h.nnz = d.nnz;
    h.module = d.module;
    const int64_t *rp = d.row_ptr;
    const int32_t *ci = d.col_idx;
    if (validate) {
        if (rp[0] != 0 || rp[d.n_dst] != d.nnz) {
            h.st = DR_ERR_OUT_OF_RANGE;
            h.err = "row_ptr[0] != 0 or row_ptr[n_dst] != nnz";
            return;
        }
        for (int32_t i = 0; i < d.n_dst; ++i) {
            if (rp[i + 1] < rp[i]) {
                h.st = DR_ERR_OUT_OF_RANGE;
                h.err = "row_ptr not monotone at row " + std::to_string(i);
                return;
            }
            for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
                if (ci[e] < 0 || ci[e] >= d.n_src) {
                    h.st = DR_ERR_OUT_OF_RANGE;
                    h.err = "col_idx out of range at row " + std::to_string(i);
                    return;
                }
                if (e > rp[i] && ci[e] <= ci[e - 1]) {
                    h.st = DR_ERR_DUPLICATE_EDGE;
                    h.err = "row " + std::to_string(i) + " not strictly increasing";
                    return;
                }
            }
        }
        if (d.val)
            for (int64_t e = 0; e < d.nnz; ++e)
                if (!std::isfinite(d.val[e])) {
                    h.st = DR_ERR_NONFINITE;
                    h.err = "non-finite edge weight";
                    return;
                }
    }
    h.weighted = false;
    if (d.val)
        for (int64_t e = 0; e < d.nnz && !h.weighted; ++e) h.weighted = d.val[e] != 1.0f;
    // CSR (int32 offsets) and degrees
    h.rowptr.resize((size_t)d.n_dst + 1);
    h.deg_in.resize(d.n_dst);
    for (int32_t i = 0; i <= d.n_dst; ++i) h.rowptr[i] = (int32_t)rp[i];
    h.col.assign(ci, ci + d.nnz);
    h.deg_out.assign((size_t)d.n_src, 0);
    for (int32_t i = 0; i < d.n_dst; ++i) {
        h.deg_in[i] = (int32_t)(rp[i + 1] - rp[i]);
        h.max_in = std::max(h.max_in, h.deg_in[i]);
    }
    for (int64_t e = 0; e < d.nnz; ++e) h.deg_out[ci[e]]++;
    for (int32_t j = 0; j < d.n_src; ++j) h.max_out = std::max(h.max_out, h.deg_out[j]);
    // optional caller inputs (dr_rel_desc): degrees >= 0, normalisers finite
    auto bad = [&](dr_status st, const std::string &m) { h.st = st; h.err = m; };
    if (d.tval && !d.col_ptr) return bad(DR_ERR_INVALID_ARGUMENT, "tval given without col_ptr");
    if (d.nnz > 0 && (d.col_ptr == nullptr) != (d.row_idx == nullptr))
        return bad(DR_ERR_INVALID_ARGUMENT, "col_ptr and row_idx must be given together");
    for (int32_t i = 0; d.deg_dst && i < d.n_dst; ++i)
        if (d.deg_dst[i] < 0) return bad(DR_ERR_OUT_OF_RANGE, "negative deg_dst");
    for (int32_t j = 0; d.deg_src && j < d.n_src; ++j)
        if (d.deg_src[j] < 0) return bad(DR_ERR_OUT_OF_RANGE, "negative deg_src");
    for (int32_t i = 0; d.norm_dst && i < d.n_dst; ++i)
        if (!std::isfinite(d.norm_dst[i])) return bad(DR_ERR_NONFINITE, "non-finite norm_dst");
    for (int32_t j = 0; d.norm_src && j < d.n_src; ++j)
        if (!std::isfinite(d.norm_src[j])) return bad(DR_ERR_NONFINITE, "non-finite norm_src");
    // normalisers (reading Q12: unweighted counts clamped to >= 1), from the
    // caller's degrees or normalisers when given
    h.c.resize(d.n_dst);
    h.s.resize(d.n_src);
    for (int32_t i = 0; i < d.n_dst; ++i) {
        const double dg = std::max(d.deg_dst ? d.deg_dst[i] : h.deg_in[i], 1);
        h.c[i] = d.norm_dst ? d.norm_dst[i]
                            : (float)(d.module == DR_SAGE_MEAN ? 1.0 / dg : 1.0 / std::sqrt(dg));
    }
    for (int32_t j = 0; j < d.n_src; ++j) {
        const double dg = std::max(d.deg_src ? d.deg_src[j] : h.deg_out[j], 1);
        h.s[j] = d.norm_src ? d.norm_src[j]
                            : (float)(d.module == DR_SAGE_MEAN ? 1.0 : 1.0 / std::sqrt(dg));
    }
    // forward per-edge weight a_e * s_j (absent when identically 1)
    bool s_one = true;
    for (int32_t j = 0; j < d.n_src && s_one; ++j) s_one = h.s[j] == 1.0f;
    if (h.weighted || d.module != DR_SAGE_MEAN || !s_one) {
        h.ew.resize(d.nnz);
        for (int64_t e = 0; e < d.nnz; ++e) h.ew[e] = (d.val ? d.val[e] : 1.0f) * h.s[ci[e]];
    }
    // CSC (Alg. 2 stage 1): the caller's, used as given when validation
    // is skipped (and its weights are known), else built by counting sort and the
    // caller's, if any, checked against it
    if (d.col_ptr && !validate && (!h.weighted || d.tval)) {
        h.colptr.resize((size_t)d.n_src + 1);
        for (int32_t j = 0; j <= d.n_src; ++j) h.colptr[j] = (int32_t)d.col_ptr[j];
        h.row.assign(d.row_idx, d.row_idx + d.nnz);
        if (h.weighted) h.ewT.assign(d.tval, d.tval + d.nnz);
        return;
    }
    h.colptr.assign((size_t)d.n_src + 1, 0);
    for (int32_t j = 0; j < d.n_src; ++j) h.colptr[j + 1] = h.colptr[j] + h.deg_out[j];
    h.row.resize(d.nnz);
    if (h.weighted) h.ewT.resize(d.nnz);
    std::vector<int32_t> fill(h.colptr.begin(), h.colptr.end() - 1);
    for (int32_t i = 0; i < d.n_dst; ++i)
        for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
            const int32_t p = fill[ci[e]]++;
            h.row[p] = i;
            if (h.weighted) h.ewT[p] = d.val[e];
        }
    if (d.col_ptr) {
        bool same = d.col_ptr[0] == 0;
        for (int32_t j = 0; same && j < d.n_src; ++j) same = d.col_ptr[j + 1] == h.colptr[j + 1];
        for (int64_t p = 0; same && p < d.nnz; ++p) same = d.row_idx[p] == h.row[p];
        if (same && d.tval) {
            std::vector<int32_t> pos(h.colptr.begin(), h.colptr.end() - 1);
            for (int32_t i = 0; same && i < d.n_dst; ++i)
                for (int64_t e = rp[i]; same && e < rp[i + 1]; ++e)
                    same = d.tval[pos[ci[e]]++] == (d.val ? d.val[e] : 1.0f);
        }
        if (!same) return bad(DR_ERR_TRANSPOSE_MISMATCH, "col_ptr/row_idx/tval is not CSR^T");
    }
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

template <typename T>
size_t vbytes(const std::vector<T> &v) {
    return align_up(v.size() * sizeof(T));
}

}  // namespace

int warp_row_threshold() {
    const int64_t v = knobs().warp_row_deg;        // experiments only
    return v >= 0 ? (int)v : 32;   // measured best on C2 (k=8) and C4 (k=16): profiles/r01/ab_*.txt
}

void *Alloc::get(size_t bytes, cudaStream_t s) {
    if (bytes == 0) bytes = 256;
    void *p = nullptr;
    if (custom) {
        p = a.alloc(a.ctx, bytes, (void *)s);
        if (!p) fail(DR_ERR_OUT_OF_MEMORY, "allocator returned NULL");
        return p;
    }
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(DR_ERR_OUT_OF_MEMORY, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    return p;
}

void Alloc::put(void *p, cudaStream_t s) {
    if (!p) return;
    if (custom) a.free(a.ctx, p, (void *)s);
    else cudaFree(p);
}

}  // namespace dr

using namespace dr;

extern "C" dr_status dr_graph_create(int32_t n_cell, int32_t n_net, const dr_rel_desc rel[3],
                                     const dr_allocator *a, int32_t n_threads, uint32_t flags,
                                     void *stream, dr_graph **out) {
    clear_error();
    dr_graph *g = nullptr;
    try {
        DR_CHECK(out && rel, DR_ERR_INVALID_ARGUMENT, "null rel/out");
        *out = nullptr;
        DR_CHECK(n_cell >= 0 && n_net >= 0, DR_ERR_INVALID_ARGUMENT, "negative node count");
        const int32_t want_dst[3] = {n_cell, n_net, n_cell};
        const int32_t want_src[3] = {n_cell, n_cell, n_net};
        const char *names[3] = {"near", "pins", "pinned"};
        for (int r = 0; r < 3; ++r) {
            const dr_rel_desc &d = rel[r];
            DR_CHECK(d.n_dst == want_dst[r] && d.n_src == want_src[r], DR_ERR_SHAPE_MISMATCH,
                     std::string(names[r]) + ": n_dst/n_src disagree with n_cell/n_net");
            DR_CHECK(d.nnz >= 0 && d.nnz < (int64_t)INT32_MAX, DR_ERR_UNSUPPORTED,
                     std::string(names[r]) + ": nnz must be < 2^31");
            DR_CHECK(d.row_ptr && (d.nnz == 0 || d.col_idx), DR_ERR_INVALID_ARGUMENT,
                     std::string(names[r]) + ": null CSR pointer");
            DR_CHECK(d.module == DR_SAGE_MEAN || d.module == DR_GRAPHCONV_SYM,
                     DR_ERR_INVALID_ARGUMENT, "bad module");
        }
        const bool validate = !(flags & DR_GRAPH_SKIP_VALIDATION);
        const bool identity = (flags & DR_GRAPH_ORDER_IDENTITY) != 0;
        cudaStream_t cs = (cudaStream_t)stream;

        // ---- phase 1: per-relation host preprocessing on worker threads (§3.4)
        HostRel h[3];
        const int nt = n_threads <= 0 ? 3 : std::min(n_threads, 3);
        {
            std::vector<std::thread> th;
            for (int w = 0; w < nt; ++w)
                th.emplace_back([&, w] {
                    for (int r = w; r < 3; r += nt) build_rel(rel[r], validate, h[r]);
                });
            for (auto &t : th) t.join();
        }
        for (int r = 0; r < 3; ++r)
            if (h[r].st != DR_OK) fail(h[r].st, std::string(names[r]) + ": " + h[r].err);
        // pinned == pins^T: CSR(pinned) must equal CSC(pins) exactly
        if (validate) {
            const bool same = h[DR_PINNED].rowptr == h[DR_PINS].colptr &&
                              h[DR_PINNED].col == h[DR_PINS].row;
            DR_CHECK(same, DR_ERR_TRANSPOSE_MISMATCH, "pinned is not the transpose of pins");
        }
        const bool pins_T = h[DR_PINNED].rowptr == h[DR_PINS].colptr &&
                            h[DR_PINNED].col == h[DR_PINS].row;
        const bool near_sym = h[DR_NEAR].rowptr == h[DR_NEAR].colptr &&
                              h[DR_NEAR].col == h[DR_NEAR].row;

        // locality ranks: cells by BFS over the near graph,
        // nets by their lowest-ranked member cell; DR_ORDER=degree drops them
        std::vector<int64_t> rank_c, rank_n;
        const bool use_loc = !identity && !knobs().order_degree;
        if (use_loc) {
            rank_c = bfs_rank(n_cell, h[DR_NEAR].rowptr, h[DR_NEAR].col);
            rank_n.assign((size_t)n_net, 0);
            const HostRel &pn = h[DR_PINS];         // rows = nets, cols = member cells
            for (int32_t j = 0; j < n_net; ++j) {
                int64_t m = (int64_t)n_cell + j;
                for (int32_t e = pn.rowptr[j]; e < pn.rowptr[j + 1]; ++e)
                    m = std::min(m, rank_c[pn.col[e]]);
                rank_n[j] = m;
            }
        }
        const int wdeg = warp_row_threshold();
        // tiled form of near for the tensor-core SpMM (tspmm.cu): unit weights,
        // dense enough neighbourhoods (mean degree >= 8); DR_TILES=0 disables
        HostTiles tl, tlT;
        const HostRel &hn = h[DR_NEAR];
        const bool want_tiles = !identity && knobs().tiles != 0 && hn.ew.empty() &&
                                hn.ewT.empty() && hn.n_dst > 0 && hn.nnz >= 8LL * hn.n_dst;
        std::thread tile_th;
        // symmetric near: one TileSet for both directions, but the backward gets
        // its own CTA split. Per-tile weights (in chunk units) once CTAs own >= 16
        // tiles: forward 1, backward 2 (its epilogue samples and writes dense dX
        // rows); with a few tiles per CTA (C2) 0 is best for both -- measured,
        // profiles/r01/ab_tile_weight.txt; DR_TS_TILE_W(_BWD) override
        HostTiles tlB;
        if (want_tiles)
            tile_th = std::thread([&] {
                build_tiles(hn.n_dst, hn.rowptr, hn.col, rank_c, tl);
                if (!near_sym) {
                    build_tiles(hn.n_src, hn.colptr, hn.row, rank_c, tlT);
                } else {
                    tlB.n_tiles = tl.n_tiles;
                    tlB.n_chunks = tl.n_chunks;
                    tlB.chunk_beg = tl.chunk_beg;
                    split_ctas(tlB, knobs().ts_tile_w_bwd >= 0 ? knobs().ts_tile_w_bwd
                                                              : (tl.n_tiles >= 16 * 148 ? 2 : 0));
                }
            });
        {
            const std::vector<int64_t> *dst_loc[3] = {&rank_c, &rank_n, &rank_c};
            const std::vector<int64_t> *src_loc[3] = {&rank_c, &rank_c, &rank_n};
            std::vector<std::thread> th;
            for (int r = 0; r < 3; ++r)
                th.emplace_back([&, r] {
                    make_order(h[r].deg_in, identity, *dst_loc[r], wdeg, h[r].order, h[r].n_hub,
                               h[r].n_warp);
                    make_order(h[r].deg_out, identity, *src_loc[r], wdeg, h[r].orderT,
                               h[r].n_hubT, h[r].n_warpT);
                });
            for (auto &t : th) t.join();
        }
        // source schedules for the fused per-source-type backward
        std::vector<int32_t> degc((size_t)n_cell), degn((size_t)n_net), ord_c, ord_n;
        for (int32_t j = 0; j < n_cell; ++j)
            degc[j] = h[DR_NEAR].deg_out[j] + h[DR_PINS].deg_out[j];
        for (int32_t j = 0; j < n_net; ++j) degn[j] = h[DR_PINNED].deg_out[j];
        int32_t hub_c = 0, hub_n = 0, warp_c = 0, warp_n = 0;
        make_order(degc, identity, rank_c, wdeg, ord_c, hub_c, warp_c);
        make_order(degn, identity, rank_n, wdeg, ord_n, hub_n, warp_n);
        if (tile_th.joinable()) tile_th.join();

        // ---- phase 2: one device block, carved per array
        g = new dr_graph();
        static std::atomic<uint64_t> next_uid{1};
        g->uid = next_uid++;
        g->n_cell = n_cell;
        g->n_net = n_net;
        g->create_stream = cs;
        if (a && a->alloc && a->free) {
            g->alloc.a = *a;
            g->alloc.custom = true;
        }
        struct Up {
            void **dst;
            const void *src;
            size_t bytes;
        };
        std::vector<Up> ups[4];            // [0..2] per relation, [3] shared
        size_t total = 0;
        auto plan = [&](int q, void **dst, const void *src, size_t bytes) {
            if (bytes == 0) { *dst = nullptr; return; }
            ups[q].push_back({dst, src, total});
            *dst = (void *)bytes;           // temporarily the size
            total += align_up(bytes);
        };
        for (int r = 0; r < 3; ++r) {
            RelDev &d = g->rel[r];
            HostRel &hr = h[r];
            d.n_dst = hr.n_dst;
            d.n_src = hr.n_src;
            d.nnz = hr.nnz;
            d.module = hr.module;
            d.fwd.n = hr.n_dst;
            d.fwd.n_hub = hr.n_hub;
            d.fwd.n_warp = hr.n_warp;
            d.bwd.n = hr.n_src;
            d.bwd.n_hub = hr.n_hubT;
            d.bwd.n_warp = hr.n_warpT;
            d.max_deg_dst = hr.max_in;
            d.max_deg_src = hr.max_out;
            plan(r, (void **)&d.rowptr, hr.rowptr.data(), hr.rowptr.size() * 4);
            plan(r, (void **)&d.col, hr.col.data(), hr.col.size() * 4);
            plan(r, (void **)&d.ew, hr.ew.data(), hr.ew.size() * 4);
            plan(r, (void **)&d.c, hr.c.data(), hr.c.size() * 4);
            plan(r, (void **)&d.s, hr.s.data(), hr.s.size() * 4);
            plan(r, (void **)&d.fwd.order, hr.order.data(), hr.order.size() * 4);
            plan(r, (void **)&d.bwd.order, hr.orderT.data(), hr.orderT.size() * 4);
            plan(r, (void **)&d.ewT, hr.ewT.data(), hr.ewT.size() * 4);
            const bool alias = (r == DR_NEAR && near_sym) || (r != DR_NEAR && pins_T);
            if (!alias) {
                plan(r, (void **)&d.colptr, hr.colptr.data(), hr.colptr.size() * 4);
                plan(r, (void **)&d.row, hr.row.data(), hr.row.size() * 4);
            }
        }
        auto plan_tiles = [&](TileSet &ts, HostTiles &ht) {
            ts.n_tiles = ht.n_tiles;
            ts.n_chunks = ht.n_chunks;
            plan(0, (void **)&ts.rows, ht.rows.data(), ht.rows.size() * 4);
            plan(0, (void **)&ts.chunk_beg, ht.chunk_beg.data(), ht.chunk_beg.size() * 4);
            plan(0, (void **)&ts.halo, ht.halo.data(), ht.halo.size() * 4);
            plan(0, (void **)&ts.abits, ht.abits.data(), ht.abits.size() * 8);
            ts.grid = ht.grid;
            plan(0, (void **)&ts.cta_beg, ht.cta_beg.data(), ht.cta_beg.size() * 4);
            plan(0, (void **)&ts.cta_chunks, ht.cta_chunks.data(), ht.cta_chunks.size() * 4);
            plan(0, (void **)&ts.cta_tiles, ht.cta_tiles.data(), ht.cta_tiles.size() * 4);
            ts.tile_stride = ht.tile_stride;
        };
        TileSet bsplit;                     // symmetric near: the backward's CTA split
        if (want_tiles) {
            plan_tiles(g->rel[DR_NEAR].tiles, tl);
            if (!near_sym) {
                plan_tiles(g->rel[DR_NEAR].tilesT, tlT);
            } else {
                bsplit.grid = tlB.grid;
                bsplit.tile_stride = tlB.tile_stride;
                plan(0, (void **)&bsplit.cta_beg, tlB.cta_beg.data(), tlB.cta_beg.size() * 4);
                plan(0, (void **)&bsplit.cta_chunks, tlB.cta_chunks.data(), tlB.cta_chunks.size() * 4);
                plan(0, (void **)&bsplit.cta_tiles, tlB.cta_tiles.data(), tlB.cta_tiles.size() * 4);
            }
        }
        g->src_cell.n = n_cell;
        g->src_cell.n_hub = hub_c;
        g->src_cell.n_warp = warp_c;
        g->src_net.n = n_net;
        g->src_net.n_hub = hub_n;
        g->src_net.n_warp = warp_n;
        plan(3, (void **)&g->src_cell.order, ord_c.data(), ord_c.size() * 4);
        plan(3, (void **)&g->src_net.order, ord_n.data(), ord_n.size() * 4);
        char *base = (char *)g->alloc.get(total, cs);
        g->blocks.push_back(base);
        g->bytes = total;
        for (int q = 0; q < 4; ++q)
            for (Up &u : ups[q]) {
                const size_t bytes = (size_t)reinterpret_cast<uintptr_t>(*u.dst);
                *u.dst = base + u.bytes;
                u.bytes = bytes;
            }
        // structural sharing (no second copy): CSC(near) = CSR(near) when symmetric;
        // CSC(pins) = CSR(pinned) and CSC(pinned) = CSR(pins) when pinned == pins^T.
        if (want_tiles && near_sym) {
            TileSet &tt = g->rel[DR_NEAR].tilesT;
            tt = g->rel[DR_NEAR].tiles;
            tt.grid = bsplit.grid;
            tt.tile_stride = bsplit.tile_stride;
            tt.cta_beg = bsplit.cta_beg;
            tt.cta_chunks = bsplit.cta_chunks;
            tt.cta_tiles = bsplit.cta_tiles;
        }
        if (near_sym) {
            g->rel[DR_NEAR].colptr = g->rel[DR_NEAR].rowptr;
            g->rel[DR_NEAR].row = g->rel[DR_NEAR].col;
        }
        if (pins_T) {
            g->rel[DR_PINNED].colptr = g->rel[DR_PINS].rowptr;
            g->rel[DR_PINNED].row = g->rel[DR_PINS].col;
            g->rel[DR_PINS].colptr = g->rel[DR_PINNED].rowptr;
            g->rel[DR_PINS].row = g->rel[DR_PINNED].col;
        }
        // ---- phase 3: uploads, one stream per relation on the worker threads
        DR_CUDA(cudaStreamSynchronize(cs));
        dr_status up_st[4] = {DR_OK, DR_OK, DR_OK, DR_OK};
        std::string up_err[4];
        {
            std::vector<std::thread> th;
            for (int q = 0; q < 4; ++q)
                th.emplace_back([&, q] {
                    cudaStream_t s = nullptr;
                    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
                    for (size_t i = 0; e == cudaSuccess && i < ups[q].size(); ++i)
                        e = cudaMemcpyAsync(*ups[q][i].dst, ups[q][i].src, ups[q][i].bytes,
                                            cudaMemcpyHostToDevice, s);
                    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                    if (s) cudaStreamDestroy(s);
                    if (e != cudaSuccess) {
                        up_st[q] = DR_ERR_CUDA;
                        up_err[q] = cudaGetErrorString(e);
                    }
                });
            for (auto &t : th) t.join();
        }
        for (int q = 0; q < 4; ++q)
            if (up_st[q] != DR_OK) fail(up_st[q], "upload: " + up_err[q]);
        *out = g;
        return DR_OK;
    } catch (const Error &e) {
        if (g) dr_graph_destroy(g);
        set_error(e.status, e.msg);
        return e.status;
    } catch (const std::bad_alloc &) {
        if (g) dr_graph_destroy(g);
        set_error(DR_ERR_OUT_OF_MEMORY, "host allocation failed");
        return DR_ERR_OUT_OF_MEMORY;
    }
}

namespace dr {

// One relation block with caller-given source normalisers (dr_shard, SURVEY §8
// f4): rows = this rank's destinations, columns = the padded global source
// space. build_rel's row normalisers c are already global (a row's edges are
// all local); the column normalisers s are replaced by the global ones and
// the forward edge weights recomputed from them. SIMT schedules only (no tiles).
void build_rel_block(const dr_rel_desc &d, const std::vector<float> &s_glob, int64_t own_col0,
                     Alloc &alloc, cudaStream_t cs, RelDev &out, std::vector<void *> &blocks,
                     size_t &bytes) {
    HostRel h;
    build_rel(d, true, h);
    if (h.st != DR_OK) fail(h.st, "shard block: " + h.err);
    DR_CHECK((int64_t)s_glob.size() == (int64_t)d.n_src, DR_ERR_SHAPE_MISMATCH,
             "shard block: s size");
    h.s = s_glob;
    if (h.weighted || d.module != DR_SAGE_MEAN) {
        h.ew.resize(d.nnz);
        for (int64_t e = 0; e < d.nnz; ++e)
            h.ew[e] = (d.val ? d.val[e] : 1.0f) * h.s[d.col_idx[e]];
    }
    const int wdeg = warp_row_threshold();
    const std::vector<int64_t> noloc;
    make_order(h.deg_in, false, noloc, wdeg, h.order, h.n_hub, h.n_warp);
    make_order(h.deg_out, false, noloc, wdeg, h.orderT, h.n_hubT, h.n_warpT);
    // tiles for the tensor-core SpMM, opt-in (DR_SHARD_TILES=1), under the rule of
    // dr_graph_create (unit weights, mean degree >= 8); the BFS links column c to
    // local row c - own_col0 (own_col0 < 0: no column is a local row). Measured at
    // C4 near (profiles/r01/shard_time_*.json): the block's tiled forward is at best
    // 10 % faster than the SIMT one (W = 2, shuffled ids) and slower with spatial
    // ids, so the SIMT kernels are the default for blocks.
    HostTiles tl, tlT;
    const bool want_tiles = knobs().shard_tiles == 1 && h.ew.empty() && h.ewT.empty() &&
                            h.n_dst > 0 && h.nnz >= 8LL * h.n_dst;
    if (want_tiles) {
        const int64_t off = own_col0 >= 0 ? -own_col0 : -(int64_t)h.n_src - h.n_dst - 1;
        const int64_t offT = own_col0 >= 0 ? own_col0 : -(int64_t)h.n_src - h.n_dst - 1;
        build_tiles(h.n_dst, h.rowptr, h.col, noloc, tl, h.n_src, off, true);
        // a block only tiles well when its row range is spatially compact (node ids
        // in a locality order): with < 4 edges per halo slot the tiles re-gather
        // almost every neighbour row per tile and the SIMT kernel is faster
        if (tl.n_chunks * (int64_t)kTsChunk * 4 > h.nnz) tl = HostTiles{};
        // the transposed tiles would span every padded source row, most of them
        // edge-free or remote with a few boundary edges (measured 2-3x slower than
        // the SIMT SSpMM at C4, W = 2..8): DR_SHARD_TILES_T=1 builds them anyway
        if (knobs().shard_tiles_t == 1) build_tiles(h.n_src, h.colptr, h.row, noloc, tlT, h.n_dst, offT, true);
    }
    out = RelDev{};
    out.n_dst = h.n_dst;
    out.n_src = h.n_src;
    out.nnz = h.nnz;
    out.module = h.module;
    out.fwd.n = h.n_dst;
    out.fwd.n_hub = h.n_hub;
    out.fwd.n_warp = h.n_warp;
    out.bwd.n = h.n_src;
    out.bwd.n_hub = h.n_hubT;
    out.bwd.n_warp = h.n_warpT;
    out.max_deg_dst = h.max_in;
    out.max_deg_src = h.max_out;
    struct Up {
        void **dst;
        const void *src;
        size_t bytes, off;
    };
    std::vector<Up> ups;
    size_t total = 0;
    auto plan = [&](void **dst, const void *src, size_t b) {
        *dst = nullptr;
        if (b == 0) return;
        ups.push_back({dst, src, b, total});
        total += align_up(b);
    };
    plan((void **)&out.rowptr, h.rowptr.data(), h.rowptr.size() * 4);
    plan((void **)&out.col, h.col.data(), h.col.size() * 4);
    plan((void **)&out.ew, h.ew.data(), h.ew.size() * 4);
    plan((void **)&out.c, h.c.data(), h.c.size() * 4);
    plan((void **)&out.s, h.s.data(), h.s.size() * 4);
    plan((void **)&out.fwd.order, h.order.data(), h.order.size() * 4);
    plan((void **)&out.bwd.order, h.orderT.data(), h.orderT.size() * 4);
    plan((void **)&out.ewT, h.ewT.data(), h.ewT.size() * 4);
    plan((void **)&out.colptr, h.colptr.data(), h.colptr.size() * 4);
    plan((void **)&out.row, h.row.data(), h.row.size() * 4);
    auto plan_tiles = [&](TileSet &ts, HostTiles &ht) {
        ts.n_tiles = ht.n_tiles;
        ts.n_chunks = ht.n_chunks;
        ts.grid = ht.grid;
        ts.tile_stride = ht.tile_stride;
        plan((void **)&ts.rows, ht.rows.data(), ht.rows.size() * 4);
        plan((void **)&ts.chunk_beg, ht.chunk_beg.data(), ht.chunk_beg.size() * 4);
        plan((void **)&ts.halo, ht.halo.data(), ht.halo.size() * 4);
        plan((void **)&ts.abits, ht.abits.data(), ht.abits.size() * 8);
        plan((void **)&ts.cta_beg, ht.cta_beg.data(), ht.cta_beg.size() * 4);
        plan((void **)&ts.cta_chunks, ht.cta_chunks.data(), ht.cta_chunks.size() * 4);
        plan((void **)&ts.cta_tiles, ht.cta_tiles.data(), ht.cta_tiles.size() * 4);
    };
    if (tl.n_tiles) plan_tiles(out.tiles, tl);
    if (tlT.n_tiles) plan_tiles(out.tilesT, tlT);
    char *base = (char *)alloc.get(total, cs);
    blocks.push_back(base);
    bytes += total;
    for (Up &u : ups) {
        *u.dst = base + u.off;
        DR_CUDA(cudaMemcpyAsync(*u.dst, u.src, u.bytes, cudaMemcpyHostToDevice, cs));
    }
    DR_CUDA(cudaStreamSynchronize(cs));      // host vectors die with this frame
}

}  // namespace dr

extern "C" dr_status dr_graph_destroy(dr_graph *g) {
    if (!g) return DR_OK;
    cudaStreamSynchronize(g->create_stream);
    for (void *p : g->blocks) g->alloc.put(p, g->create_stream);
    delete g;
    return DR_OK;
}

extern "C" dr_status dr_graph_info(const dr_graph *g, dr_graph_info_t *info) {
    clear_error();
    if (!g || !info) {
        set_error(DR_ERR_INVALID_ARGUMENT, "null graph/info");
        return DR_ERR_INVALID_ARGUMENT;
    }
    std::memset(info, 0, sizeof(*info));
    info->n_cell = g->n_cell;
    info->n_net = g->n_net;
    for (int r = 0; r < 3; ++r) {
        info->nnz[r] = g->rel[r].nnz;
        info->max_deg_dst[r] = g->rel[r].max_deg_dst;
        info->max_deg_src[r] = g->rel[r].max_deg_src;
        info->hub_rows_dst[r] = g->rel[r].fwd.n_hub;
        info->tiles[r] = g->rel[r].tiles.n_tiles;
        info->tiles_T[r] = g->rel[r].tilesT.n_tiles;
        info->chunks[r] = g->rel[r].tiles.n_chunks;
        info->chunks_T[r] = g->rel[r].tilesT.n_chunks;
    }
    info->hub_rows_src[0] = g->src_cell.n_hub;
    info->hub_rows_src[1] = g->src_net.n_hub;
    info->device_bytes = g->bytes;
    return DR_OK;
}

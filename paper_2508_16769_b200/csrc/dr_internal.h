// dr_internal.h — internal types of libdr (B200 / sm_100a). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dr.h"

namespace dr {

// ------------------------------------------------------------------ errors
struct Error {
    dr_status status;
    std::string msg;
};
void set_error(dr_status s, const std::string &msg);
void clear_error();
[[noreturn]] void fail(dr_status s, const std::string &msg);

#define DR_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            ::dr::fail(DR_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)
#define DR_CHECK(cond, status, msg)                                                          \
    do {                                                                                     \
        if (!(cond)) ::dr::fail(status, msg);                                                \
    } while (0)

// Experiment / profiling switches (knobs.cpp): read once from the environment
// at library load, overridable through dr_debug_set; never read on a launch path.
struct Knobs {
    int64_t nvtx = 0;            // DR_NVTX: NVTX range per launch named by its profile tag
    int64_t no_graph = 0;        // DR_NO_GRAPH: train steps run eagerly (no CUDA graph)
    int64_t dense_simt = 0;      // DR_DENSE_SIMT: SIMT projections / dW instead of tcgen05
    int64_t tspmm = 1;           // DR_TSPMM=0: SIMT kernels for near instead of the tiled ones
    int64_t ts_zerofill = 0;     // DR_TS_ZEROFILL: TMA zero fill of the tiled forward's B tile
    int64_t ts_debug = 0;        // DR_TS_DEBUG: per-role cycle counters of the tiled SpMM
    int64_t tc2_debug = 0;       // DR_TC2_DEBUG: per-role cycle counters of the tc2 GEMMs
    int64_t bwd_p = 0;           // DR_BWD_P: pairs per lane of the SIMT SSpMM (0 = chosen)
    int64_t drelu_bs = 0;        // DR_DRELU_BS: binary-search D-ReLU for every k
    int64_t drelu_tpr = 1;       // DR_DRELU_TPR: 0 warp-per-row only, 1 thread-per-row where faster, 2 wherever supported
    int64_t tiles = 1;           // DR_TILES=0: no BFS-ball tiles at graph creation
    int64_t order_degree = 0;    // DR_ORDER=degree: degree buckets without the locality rank
    int64_t warp_row_deg = -1;   // DR_WARP_ROW_DEG: warp-row degree threshold (-1 = 32)
    int64_t ts_tile_w = -1;      // DR_TS_TILE_W: forward CTA-split tile weight (-1 = adaptive)
    int64_t ts_tile_w_bwd = -1;  // DR_TS_TILE_W_BWD: backward CTA-split tile weight
    int64_t ts_order_rr = 0;     // DR_TS_ORDER=rr: round-robin tile assignment
    int64_t shard_tiles = 0;     // DR_SHARD_TILES: tiled forward for shard blocks
    int64_t shard_tiles_t = 0;   // DR_SHARD_TILES_T: tiled backward for shard blocks
    int64_t order_block = -2;    // DR_ORDER_BLOCK: log2 rows per locality block of the SIMT orders (-1: degree-major, -2: by size)
    int64_t z_split = 1;         // DR_Z_SPLIT=0: Z stored fp32 (converted by each consumer)
    int64_t tc2_ewg = 1;         // DR_TC2_EWG: epilogue warpgroups of the row GEMM (1 default; 0 auto = 2 for the head / dZ' with root; 2 forced where smem permits)
    int64_t seq_streams = 0;     // DR_SEQ: every relation on the caller's stream (A/B of the 3-stream schedule)
    int64_t spmm_wpc = 8;        // DR_SPMM_WPC: warps per CTA of the SIMT SpMM / SSpMM (8, 4, 2)
    int64_t ts_sa = 0;           // DR_TS_SA: cap on the tiled SpMM's A stages (0: as many as fit, <= 4)
    int64_t dw_dual = 1;         // DR_DW_DUAL: near + pinned weight gradients in one reduce launch (dual B)
    int64_t tpr_stream = 1;      // DR_TPR_STREAM: thread-per-row network in rolled chunks: 1 epilogue + D = 128 standalone, 2 everywhere, 0 never
    int64_t drelu_coop = -2;     // DR_DRELU_COOP: lanes per row of the thread-per-row D-ReLU (-2 auto, 0 off)
    int64_t head_fuse = 1;       // DR_HEAD_FUSE=0: trainer head + MSE as its own kernels
    int64_t chain = 1;           // DR_CHAIN=0: trainer without the fused next-layer D-ReLU
    int64_t skip_dead_net = 1;   // DR_SKIP_DEAD_NET=0: trainer computes the last layer's Y_net
};
const Knobs &knobs();

// Opt a kernel into > 48 KB of dynamic shared memory on the current device (once).
void ensure_smem(const void *fn, size_t bytes);

// Launch bookkeeping: count kernels and surface launch errors immediately.
void note_launch(const char *name);

// Optional per-launch device timing (dr_profile_begin/end): events recorded on
// the launch stream around the kernel; the name is "<base>.<current tag>".
struct ProfScope {
    cudaStream_t s = nullptr;
    cudaEvent_t a = nullptr;
    const char *base = nullptr;
    bool nvtx = false;
    ProfScope(const char *base, cudaStream_t s);
    ~ProfScope();
};
// Tag naming the relation / role of the launches issued while it is alive.
struct TagScope {
    std::string prev;
    explicit TagScope(const char *tag);
    ~TagScope();
};

// ------------------------------------------------------------------ allocation
struct Alloc {
    dr_allocator a{};
    bool custom = false;
    void *get(size_t bytes, cudaStream_t s);
    void put(void *p, cudaStream_t s);
};

// ------------------------------------------------------------------ device graph
// Rows whose work exceeds this many neighbours go to the CTA-per-row kernels
// (Alg. 1 stage 2 "high degree" class); the rest are packed several
// rows per warp (one sub-warp of k/P lanes per row, "partition into
// ceil(32/K) parts").
constexpr int kHubDeg = 256;

// A processing order over the rows of one kernel (destinations for the
// forward, sources for the backward), split into the degree classes of Alg. 1
// stage 2: [hubs | warp rows | sub-warp rows]. Hubs (deg >
// kHubDeg) get a CTA each, warp rows (warp_deg < deg <= kHubDeg) a warp each,
// sub-warp rows (deg <= warp_deg) share a warp. Inside the warp and sub-warp
// classes rows are grouped by power-of-two degree bucket (descending, so a warp
// holds rows of similar work) and ordered by a locality rank inside a bucket
// (BFS over the near graph), so rows processed at the same time share
// neighbours and their gathers hit L2. Fixed at graph creation.
struct Sched {
    int32_t n = 0;
    int32_t *order = nullptr;            // device [n]
    int32_t n_hub = 0, n_warp = 0;
};
// Degree above which a non-hub row gets a whole warp (its R sub-warps take
// every R-th neighbour); 32 measured best for k = 8 and 16 (profiles/r01);
// DR_WARP_ROW_DEG overrides it at graph creation (experiments only).
int warp_row_threshold();

// Tiled form of a square, unit-weight relation for the tensor-core SpMM
// (tspmm.cu): the rows are cut into tiles of <= 128 rows grown as BFS balls
// over the relation itself (compact neighbourhoods), and each tile lists its
// halo = the distinct column ids its rows touch, padded to 64-id chunks (-1).
// The tile's adjacency restricted to one chunk is a 128 x 64 bit matrix, stored
// as one 64-bit mask per tile row (1 KB per chunk, whatever the density). A
// tile's aggregation is then the dense product Adj_tile[128 x U] * X_halo[U x D]
// with a 0/1 adjacency operand, one 64-wide K chunk at a time (SURVEY §7.3-2a
// locality, made explicit).
constexpr int kTsRows = 128;
constexpr int kTsChunk = 64;
struct TileSet {
    int32_t n_tiles = 0;
    int64_t n_chunks = 0;
    int32_t *rows = nullptr;        // [n_tiles * 128], -1 padded
    int32_t *chunk_beg = nullptr;   // [n_tiles + 1] chunk range of a tile
    int32_t *halo = nullptr;        // [n_chunks * 64], -1 padded
    uint64_t *abits = nullptr;      // [n_chunks * 128] row masks: bit u of [c][m] <=> edge (m, 64 c + u)
    int32_t grid = 0;               // persistent CTAs of the kernels (min(n_tiles, 148))
    int32_t *cta_beg = nullptr;     // [grid + 1] CTA b's chunks are cta_chunks[cta_beg[b], cta_beg[b+1])
    int32_t *cta_chunks = nullptr;  //   in processing order;
    int32_t *cta_tiles = nullptr;   // [grid][2] its tiles: first, count (step tile_stride)
    int32_t tile_stride = 1;
};

struct RelDev {
    int32_t n_dst = 0, n_src = 0;
    int64_t nnz = 0;
    dr_module module = DR_SAGE_MEAN;
    // forward: CSR rows = destinations
    int32_t *rowptr = nullptr;   // [n_dst+1]
    int32_t *col = nullptr;      // [nnz]
    float *ew = nullptr;         // [nnz] a_e * s_col(e); nullptr when identically 1
    float *c = nullptr;          // [n_dst]
    float *s = nullptr;          // [n_src]
    Sched fwd;                   // destination rows
    // backward: CSC rows = sources
    int32_t *colptr = nullptr;   // [n_src+1]
    int32_t *row = nullptr;      // [nnz]
    float *ewT = nullptr;        // [nnz] a_ij in CSC order; nullptr when identically 1
    Sched bwd;                   // source rows of this relation alone (standalone dr_spmm_bwd)
    TileSet tiles;               // tiled CSR (rows = dst); n_tiles == 0 when not built
    TileSet tilesT;              // tiled CSC (rows = src); aliases `tiles` when symmetric
    int32_t max_deg_dst = 0, max_deg_src = 0;
};

// Source-side schedules for the fused per-source-type SSpMM (cell sources sum
// near + pins, net sources use pinned; Alg. 2 stage 2 "for each source node
// type") are plain Scheds over the combined CSC degree.
using SrcSched = Sched;

}  // namespace dr

struct dr_graph {
    uint64_t uid = 0;                    // unique per created graph (CUDA-graph cache key)
    int32_t n_cell = 0, n_net = 0;
    dr::RelDev rel[3];
    dr::SrcSched src_cell, src_net;
    dr::Alloc alloc;
    std::vector<void *> blocks;
    size_t bytes = 0;
    cudaStream_t create_stream = nullptr;
};

// one relation's destination-row block on one rank (shard.cpp, f4)
struct dr_shard {
    int32_t world = 1, rank = 0, max_src = 0;
    int64_t dst_begin = 0, dst_end = 0, src_begin = 0, src_end = 0;
    int32_t n_src_glob = 0;
    dr::RelDev rel;                 // rows = local destinations, cols = padded sources
    dr::Alloc alloc;
    std::vector<void *> blocks;
    size_t bytes = 0;
    cudaStream_t stream = nullptr;
};

namespace dr {

// ------------------------------------------------------------------ kernels (launchers)
// D-ReLU (Eq. 2-3): x [n x dim] (ld ldx) -> CBSR val [n x k], idx [n x k] (uint8).
// sorted: rows in value-descending order (ties: lower column first), k <= 32.
void launch_drelu(const float *x, int64_t n, int dim, int64_t ldx, int k, float *val,
                  uint8_t *idx, cudaStream_t s, bool sorted = false);

// NEXT-2 per-neighbour-group K (reading Q26): a destination row with in-degree d
// keeps the first K(d) entries of each neighbour's value-sorted CBSR row,
// K(d) = kb[0] (d <= thr[0]), kb[1] (d <= thr[1]), kb[2] (otherwise). ng.on == 0: off.
// f4, fused exchange over peer memory: the source row j of the padded global
// space lives in owner q = j / m's buffers at local row j - q m (read in place by
// the SpMM, through NVLink when q is another GPU); the backward's per-source
// contributions go to the owner's inbox, slot `rank` (written in place).
constexpr int kMaxPeers = 8;
struct PeerSrc {
    const float *pv[kMaxPeers];
    const uint8_t *pi[kMaxPeers];
    float *pg[kMaxPeers];
    int m, rank;
};
struct NgSched {
    int on = 0;
    int thr0 = 0, thr1 = 0, kb0 = 0, kb1 = 0, kb2 = 0;
    const uint8_t *kT = nullptr;     // backward: K(deg of row[e]) per CSC edge e (launch_ng_edge_k)
};
// kT[e] = K(deg_dst(row[e])) for every CSC edge of r (one byte per edge), so the
// backward reads its destinations' K coalesced beside row[] instead of gathering
// two rowptr entries per edge.
// dx[i, :] = 0 except dx[i, idx[i, t]] = g[i, t] (the D-ReLU mask gradient scatter)
// f4 sharded layer: out[e] = root[e] (root may be null) + sum over nslots slots
// (slot_stride apart) of inbox[e], fixed order; out may alias root
void launch_inbox_root(const float *inbox, int nslots, int64_t slot_stride, const float *root,
                       int64_t n, float *out, cudaStream_t s);
// f4: out = fixed-order sum over `world` stacked [n] blocks of `inbox`
void launch_inbox_sum(const float *inbox, int world, int64_t n, float *out, cudaStream_t s);
void launch_cbsr_scatter(const float *g, const uint8_t *idx, int64_t n, int k, int dim, float *dx,
                         cudaStream_t s);
// A relation block uploaded with caller-given column normalisers (graph.cpp; dr_shard).
// own_col0: the block's columns [own_col0, own_col0 + n_dst) are its own rows
// (square relation, same source and destination partition), else -1.
void build_rel_block(const dr_rel_desc &d, const std::vector<float> &s_glob, int64_t own_col0,
                     Alloc &alloc, cudaStream_t cs, RelDev &out, std::vector<void *> &blocks,
                     size_t &bytes);
void launch_ng_edge_k(const RelDev &r, const NgSched &ng, uint8_t *kT, cudaStream_t s);

// DR-SpMM forward of one relation: z [n_dst x dim] = diag(c) A diag(s) densify(H).
// z_split: write Z rows as [hi | lo] bf16 halves (the tc2 operand format).
void launch_spmm_fwd(const RelDev &r, const float *hval, const uint8_t *hidx, int k, int dim,
                     float *z, cudaStream_t s, bool z_split = false, NgSched ng = NgSched{},
                     const PeerSrc *peer = nullptr);

// SSpMM backward for one source node type, summing up to two relations that
// share the source type. Term q in {0,1}: relation rel[q] (CSC), its dz, and
// whether the kernel applies c_i per edge (standalone ABI) or dz is already
// row-scaled (fused path). root (n_src x k) is added if non-null.
struct BwdTerm {
    const RelDev *rel = nullptr;
    const float *dz = nullptr;
    bool apply_c = false;
};
void launch_spmm_bwd(const SrcSched &sched, int n_src, BwdTerm t0, BwdTerm t1,
                     const float *root, const uint8_t *hidx, int k, int dim, float *g_kept,
                     float *dx, bool accumulate, cudaStream_t s, NgSched ng = NgSched{},
                     const PeerSrc *peer = nullptr);

// Tensor-core tiled SpMM (tspmm.cu) of a relation with a TileSet: forward into
// z; backward for the tiled relation's source rows alone, with an optional
// extra [n_src x k] term added at the kept entries (root + other relations).
bool tspmm_supported(const TileSet &ts, int dim, int k);
void launch_tspmm_fwd(const RelDev &r, const float *hval, const uint8_t *hidx, int k, int dim,
                      float *z, cudaStream_t s, bool z_split = false);
// dz_split: dz holds [hi | lo] bf16 rows (tc2 dz epilogue, Tc2RowsDesc::dz_split).
void launch_tspmm_bwd(const RelDev &r, const float *dz, bool dz_split, bool apply_c,
                      const float *extra, const uint8_t *hidx, int k, int dim, float *g_kept,
                      float *dx, cudaStream_t s);

}  // namespace dr

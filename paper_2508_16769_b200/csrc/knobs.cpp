// knobs.cpp — experiment / profiling switches of libdr, read ONCE from the
// environment when the library loads (never on a launch path), and settable
// afterwards through dr_debug_set (tests and A/B tools). None of them changes
// a result except by choosing between two parity-tested kernel paths.
#include <cstdlib>
#include <cstring>
#include <string>

#include "dr_internal.h"

namespace dr {

static int64_t env_i(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return (e && *e) ? (int64_t)atoll(e) : dflt;
}

static Knobs read_env() {
    Knobs k;
    k.nvtx = env_i("DR_NVTX", 0);
    k.no_graph = env_i("DR_NO_GRAPH", 0);
    k.dense_simt = env_i("DR_DENSE_SIMT", 0);
    k.tspmm = env_i("DR_TSPMM", 1);
    k.ts_zerofill = env_i("DR_TS_ZEROFILL", 0);
    k.ts_debug = env_i("DR_TS_DEBUG", 0);
    k.tc2_debug = env_i("DR_TC2_DEBUG", 0);
    k.bwd_p = env_i("DR_BWD_P", 0);
    k.drelu_bs = env_i("DR_DRELU_BS", 0);
    k.drelu_tpr = env_i("DR_DRELU_TPR", 1);
    k.tiles = env_i("DR_TILES", 1);
    const char *o = getenv("DR_ORDER");
    k.order_degree = (o && std::string(o) == "degree") ? 1 : 0;
    k.warp_row_deg = env_i("DR_WARP_ROW_DEG", -1);
    k.ts_tile_w = env_i("DR_TS_TILE_W", -1);
    k.ts_tile_w_bwd = env_i("DR_TS_TILE_W_BWD", -1);
    const char *r = getenv("DR_TS_ORDER");
    k.ts_order_rr = (r && std::string(r) == "rr") ? 1 : 0;
    k.shard_tiles = env_i("DR_SHARD_TILES", 0);
    k.shard_tiles_t = env_i("DR_SHARD_TILES_T", 0);
    k.chain = env_i("DR_CHAIN", 1);
    k.head_fuse = env_i("DR_HEAD_FUSE", 1);
    k.drelu_coop = env_i("DR_DRELU_COOP", -2);
    k.tpr_stream = env_i("DR_TPR_STREAM", 1);
    k.dw_dual = env_i("DR_DW_DUAL", 1);
    k.spmm_wpc = env_i("DR_SPMM_WPC", 8);
    k.ts_sa = env_i("DR_TS_SA", 0);
    k.seq_streams = env_i("DR_SEQ", 0);
    k.tc2_ewg = env_i("DR_TC2_EWG", 1);
    k.z_split = env_i("DR_Z_SPLIT", 1);
    k.order_block = env_i("DR_ORDER_BLOCK", -2);
    k.skip_dead_net = env_i("DR_SKIP_DEAD_NET", 1);
    return k;
}

static Knobs g_knobs = read_env();

const Knobs &knobs() { return g_knobs; }

}  // namespace dr

using namespace dr;

extern "C" dr_status dr_debug_set(const char *name, int64_t value) {
    if (!name) return DR_ERR_INVALID_ARGUMENT;
    struct {
        const char *n;
        int64_t *p;
    } tab[] = {
        {"nvtx", &g_knobs.nvtx},
        {"no_graph", &g_knobs.no_graph},
        {"dense_simt", &g_knobs.dense_simt},
        {"tspmm", &g_knobs.tspmm},
        {"ts_zerofill", &g_knobs.ts_zerofill},
        {"ts_debug", &g_knobs.ts_debug},
        {"tc2_debug", &g_knobs.tc2_debug},
        {"bwd_p", &g_knobs.bwd_p},
        {"drelu_bs", &g_knobs.drelu_bs},
        {"drelu_tpr", &g_knobs.drelu_tpr},
        {"tiles", &g_knobs.tiles},
        {"order_degree", &g_knobs.order_degree},
        {"warp_row_deg", &g_knobs.warp_row_deg},
        {"ts_tile_w", &g_knobs.ts_tile_w},
        {"ts_tile_w_bwd", &g_knobs.ts_tile_w_bwd},
        {"ts_order_rr", &g_knobs.ts_order_rr},
        {"shard_tiles", &g_knobs.shard_tiles},
        {"shard_tiles_t", &g_knobs.shard_tiles_t},
        {"chain", &g_knobs.chain},
        {"head_fuse", &g_knobs.head_fuse},
        {"drelu_coop", &g_knobs.drelu_coop},
        {"tpr_stream", &g_knobs.tpr_stream},
        {"dw_dual", &g_knobs.dw_dual},
        {"spmm_wpc", &g_knobs.spmm_wpc},
        {"ts_sa", &g_knobs.ts_sa},
        {"seq_streams", &g_knobs.seq_streams},
        {"tc2_ewg", &g_knobs.tc2_ewg},
        {"z_split", &g_knobs.z_split},
        {"order_block", &g_knobs.order_block},
        {"skip_dead_net", &g_knobs.skip_dead_net},
    };
    for (auto &t : tab)
        if (std::strcmp(t.n, name) == 0) {
            *t.p = value;
            return DR_OK;
        }
    return DR_ERR_INVALID_ARGUMENT;
}

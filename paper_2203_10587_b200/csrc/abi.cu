// C ABI of libacopf_b200.so: batch planning on the host, device residency,
// and the evaluation launch.  See include/acopf_b200.h for the contract.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <queue>
#include <mutex>
#include <thread>
#include <atomic>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/acopf_b200.h"
#include "eval_kernel.cuh"
#include "sl_kernel.cuh"
#include "kkt.cuh"
#include "planner.hpp"
#include "writer.hpp"

using namespace acopf;

namespace {
thread_local std::string g_err;

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    template <class T>
    T* upload(const std::vector<T>& v) {
        release();                      // a re-upload (new layout) replaces the buffer
        n = std::max<size_t>(sizeof(T) * v.size(), 16);
        cuda_check(cudaMalloc(&p, n), "cudaMalloc");
        if (!v.empty()) cuda_check(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice), "H2D");
        return static_cast<T*>(p);
    }
    void* alloc(size_t bytes) {
        release();
        n = std::max<size_t>(bytes, 16);
        cuda_check(cudaMalloc(&p, n), "cudaMalloc");
        // setup-time zeroing on the legacy stream: synchronise so it cannot land
        // after work later queued on the handle's non-blocking stream
        cuda_check(cudaMemset(p, 0, n), "cudaMemset");
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        return p;
    }
};

struct StageInfo {
    int topo = 0;
    std::vector<int> removed;        // topology-local branch ids, sorted
    std::vector<int> removed_rated;  // their rated indices (sorted), rated only
    std::vector<int> removed_rowsz;
    int64_t pd_off = 0, cost_off = 0;
    double w = 1.0;
    std::vector<int> table;          // per tile: table index in the blob list
    // sizes
    int64_t n = 0, m_eq = 0, m_ineq = 0, nnz_jeq = 0, nnz_jin = 0, nnz_h = 0, hpg_local = 0;
    std::vector<int> tile_off;       // per tile 4 offsets (P, Q, VA, VM), stage-local
};
}  // namespace

struct acopf_topo {
    Topo t;
};

struct acopf_batch {
    int device = 0;
    std::vector<const Topo*> topos;
    std::vector<std::vector<int>> base_table;            // topo -> per tile -> table id
    std::vector<TileTable> tables;
    std::map<std::pair<int, std::pair<std::vector<int>, int>>, int> patch_cache;
    std::vector<StageInfo> stages;
    std::vector<double> pd, qd, ca, cb, cc;
    // layout
    bool laid_out = false, uploaded = false;
    std::vector<int32_t> obj_slot;
    std::vector<int64_t> off6;
    std::vector<int64_t> cp_row, cp_jpos, cp_a, cp_b;
    std::vector<int8_t> cp_first;
    int obj_mode = 0, n_obj = 0;
    // flat-buffer totals implied by the layout (set_layout): x rows, constraint
    // rows, J values, H values, objective slots
    int64_t tot_n = 0, tot_m = 0, tot_j = 0, tot_h = 0, tot_obj = 0;
    // device
    cudaStream_t stream = nullptr;
    DevBuf d_topo, d_stage, d_items, d_recs, d_aux, d_blob, d_pd, d_qd, d_ca, d_cb, d_cc, d_rem, d_remsz;
    DevBuf d_cpruns, d_objterms, d_xi, d_auxdone;
    int max_nb = 0;
    int n_gen_items = 0;             // aux items [0, n_gen_items) are generator chunks, the rest coupling runs
    std::vector<std::unique_ptr<DevBuf>> topo_bufs;
    EvalParams params{};
    size_t smem = 0, aux_smem = 0;
    int64_t launches = 0;
    // host staging for eval_host
    DevBuf h_x, h_m, h_obj, h_g, h_c, h_j, h_h;
    // stage-lane path for full evaluations (sl_kernel.cuh): SL tiles per base table
    // (topology, tile) (empty: a bus needs more term slots; that tile stays on the tile
    // kernel), groups of 32 stages, items, and the tile-kernel items of the rest
    bool sl_on = false;
    std::vector<std::vector<SLTile>> sl_tiles;     // index: topo * ntile_max + tile
    int sl_ntile_max = 0;
    SLParams slp{};
    size_t sl_smem = 0;
    int n_res_items = 0;
    DevBuf d_sl_groups, d_sl_items, d_sl_boff, d_sl_bytes, d_sl_runoff, d_sl_tileout, d_sl_blob, d_sl_x;
    DevBuf d_res_items, d_res_recs;

    // host-buffer pipeline (independent layouts): chunks of whole stage groups
    struct Pipe { int s0, s1, bus_first, bus_count, aux_first, aux_count; };
    std::vector<Pipe> pipe;
    int pipe_mode = 0;               // 1: independent stages ([eq; ineq] per stage); 2: composite
                                     // (stage blocks in order in every region, coupling rows after)
    std::vector<Pipe> il_chunks;     // device evaluation with interleaved inputs: chunks whose pre-pass
                                     // overlaps the previous chunk's tile kernel (two streams)
    cudaStream_t pipe_streams[3] = {nullptr, nullptr, nullptr};
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev_il = nullptr, ev_ilj[2] = {nullptr, nullptr};
    // CUDA graphs of single-stream host evaluations (acopf_batch_eval_host without the
    // chunked pipeline, on the library's stream, pinned host buffers): one per (what,
    // multipliers given, sizes, staging buffers); the host ends of its copies are patched
    // per call, so a batch-1 callback is one graph launch instead of 4-6 API calls
    struct HostGraph {
        uint32_t what = 0;
        bool mult = false;
        double obj_factor = 0.0;
        int64_t sz[7] = {};                       // x, mult, obj, grad, cons, jac, hess (doubles)
        const void* dev[7] = {};                  // the device staging buffers captured
        const void* host[7] = {};                 // host pointers the copies currently use
        cudaGraphNode_t node[7] = {};
        cudaMemcpy3DParms parm[7] = {};           // the captured copy parameters (host end patched)
        cudaGraph_t graph = nullptr;             // kept: its node handles address the exec's copies
        cudaGraphExec_t exec = nullptr;
        int64_t n_launches = 0;
    };
    std::vector<HostGraph> host_graphs;
    bool host_graphs_off = false;
    int host_graph_captures = 0;             // (a caller whose keys never repeat, e.g. a new
                                             // obj_factor per call, gets the plain path after 32)
    ~acopf_batch() {
        for (auto& g : host_graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        for (cudaEvent_t e : {ev_il, ev_ilj[0], ev_ilj[1]}) if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
        if (aux_stream) cudaStreamDestroy(aux_stream);
        for (auto& ps : pipe_streams) if (ps) cudaStreamDestroy(ps);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
    }
};

// ---------------------------------------------------------------------------
// Multi-GPU (one process per GPU): NCCL loaded at run time (dlopen), so the
// library has no link-time NCCL dependency and shares the process's NCCL
// (torch's) when one is already loaded.
struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);     // the process's NCCL (torch's) first
            if (!h) h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) { err = "libnccl.so.2 not found"; return; }
        api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
        api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
        api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
        api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy)
        throw std::runtime_error("NCCL unavailable: " + (err.empty() ? std::string("missing symbols") : err));
    return api;
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " +
                                 (nccl().GetErrorString ? nccl().GetErrorString(r) : std::to_string((int)r)));
}

// One rank's share of a sharded composite: its batch (its stages, composite
// layout with a halo, ACOPF_OBJ_TERMS) plus the exchange plan and buffers.
struct acopf_multi {
    acopf_batch* b = nullptr;
    int rank = 0, world = 1;
    ncclComm_t comm = nullptr;
    std::vector<int64_t> export_idx;         // local x indices this rank sends (sorted)
    std::vector<int64_t> halo_src;           // per halo value: position in the gathered buffer
    int64_t export_max = 1, halo_dst0 = 0;
    std::vector<int32_t> obj_counts;         // objective terms per rank (stage order)
    int obj_max = 1;
    DevBuf d_export, d_halo_src, d_send, d_recv, d_obj_send, d_obj_recv, d_counts;
    cudaStream_t halo_stream = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_halo = nullptr, ev_gen = nullptr;
    ~acopf_multi() {
        if (comm) nccl().CommDestroy(comm);
        if (halo_stream) cudaStreamDestroy(halo_stream);
        for (cudaEvent_t e : {ev_fork, ev_halo, ev_gen}) if (e) cudaEventDestroy(e);
    }
};

// Upload everything the kernels read and build the work lists.
static void upload(acopf_batch* b) {
    cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
    const int S = (int)b->stages.size();
    const int64_t n_coupling = (int64_t)b->cp_row.size();
    if (!b->stream) cuda_check(cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking), "stream");
    if (!b->aux_stream) cuda_check(cudaStreamCreateWithFlags(&b->aux_stream, cudaStreamNonBlocking), "stream");
    if (!b->ev_fork) cuda_check(cudaEventCreateWithFlags(&b->ev_fork, cudaEventDisableTiming), "event");
    if (!b->ev_join) cuda_check(cudaEventCreateWithFlags(&b->ev_join, cudaEventDisableTiming), "event");
    for (cudaEvent_t* e : {&b->ev_il, &b->ev_ilj[0], &b->ev_ilj[1]})
        if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");

    // topologies (only what the aux kernel needs; the bus kernel reads tile tables)
    std::vector<DTopo> dt;
    b->topo_bufs.clear();
    size_t max_leaf = 1, max_ng = 0;
    for (const Topo* T : b->topos) {
        max_ng = std::max<size_t>(max_ng, (size_t)T->ng);
        DTopo d{};
        d.nb = T->nb; d.nbr = T->nbr; d.ng = T->ng; d.nr = T->nr;
        std::vector<int> leaf;
        for (size_t l = 0; l < T->leaf_start.size(); ++l) { leaf.push_back(T->leaf_start[l]); leaf.push_back(T->leaf_len[l]); }
        b->topo_bufs.emplace_back(new DevBuf());
        d.leaf = b->topo_bufs.back()->upload(leaf);
        d.nleaf = (int)T->leaf_start.size();
        max_leaf = std::max(max_leaf, T->leaf_start.size());
        dt.push_back(d);
    }
    // blob of tile tables (each 16-byte aligned, sized for one bulk copy).  Each
    // staging segment is shifted by a free slot when needed so that its 16-byte
    // parity matches its output run's (first stage using the table; these
    // layouts keep every stage's CSR bases even), so the copy-out is a TMA
    // bulk store
    std::vector<uint8_t> blob;
    std::vector<int64_t> table_off(b->tables.size());
    std::vector<int> table_bytes(b->tables.size()), table_shift_n(b->tables.size(), 0);
    std::vector<int> table_mask(b->tables.size(), -1);
    for (int s = 0; s < S; ++s) {
        const StageInfo& st = b->stages[s];
        const int64_t* o = &b->off6[6 * s];
        for (size_t t = 0; t < st.table.size(); ++t) {
            int& m = table_mask[st.table[t]];
            if (m >= 0) continue;
            const TileTable& tt = b->tables[st.table[t]];
            const int Sst[4] = {0, tt.L[0], tt.L[0] + tt.L[1], tt.L[0] + tt.L[1] + tt.L[2]};
            m = 0;
            for (int q = 0, c = 0; q < 4; ++q) {
                const int64_t g = (q < 2 ? o[3] : o[5]) + st.tile_off[4 * t + q];
                const int sh = (int)((g - Sst[q] - c) & 1);
                m |= sh << q;
                c += sh;
            }
        }
    }
    for (size_t i = 0; i < b->tables.size(); ++i) {
        table_off[i] = (int64_t)blob.size();
        const unsigned m = table_mask[i] < 0 ? 0u : (unsigned)table_mask[i];
        b->tables[i].serialise(*b->topos[b->tables[i].topo], blob, m);
        table_bytes[i] = (int)(blob.size() - table_off[i]);
        table_shift_n[i] = __builtin_popcount(m);
    }
    // stages and removed lists
    std::vector<DStage> ds(S);
    std::vector<int> rem, remsz;
    long long fl_off = 0, inj_off = 0;
    for (int s = 0; s < S; ++s) {
        const StageInfo& st = b->stages[s];
        DStage& d = ds[s];
        const int64_t* o = &b->off6[6 * s];
        d.var_off = o[0]; d.eq_row = o[1]; d.ineq_row = o[2];
        d.jeq_base = o[3]; d.jineq_base = o[4]; d.h_base = o[5];
        d.hpg_local = st.hpg_local;
        d.pd_off = st.pd_off;
        d.cost_off = st.cost_off;
        d.rem_off = (long long)rem.size();
        d.nrem = (int)st.removed_rated.size();
        rem.insert(rem.end(), st.removed_rated.begin(), st.removed_rated.end());
        remsz.insert(remsz.end(), st.removed_rowsz.begin(), st.removed_rowsz.end());
        d.topo = st.topo;
        d.obj_slot = b->obj_slot[s];
        d.w = st.w;
        d.fl_off = fl_off; d.inj_off = inj_off;
        d.nb = b->topos[st.topo]->nb; d.ng = b->topos[st.topo]->ng; d.nbr = b->topos[st.topo]->nbr;
        fl_off += 4LL * b->topos[st.topo]->nbr;
        inj_off += 2LL * b->topos[st.topo]->nb;
    }
    // tile work: for every tile, the stages sharing one table, in groups of G consecutive
    // stages (G: the starting rule below, then the makespan model further down)
    int64_t total_recs = 0;
    for (const StageInfo& st : b->stages) total_recs += (int64_t)st.table.size();
    // stages per item: enough items to fill the GPU a few times over, and few
    // enough that the inputs (x, multipliers) of the stage groups in flight stay
    // L2-resident (ACOPF_L2_INPUT_MB per group; gathers otherwise re-read HBM)
    const char* wenv = getenv("ACOPF_ITEM_WAVES");     // development aid: items per resident CTA slot
    int n_sm = 148;                                     // B200; the device's own count when it is visible
    if (cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, b->device) != cudaSuccess || n_sm <= 0) {
        cudaGetLastError();
        n_sm = 148;
    }
    const int64_t target_items = (int64_t)n_sm * (WARP_MINB / TILE_WARPS) * (wenv ? std::max(1, atoi(wenv)) : 6);
    double in_bytes = 0.0;
    for (const StageInfo& st : b->stages) in_bytes += 8.0 * (double)(st.n + st.m_eq + st.m_ineq);
    const double per_stage = in_bytes / std::max(1, S);
    const char* l2env = getenv("ACOPF_L2_INPUT_MB");
    const double l2_budget = (l2env ? atof(l2env) : 32.0) * 1048576.0;
    const int64_t g_l2 = std::max<int64_t>(1, (int64_t)(l2_budget / std::max(1.0, per_stage)));
    const char* genv = getenv("ACOPF_MAX_G");          // development aid
    const int64_t g_max = genv ? std::max(1, atoi(genv)) : 64;
    // starting rule: about 6 items per resident CTA slot, at least two stages per item where
    // the L2 budget allows (one-stage items pay the table load per stage)
    int G = (int)std::max<int64_t>(std::min<int64_t>(2, g_l2),
                                   std::min<int64_t>({g_max, total_recs / target_items, g_l2}));
    size_t max_smem = 0;
    std::vector<std::pair<int, int>> tiles;       // (topo, tile)
    for (size_t ti = 0; ti < b->topos.size(); ++ti)
        for (size_t t = 0; t < b->base_table[ti].size(); ++t) tiles.push_back({(int)ti, (int)t});
    // resident tile CTAs per SM: the register budget's WARP_MINB / TILE_WARPS, fewer when the
    // largest table's shared memory (+1 KB reserved per CTA) does not fit that many
    size_t smem_all = 0;
    for (size_t i = 0; i < b->tables.size(); ++i)
        smem_all = std::max(smem_all, tile_smem_bytes(table_bytes[i], b->tables[i].nArea + table_shift_n[i]));
    const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(WARP_MINB / TILE_WARPS, 233472 / (int64_t)(smem_all + 1024 + 256)));
    const int64_t slots = (int64_t)n_sm * per_sm;
    // The run length G by a list-scheduling model of the block scheduler: items in launch
    // order (stage-group-major), each to the earliest-free CTA slot, an item costing its
    // stage count plus a fixed 0.3 stage (table load, first gathers); G minimises the
    // modelled makespan within the L2 cap (ties: the longer runs).  The model tracks the
    // measured cfg1 times over G = 7..50 (correlation 0.97): wave quantisation, not the
    // per-item cost alone, decides (cfg1 G = 20: +11%, G = 24: -3.5%); small workloads come
    // out as one wave of long items (cfg3: 10 stages, 430 items for 444 slots).
    {
        const char* me = getenv("ACOPF_G_MODEL");            // development aid: 0 = the rule above
        const bool model = me ? atoi(me) != 0 : true;
        const int g_hi = (int)std::max<int64_t>(1, std::min<int64_t>(g_max, g_l2));
        // items a run length makes (tile x group x distinct table)
        int64_t n_items_g = 0;
        auto makespan = [&](int g) {
            n_items_g = 0;
            std::priority_queue<double, std::vector<double>, std::greater<double>> free_at;
            for (int64_t k = 0; k < slots; ++k) free_at.push(0.0);
            double end = 0.0;
            std::vector<int> tb;
            for (int g0 = 0; g0 < S; g0 += g) {
                const int g1 = std::min(S, g0 + g);
                for (auto [topo, t] : tiles) {
                    tb.clear();
                    for (int s = g0; s < g1; ++s)
                        if (b->stages[s].topo == topo) tb.push_back(b->stages[s].table[t]);
                    std::sort(tb.begin(), tb.end());
                    for (size_t a = 0; a < tb.size();) {
                        size_t e = a;
                        while (e < tb.size() && tb[e] == tb[a]) ++e;
                        const double t0 = free_at.top() + (double)(e - a) + 0.3;
                        free_at.pop();
                        free_at.push(t0);
                        ++n_items_g;
                        end = std::max(end, t0);
                        a = e;
                    }
                }
            }
            return end;
        };
        if (model && total_recs > 0 && !tiles.empty()) {
            // candidates: every G up to the cap for small workloads, else around the rule's G
            // one wave of long items only for small workloads (<= 12 tile-stages per slot);
            // otherwise at least two items per slot, so the dynamic scheduling can absorb the
            // tiles' unequal stage times the model does not see (cfg1 G = 48/50: 1.4 waves, +4%)
            const bool small = total_recs <= 64 * slots, tiny = total_recs <= 12 * slots;
            const int lo = small ? 1 : std::max(1, G / 3), hi = small ? g_hi : std::min(g_hi, 4 * G);
            // (the rule's G stays unless the model predicts at least 1% less: cfg2 G = 13 was
            // modelled 0.6% faster and measured 0.3% slower)
            const int G_rule = G;
            const double rule = makespan(G_rule) * ((!tiny && n_items_g < 2 * slots) ? 1e9 : 1.0);
            double best = 1e300;
            int G_best = G_rule;
            for (int g = lo; g <= hi; ++g) {
                const double m = makespan(g);
                if (!tiny && n_items_g < 2 * slots) continue;
                if (m < best * 0.995 || (m <= best * 1.005 && g > G_best)) { best = m; G_best = g; }
            }
            if (best < rule * 0.99) G = G_best;
            else best = rule;
            if (getenv("ACOPF_DEBUG_PLAN"))
                fprintf(stderr, "plan: run length G = %d (modelled makespan %.1f stage-times, %lld slots)\n", G, best,
                        (long long)slots);
        }
    }
    if (const char* ge = getenv("ACOPF_G")) G = std::max(1, atoi(ge));      // development aid: exact G
    std::vector<int> table_area(b->tables.size());
    for (size_t i = 0; i < b->tables.size(); ++i) table_area[i] = b->tables[i].nArea + table_shift_n[i];
    // tile-kernel items over the (tile, stage) pairs `keep` accepts, stage-group-major
    // (warps running together share one group's x/mult in L2)
    auto build_items = [&](auto keep, std::vector<DBusItem>& items, std::vector<DRec>& recs) {
        std::map<int, std::vector<int>> by_table;     // table id -> stages (in order)
        for (int g0 = 0; g0 < S; g0 += G) {
            const int g1 = std::min(S, g0 + G);
            for (auto [topo, t] : tiles) {
                by_table.clear();
                for (int s = g0; s < g1; ++s)
                    if (b->stages[s].topo == topo && keep(t, s)) by_table[b->stages[s].table[t]].push_back(s);
                for (auto& kv : by_table) {
                    DBusItem it{};
                    it.blob_off = table_off[kv.first];
                    it.bytes = table_bytes[kv.first];
                    it.rec_off = (int)tile_rec_off(table_bytes[kv.first], table_area[kv.first]);
                    it.first = (int)recs.size();
                    it.count = (int)kv.second.size();
                    for (int s : kv.second) {
                        const StageInfo& st = b->stages[s];
                        const DStage& d = ds[s];
                        DRec r{};
                        r.var_off = d.var_off; r.eq_row = d.eq_row; r.ineq_row = d.ineq_row; r.pd_off = d.pd_off;
                        r.jineq = d.jineq_base;
                        r.oP = d.jeq_base + st.tile_off[4 * t + 0]; r.oQ = d.jeq_base + st.tile_off[4 * t + 1];
                        r.oA = d.h_base + st.tile_off[4 * t + 2]; r.oV = d.h_base + st.tile_off[4 * t + 3];
                        r.fl_off = d.fl_off; r.inj_off = d.inj_off; r.rem_off = d.rem_off;
                        r.w = d.w; r.nrem = d.nrem; r.nb = d.nb; r.ng = d.ng; r.nbr = d.nbr;
                        if (d.nrem > 0) { r.rr0 = st.removed_rated[0]; r.rz0 = st.removed_rowsz[0]; }
                        if (d.nrem > 1) { r.rr1 = st.removed_rated[1]; r.rz1 = st.removed_rowsz[1]; }
                        r.stage = s;
                        recs.push_back(r);
                    }
                    items.push_back(it);
                    max_smem = std::max(max_smem, tile_smem_bytes(table_bytes[kv.first], table_area[kv.first]));
                }
            }
        }
    };
    std::vector<DBusItem> items;
    std::vector<DRec> recs;
    build_items([](int, int) { return true; }, items, recs);
    // ---- stage-lane path (full evaluations) ----
    b->sl_on = false;
    b->n_res_items = 0;
    std::vector<DBusItem> res_items;
    std::vector<DRec> res_recs;
    {
        // ACOPF_SL=1 enables the stage-lane path (measured slower than the tile kernel on
        // every configuration so far; kept behind the switch with its tests)
        const char* sle = getenv("ACOPF_SL");
        if (sle && atoi(sle) != 0) {
            int ntmax = 0;
            for (size_t ti = 0; ti < b->topos.size(); ++ti) ntmax = std::max(ntmax, (int)b->base_table[ti].size());
            if (b->sl_tiles.empty() || b->sl_ntile_max != ntmax) {
                b->sl_ntile_max = ntmax;
                b->sl_tiles.assign(b->topos.size() * (size_t)ntmax, {});
                std::vector<std::pair<int, int>> jobs = tiles;
                std::atomic<size_t> next{0};
                auto work = [&] {
                    for (size_t j; (j = next.fetch_add(1)) < jobs.size();) {
                        const auto [topo, t] = jobs[j];
                        std::vector<SLTile> v;
                        if (!build_sl_tiles(*b->topos[topo], b->tables[b->base_table[topo][t]], t, v)) v.clear();
                        b->sl_tiles[(size_t)topo * ntmax + t] = std::move(v);
                    }
                };
                const int nt = (int)std::min<size_t>({(size_t)std::max(1u, std::thread::hardware_concurrency()),
                                                      (size_t)32, jobs.size()});
                std::vector<std::thread> pool;
                for (int i = 1; i < nt; ++i) pool.emplace_back(work);
                work();
                for (auto& th : pool) th.join();
            }
            // global SL tile list
            std::vector<int> first((size_t)b->topos.size() * ntmax, -1), count((size_t)b->topos.size() * ntmax, 0);
            std::vector<long long> boff;
            std::vector<int> bytes, runoff;
            std::vector<uint8_t> sblob;
            int table_max = 16, stride = 1;
            for (auto [topo, t] : tiles) {
                const auto& v = b->sl_tiles[(size_t)topo * ntmax + t];
                if (v.empty()) continue;
                first[(size_t)topo * ntmax + t] = (int)boff.size();
                count[(size_t)topo * ntmax + t] = (int)v.size();
                for (const SLTile& u : v) {
                    boff.push_back((long long)sblob.size());
                    bytes.push_back((int)u.blob.size());
                    sblob.insert(sblob.end(), u.blob.begin(), u.blob.end());
                    for (int q = 0; q < 4; ++q) runoff.push_back(u.off[q]);
                    table_max = std::max(table_max, (int)u.blob.size());
                    stride = std::max(stride, u.L[0] + u.L[1] + u.L[2] + u.L[3] + 4);
                }
            }
            table_max = (table_max + 127) & ~127;
            if (!(stride & 1)) ++stride;
            // groups: stages ordered by (topology, removed branches, index), runs of <= 32 of one topology
            std::vector<int> order(S);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int a, int c) {
                const StageInfo &x = b->stages[a], &y = b->stages[c];
                if (x.topo != y.topo) return x.topo < y.topo;
                return x.removed < y.removed;
            });
            std::vector<SLGroup> groups;
            long long xt = 0, mtt = 0, xg = 0;
            for (int i = 0; i < S;) {
                SLGroup G{};
                for (int l = 0; l < 32; ++l) G.stage[l] = -1;
                G.topo = b->stages[order[i]].topo;
                int l = 0;
                while (i < S && l < 32 && b->stages[order[i]].topo == G.topo) G.stage[l++] = order[i++];
                G.nlanes = l;
                const Topo& T = *b->topos[G.topo];
                G.xt_off = xt; G.mt_off = mtt; G.xg_off = xg;
                xt += 128LL * T.nb; mtt += 64LL * T.nr; xg += 64LL * T.ng;
                groups.push_back(G);
            }
            const int ng_ = (int)groups.size();
            std::vector<long long> tile_out((size_t)ng_ * ntmax * 128, -1);
            std::vector<SLItem> sitems;
            auto covered = [&](int t, int s) {
                const StageInfo& st = b->stages[s];
                return first[(size_t)st.topo * ntmax + t] >= 0 && st.table[t] == b->base_table[st.topo][t];
            };
            const int K = 4;                                  // SL tiles per warp item
            for (int g = 0; g < ng_; ++g) {
                const SLGroup& G = groups[g];
                for (int t = 0; t < (int)b->base_table[G.topo].size(); ++t) {
                    const int f = first[(size_t)G.topo * ntmax + t];
                    if (f < 0) continue;
                    bool any = false;
                    long long* to = &tile_out[((size_t)g * ntmax + t) * 128];
                    for (int l = 0; l < 32; ++l) {
                        const int s2 = G.stage[l];
                        if (s2 < 0 || !covered(t, s2)) continue;
                        any = true;
                        const StageInfo& st = b->stages[s2];
                        to[l] = ds[s2].jeq_base + st.tile_off[4 * t + 0];
                        to[32 + l] = ds[s2].jeq_base + st.tile_off[4 * t + 1];
                        to[64 + l] = ds[s2].h_base + st.tile_off[4 * t + 2];
                        to[96 + l] = ds[s2].h_base + st.tile_off[4 * t + 3];
                    }
                    if (!any) continue;
                    const int n = count[(size_t)G.topo * ntmax + t];
                    for (int u = 0; u < n; u += K) sitems.push_back(SLItem{g, t, f + u, f + std::min(n, u + K)});
                }
            }
            if (!sitems.empty()) {
                build_items([&](int t, int s2) { return !covered(t, s2); }, res_items, res_recs);
                SLParams& Q = b->slp;
                Q = SLParams{};
                Q.groups = b->d_sl_groups.upload(groups);
                Q.items = b->d_sl_items.upload(sitems);
                Q.sl_blob_off = b->d_sl_boff.upload(boff);
                Q.sl_bytes = b->d_sl_bytes.upload(bytes);
                Q.sl_run_off = b->d_sl_runoff.upload(runoff);
                Q.tile_out = b->d_sl_tileout.upload(tile_out);
                Q.blob = b->d_sl_blob.upload(sblob);
                Q.n_items = (int)sitems.size();
                Q.n_groups = ng_;
                Q.ntile_max = ntmax;
                Q.stride = stride;
                Q.table_max = table_max;
                double* xb = static_cast<double*>(b->d_sl_x.alloc(sizeof(double) * (size_t)(xt + mtt + xg + 1)));
                Q.xt = xb;
                Q.mt = xb + xt;
                Q.xg = xb + xt + mtt;
                b->sl_smem = 2 * (size_t)table_max + 32 * (size_t)stride * 8;
                if (b->sl_smem > (size_t)SMEM_LIMIT_BYTES) throw std::runtime_error("SL working set exceeds shared memory");
                cuda_check(cudaFuncSetAttribute(acopf_sl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)b->sl_smem), "cudaFuncSetAttribute(sl)");
                b->sl_on = true;
                b->n_res_items = (int)res_items.size();
                if (!res_items.empty()) {
                    b->d_res_items.upload(res_items);
                    b->d_res_recs.upload(res_recs);
                }
            }
        }
    }
    if (max_smem > (size_t)SMEM_LIMIT_BYTES) throw std::runtime_error("tile working set exceeds shared memory");
    // aux work: generator chunks per stage, then coupling chunks
    std::vector<DAuxItem> aux;
    std::vector<int> aux_first_of_stage(S + 1, 0);
    for (int s = 0; s < S; ++s) {
        const Topo& T = *b->topos[b->stages[s].topo];
        int nch = std::max(1, (T.ng + GEN_CHUNK - 1) / GEN_CHUNK);
        aux_first_of_stage[s] = (int)aux.size();
        for (int c = 0; c < nch; ++c) aux.push_back(DAuxItem{0, s, c, 0});
    }
    aux_first_of_stage[S] = (int)aux.size();
    b->n_gen_items = (int)aux.size();
    // pipeline chunks for host-buffer evaluation of independent layouts: about 8
    // chunks of whole stage groups (bus items are stage-group-major)
    b->pipe.clear();
    // the chunked copies move [off6(s0), off6(s1)) ranges: only valid when every
    // stage's blocks are contiguous and in stage order ([eq; ineq] rows, [Jeq; Jineq]
    // values, x, H values, objective slot s)
    bool contiguous = true, composite = S >= 2;
    for (int s = 0; s < S && contiguous; ++s) {
        const StageInfo& st = b->stages[s];
        const int64_t* o = &b->off6[6 * s];
        const int64_t nx[6] = {o[0] + st.n, o[2] + st.m_ineq, 0, o[4] + st.nnz_jin, 0, o[5] + st.nnz_h};
        contiguous = b->obj_slot[s] == s && o[1] + st.m_eq == o[2] && o[3] + st.nnz_jeq == o[4];
        if (s == 0) contiguous = contiguous && o[0] == 0 && o[1] == 0 && o[3] == 0 && o[5] == 0;
        if (s + 1 < S) {
            const int64_t* q = &b->off6[6 * (s + 1)];
            contiguous = contiguous && q[0] == nx[0] && q[1] == nx[1] && q[3] == nx[3] && q[5] == nx[5];
        }
    }
    // composite layouts: every region (x, eq rows, ineq rows, J eq, J ineq, H) holds the stage
    // blocks in stage order; coupling rows / J entries lie outside them
    for (int s = 0; s + 1 < S && composite; ++s) {
        const StageInfo& st = b->stages[s];
        const int64_t *o = &b->off6[6 * s], *q = &b->off6[6 * (s + 1)];
        composite = q[0] == o[0] + st.n && q[1] == o[1] + st.m_eq && q[2] == o[2] + st.m_ineq &&
                    q[3] == o[3] + st.nnz_jeq && q[4] == o[4] + st.nnz_jin && q[5] == o[5] + st.nnz_h &&
                    b->obj_slot[s] == s && b->obj_slot[s + 1] == s + 1;
    }
    composite = composite && b->obj_mode != 0 && !contiguous;
    {   // small composites gain nothing from chunked copies (cfg3, 73 MB of outputs: -5%)
        double out_bytes = 0.0;
        for (const StageInfo& st : b->stages) out_bytes += 8.0 * (st.n + st.m_eq + st.m_ineq + st.nnz_jeq + st.nnz_jin + st.nnz_h);
        composite = composite && out_bytes > 256.0 * 1048576.0;
    }
    b->pipe_mode = 0;
    if ((b->obj_mode == 0 && n_coupling == 0 && S >= 2 && contiguous) || composite) {
        b->pipe_mode = composite ? 2 : 1;
        const int ngroups = (S + G - 1) / G;
        const int nchunks = getenv("ACOPF_PIPE_CHUNKS") ? std::max(1, atoi(getenv("ACOPF_PIPE_CHUNKS"))) : 8;   // development aid
        const int per = std::max(1, (ngroups + nchunks - 1) / nchunks);
        int item = 0;
        for (int g0 = 0; g0 < ngroups; g0 += per) {
            acopf_batch::Pipe pc{};
            pc.s0 = g0 * G;
            pc.s1 = std::min(S, (g0 + per) * G);
            pc.bus_first = item;
            while (item < (int)items.size() && recs[items[item].first].stage < pc.s1) ++item;
            pc.bus_count = item - pc.bus_first;
            pc.aux_first = aux_first_of_stage[pc.s0];
            pc.aux_count = aux_first_of_stage[pc.s1] - pc.aux_first;
            b->pipe.push_back(pc);
        }
        for (auto& ps : b->pipe_streams)
            if (!ps) cuda_check(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking), "stream");
    }
    // interleave overlap: when the interleaved inputs exceed L2 (cfg4: 0.8 GB), the
    // pre-pass of stage chunk c + 1 runs beside the tile kernel of chunk c
    b->il_chunks.clear();
    {
        int64_t il_bytes = 0;
        int nbmax = 0;
        for (const StageInfo& st : b->stages) nbmax = std::max(nbmax, b->topos[st.topo]->nb);
        for (const StageInfo& st : b->stages) il_bytes += 32LL * b->topos[st.topo]->nb;
        const char* ie = getenv("ACOPF_INTERLEAVE");
        const bool il = ie ? atoi(ie) != 0 : nbmax >= INTERLEAVE_MIN_BUSES;
        const char* ce = getenv("ACOPF_IL_CHUNKS");                // development aid
        const int nch = ce ? std::max(1, atoi(ce)) : 1;   // measured no gain: off by default
        if (il && (il_bytes > 256LL * 1048576 || ce) && nch > 1) {
            const int ngroups = (S + G - 1) / G;
            const int per = std::max(1, (ngroups + nch - 1) / nch);
            int item = 0;
            for (int g0 = 0; g0 < ngroups; g0 += per) {
                acopf_batch::Pipe pc{};
                pc.s0 = g0 * G;
                pc.s1 = std::min(S, (g0 + per) * G);
                pc.bus_first = item;
                while (item < (int)items.size() && recs[items[item].first].stage < pc.s1) ++item;
                pc.bus_count = item - pc.bus_first;
                b->il_chunks.push_back(pc);
            }
            if (item != (int)items.size()) b->il_chunks.clear();      // items not stage-group-major: no chunks
            for (auto& ps : b->pipe_streams)
                if (!ps) cuda_check(cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking), "stream");
        }
    }
    // coupling rows as runs (row, J position, child and base columns advancing
    // together), packed into items of at most CP_CHUNK rows
    std::vector<DCpRun> runs;
    for (int64_t i = 0; i < n_coupling; ++i) {
        if (!runs.empty()) {
            DCpRun& R = runs.back();
            if (R.n < CP_CHUNK && b->cp_row[i] == R.row0 + R.n && b->cp_jpos[i] == R.jpos0 + 2 * R.n &&
                b->cp_a[i] == R.a0 + R.n && b->cp_b[i] == R.b0 + R.n && (int)b->cp_first[i] == R.base_first) {
                R.n++;
                continue;
            }
        }
        runs.push_back(DCpRun{b->cp_row[i], b->cp_jpos[i], b->cp_a[i], b->cp_b[i], 1, (int)b->cp_first[i]});
    }
    for (size_t r = 0; r < runs.size();) {
        size_t e = r;
        int rows = 0;
        while (e < runs.size() && (e == r || rows + runs[e].n <= CP_CHUNK)) rows += runs[e++].n;
        aux.push_back(DAuxItem{1, (int)r, (int)(e - r), 0});
        r = e;
    }
    b->n_obj = S;

    EvalParams& P = b->params;
    P = EvalParams{};
    P.topos = b->d_topo.upload(dt);
    P.stages = b->d_stage.upload(ds);
    P.bus_items = b->d_items.upload(items);
    P.bus_recs = b->d_recs.upload(recs);
    P.aux_items = b->d_aux.upload(aux);
    P.blob = b->d_blob.upload(blob);
    P.pd = b->d_pd.upload(b->pd);
    P.qd = b->d_qd.upload(b->qd);
    P.ca = b->d_ca.upload(b->ca);
    P.cb = b->d_cb.upload(b->cb);
    P.cc = b->d_cc.upload(b->cc);
    P.rem_ridx = b->d_rem.upload(rem);
    P.rem_rowsz = b->d_remsz.upload(remsz);
    P.cp_runs = b->d_cpruns.upload(runs);
    P.n_bus_items = (int)items.size();
    P.n_aux_items = (int)aux.size();
    P.n_obj = S;
    P.obj_mode = b->obj_mode;
    P.obj_terms = static_cast<double*>(b->d_objterms.alloc(sizeof(double) * std::max(S, 1)));
    P.aux_done = static_cast<unsigned*>(b->d_auxdone.alloc(sizeof(unsigned)));
    // interleaved (VA, VM, muP, muQ) per stage and bus, indexed 4 (var_off + bus)
    {
        int64_t xi_len = 4;
        b->max_nb = 0;
        for (const DStage& d : ds) {
            xi_len = std::max<int64_t>(xi_len, 4 * (d.var_off + d.nb));
            b->max_nb = std::max(b->max_nb, d.nb);
        }
        // networks whose per-stage inputs (32 B per bus) exceed what L1 keeps
        // resident; ACOPF_INTERLEAVE=0/1 overrides (development aid)
        const char* ie = getenv("ACOPF_INTERLEAVE");
        const bool use = ie ? atoi(ie) != 0 : b->max_nb >= INTERLEAVE_MIN_BUSES;
        P.xi = use ? static_cast<double*>(b->d_xi.alloc(sizeof(double) * (size_t)xi_len)) : nullptr;
    }
    b->smem = (max_smem + 15) & ~size_t(15);
    // development aid: extra shared memory per CTA (lowers the resident CTAs per SM)
    if (const char* e = getenv("ACOPF_SMEM_PAD_KB")) b->smem += 1024 * (size_t)atoi(e);
    // objective blocks stage their stage's cost terms when they fit (64 KB)
    // (up to 16 KB: larger aux blocks crowd the tile kernel's CTAs off the SMs;
    // a full carve-out preference for both kernels costs the tile kernel its L1)
    const char* se = getenv("ACOPF_OBJ_STAGE_KB");          // development aid
    P.obj_staged = sizeof(double) * (9 * max_leaf + max_ng) <= 1024 * (size_t)(se ? atoi(se) : 16) ? 1 : 0;
    b->aux_smem = sizeof(double) * (9 * max_leaf + (P.obj_staged ? max_ng : 0));
    // the dynamic shared-memory limits only grow (per device): every live batch
    // keeps launching with its own size
    {
        static std::mutex mu;
        static std::map<int, std::pair<size_t, size_t>> limit;     // device -> (tile, aux)
        std::lock_guard<std::mutex> lock(mu);
        auto& lim = limit[b->device];
        if (b->smem > lim.first) {
            for (auto fn : {acopf_tile_kernel<0u>, acopf_tile_kernel<ACOPF_ALL>})
                cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b->smem),
                           "cudaFuncSetAttribute(tile)");
            lim.first = b->smem;
        }
        if (b->aux_smem > lim.second) {          // (the kernel also has static shared memory)
            cuda_check(cudaFuncSetAttribute(acopf_aux_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)b->aux_smem), "cudaFuncSetAttribute(aux)");
            lim.second = b->aux_smem;
        }
    }
    b->uploaded = true;
}

extern "C" {

const char* acopf_last_error(void) { return g_err.c_str(); }
int acopf_version(void) { return 1; }

int acopf_topo_create(int32_t nb, int32_t nbr, int32_t ng, const int32_t* fo, const int32_t* to,
                      const double* adm, const uint8_t* rated, const int32_t* gbus, const double* gs,
                      const double* bs, acopf_topo** out) {
    return guard([&] {
        if (nb < 0 || nbr < 0 || ng < 0) throw std::runtime_error("negative size");
        auto* h = new acopf_topo();
        Topo& T = h->t;
        T.nb = nb; T.nbr = nbr; T.ng = ng;
        T.fo.assign(fo, fo + nbr);
        T.to.assign(to, to + nbr);
        T.adm.assign(adm, adm + 8 * (size_t)nbr);
        T.ridx.assign(nbr, -1);
        int r = 0;
        for (int k = 0; k < nbr; ++k) {
            if (fo[k] < 0 || fo[k] >= nb || to[k] < 0 || to[k] >= nb) { delete h; throw std::runtime_error("branch bus slot out of range"); }
            if (rated[k]) T.ridx[k] = r++;
        }
        T.gbus.assign(gbus, gbus + ng);
        for (int g = 0; g < ng; ++g)
            if (gbus[g] < 0 || gbus[g] >= nb) { delete h; throw std::runtime_error("generator bus slot out of range"); }
        T.gs.assign(gs, gs + nb);
        T.bs.assign(bs, bs + nb);
        T.finalize();
        *out = h;
    });
}

int acopf_topo_destroy(acopf_topo* t) {
    delete t;
    return 0;
}

// Build tile tables in parallel: out[i] = build_tile(*topo[i], tile[i], live[i]).
struct TableTask { const Topo* topo; int topo_id, tile; const std::vector<int>* removed; };
static void build_tables(const std::vector<TableTask>& tasks, std::vector<TileTable>& tables, size_t first) {
    if (tasks.empty()) return;
    tables.resize(first + tasks.size());
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = (int)std::min<size_t>({(size_t)hw, (size_t)32, tasks.size()});
    std::atomic<size_t> next{0};
    std::string err;
    std::mutex mu;
    auto work = [&] {
        for (size_t i; (i = next.fetch_add(1)) < tasks.size();) {
            const TableTask& k = tasks[i];
            try {
                tables[first + i] = build_tile(*k.topo, k.tile, Live{k.removed});
                tables[first + i].topo = k.topo_id;
            } catch (const std::exception& e) {
                std::lock_guard<std::mutex> lock(mu);
                if (err.empty()) err = e.what();
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (!err.empty()) throw std::runtime_error(err);
}

int acopf_batch_create(int32_t device, int32_t n_topos, acopf_topo* const* topos, int32_t n_stages,
                       const int32_t* stage_topo, const int64_t* removed_ptr, const int32_t* removed_idx,
                       const int32_t* stage_load, const int64_t* load_off, int64_t n_load_values,
                       const double* pd, const double* qd, const int32_t* stage_cost,
                       const int64_t* cost_off, int64_t n_cost_values, const double* ca, const double* cb,
                       const double* cc, const double* weight, acopf_batch** out) {
    return guard([&] {
        std::unique_ptr<acopf_batch> B(new acopf_batch());
        B->device = device;
        for (int i = 0; i < n_topos; ++i) B->topos.push_back(&topos[i]->t);
        // base tile tables (built in parallel)
        {
            std::vector<TableTask> tasks;
            for (int i = 0; i < n_topos; ++i) {
                const Topo& T = *B->topos[i];
                std::vector<int> ids;
                for (size_t t = 0; t + 1 < T.tile_b0.size(); ++t) {
                    ids.push_back((int)tasks.size());
                    tasks.push_back(TableTask{&T, i, (int)t, nullptr});
                }
                B->base_table.push_back(ids);
            }
            build_tables(tasks, B->tables, 0);
        }
        for (int i = 0; i < n_topos; ++i) {
            const Topo& T = *B->topos[i];
            const std::vector<int>& ids = B->base_table[i];
            if (getenv("ACOPF_DEBUG_PLAN")) {     // planner statistics (development aid)
                size_t tb = 0, ar = 0, mx = 0, ends = 0, terms = 0, slots = 0;
                for (int id : ids) {
                    std::vector<uint8_t> blob;
                    const TileTable& tt = B->tables[id];
                    tt.serialise(T, blob);
                    tb += blob.size();
                    ar += 8 * (size_t)tt.nArea;
                    mx = std::max(mx, tile_smem_bytes((int)blob.size(), tt.nArea));
                    ends += tt.ends.size();
                    for (size_t r = 0; r < tt.sround.size() / 2; ++r) slots += 32 * (size_t)tt.sround[2 * r + 1];
                    terms += tt.nega.size();
                }
                std::vector<size_t> sm;
                for (int id : ids) {
                    std::vector<uint8_t> blob;
                    B->tables[id].serialise(T, blob);
                    sm.push_back(tile_smem_bytes((int)blob.size(), B->tables[id].nArea));
                }
                std::sort(sm.begin(), sm.end());
                fprintf(stderr, "plan: smem p50 %zu p90 %zu p99 %zu max %zu\n", sm[sm.size() / 2], sm[sm.size() * 9 / 10],
                        sm[sm.size() * 99 / 100], sm.back());
                fprintf(stderr, "plan: topo %d: %zu tiles, %.1f ends/tile, table %.0f B, area %.0f B, max smem %zu, "
                        "sum-round slots %.0f, -0.0 pads %.0f per tile\n", i, ids.size(), (double)ends / ids.size(),
                        (double)tb / ids.size(), (double)ar / ids.size(), mx, (double)slots / ids.size(),
                        (double)terms / ids.size());
            }
        }
        B->pd.assign(pd, pd + n_load_values);
        B->qd.assign(qd, qd + n_load_values);
        B->ca.assign(ca, ca + n_cost_values);
        B->cb.assign(cb, cb + n_cost_values);
        B->cc.assign(cc, cc + n_cost_values);
        B->stages.resize(n_stages);
        std::vector<TableTask> patch_tasks;             // patched tables, built in parallel below
        const size_t patch_first = B->tables.size();
        for (int s = 0; s < n_stages; ++s) {
            StageInfo& S = B->stages[s];
            S.topo = stage_topo[s];
            if (S.topo < 0 || S.topo >= n_topos) throw std::runtime_error("stage topology index out of range");
            const Topo& T = *B->topos[S.topo];
            S.removed.assign(removed_idx + removed_ptr[s], removed_idx + removed_ptr[s + 1]);
            std::sort(S.removed.begin(), S.removed.end());
            S.removed.erase(std::unique(S.removed.begin(), S.removed.end()), S.removed.end());
            S.pd_off = load_off[stage_load[s]];
            S.cost_off = cost_off[stage_cost[s]];
            S.w = weight[s];
            if (S.pd_off < 0 || S.pd_off + T.nb > n_load_values) throw std::runtime_error("load set out of range");
            if (S.cost_off < 0 || S.cost_off + T.ng > n_cost_values) throw std::runtime_error("cost set out of range");
            // tables: base unless the tile holds an endpoint of a removed branch
            S.table = B->base_table[S.topo];
            std::vector<int> touched;
            for (int k : S.removed) {
                if (k < 0 || k >= T.nbr) throw std::runtime_error("removed branch out of range");
                if (T.ridx[k] >= 0) {
                    S.removed_rated.push_back(T.ridx[k]);
                    S.removed_rowsz.push_back(T.rowsz[T.ridx[k]]);
                }
                for (int bus : {T.fo[k], T.to[k]}) {
                    int t = int(std::upper_bound(T.tile_b0.begin(), T.tile_b0.end(), bus) - T.tile_b0.begin()) - 1;
                    touched.push_back(t);
                }
            }
            {   // keep rated lists sorted together
                std::vector<int> order(S.removed_rated.size());
                std::iota(order.begin(), order.end(), 0);
                std::sort(order.begin(), order.end(), [&](int a, int b) { return S.removed_rated[a] < S.removed_rated[b]; });
                std::vector<int> rr, rz;
                for (int o : order) { rr.push_back(S.removed_rated[o]); rz.push_back(S.removed_rowsz[o]); }
                S.removed_rated = rr;
                S.removed_rowsz = rz;
            }
            std::sort(touched.begin(), touched.end());
            touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
            for (int t : touched) {
                auto key = std::make_pair(S.topo, std::make_pair(S.removed, t));
                auto it = B->patch_cache.find(key);
                if (it == B->patch_cache.end()) {
                    it = B->patch_cache.emplace(key, (int)(patch_first + patch_tasks.size())).first;
                    patch_tasks.push_back(TableTask{&T, S.topo, t, &S.removed});
                }
                S.table[t] = it->second;
            }
        }
        build_tables(patch_tasks, B->tables, patch_first);
        for (int s = 0; s < n_stages; ++s) {
            StageInfo& S = B->stages[s];
            const Topo& T = *B->topos[S.topo];
            // sizes and stage-local segment offsets
            const int ntile = (int)S.table.size();
            int64_t LP = 0, LQ = 0, LA = 0, LV = 0;
            for (int t = 0; t < ntile; ++t) {
                const TileTable& tt = B->tables[S.table[t]];
                LP += tt.L[0]; LQ += tt.L[1]; LA += tt.L[2]; LV += tt.L[3];
            }
            S.tile_off.assign(4 * ntile, 0);
            int64_t aP = 0, aQ = LP, aA = 0, aV = LA;
            for (int t = 0; t < ntile; ++t) {
                const TileTable& tt = B->tables[S.table[t]];
                S.tile_off[4 * t + 0] = (int)aP; aP += tt.L[0];
                S.tile_off[4 * t + 1] = (int)aQ; aQ += tt.L[1];
                S.tile_off[4 * t + 2] = (int)aA; aA += tt.L[2];
                S.tile_off[4 * t + 3] = (int)aV; aV += tt.L[3];
            }
            int64_t ineq = 0;
            for (int r = 0; r < T.nr; ++r) ineq += T.rowsz[r];
            for (int z : S.removed_rowsz) ineq -= z;
            S.n = 2LL * T.nb + 2LL * T.ng;
            S.m_eq = 2LL * T.nb;
            S.m_ineq = 2LL * (T.nr - (int64_t)S.removed_rated.size());
            S.nnz_jeq = LP + LQ;
            S.nnz_jin = ineq;
            S.hpg_local = LA + LV;
            S.nnz_h = LA + LV + T.ng;
            if (S.nnz_jeq + S.nnz_jin >= (1LL << 31) || S.nnz_h >= (1LL << 31))
                throw std::runtime_error("stage too large for 32-bit offsets");
        }
        *out = B.release();
    });
}

int acopf_batch_destroy(acopf_batch* b) {
    if (b) {
        cudaSetDevice(b->device);
        delete b;
    }
    return 0;
}

int acopf_batch_stage_sizes(const acopf_batch* b, int64_t* out6) {
    return guard([&] {
        for (size_t s = 0; s < b->stages.size(); ++s) {
            const StageInfo& S = b->stages[s];
            int64_t* o = out6 + 6 * s;
            o[0] = S.n; o[1] = S.m_eq; o[2] = S.m_ineq; o[3] = S.nnz_jeq; o[4] = S.nnz_jin; o[5] = S.nnz_h;
        }
    });
}


int acopf_batch_set_layout(acopf_batch* b, const int64_t* offsets6, int32_t obj_mode, const int32_t* obj_slot,
                           int64_t n_coupling, const int64_t* cp_row, const int64_t* cp_jpos, const int64_t* cp_a,
                           const int64_t* cp_b, const int8_t* cp_base_first) {
    return guard([&] {
        if (obj_mode < 0 || obj_mode > 2) throw std::runtime_error("bad objective mode");
        const int S = (int)b->stages.size();
        b->off6.assign(offsets6, offsets6 + 6 * (size_t)S);
        b->obj_slot.assign(obj_slot, obj_slot + S);
        b->cp_row.assign(cp_row, cp_row + n_coupling);
        b->cp_jpos.assign(cp_jpos, cp_jpos + n_coupling);
        b->cp_a.assign(cp_a, cp_a + n_coupling);
        b->cp_b.assign(cp_b, cp_b + n_coupling);
        b->cp_first.assign(cp_base_first, cp_base_first + n_coupling);
        b->obj_mode = obj_mode;
        int64_t tn = 0, tm = 0, tj = 0, th = 0, to = obj_mode == 1 ? 1 : 0;
        for (int s = 0; s < S; ++s) {
            const StageInfo& st = b->stages[s];
            const int64_t* o = &b->off6[6 * s];
            if (o[0] < 0 || o[1] < 0 || o[2] < 0 || o[3] < 0 || o[4] < 0 || o[5] < 0)
                throw std::runtime_error("negative layout offset");
            tn = std::max(tn, o[0] + st.n);
            tm = std::max({tm, o[1] + st.m_eq, o[2] + st.m_ineq});
            tj = std::max({tj, o[3] + st.nnz_jeq, o[4] + st.nnz_jin});
            th = std::max(th, o[5] + st.nnz_h);
            if (obj_mode != 1) {
                if (obj_slot[s] < 0) throw std::runtime_error("negative objective slot");
                to = std::max<int64_t>(to, (int64_t)obj_slot[s] + 1);
            }
        }
        for (int64_t c = 0; c < n_coupling; ++c) {
            if (cp_row[c] < 0 || cp_jpos[c] < 0 || cp_a[c] < 0 || cp_b[c] < 0)
                throw std::runtime_error("negative coupling index");
            tm = std::max(tm, cp_row[c] + 1);
            tj = std::max(tj, cp_jpos[c] + 2);
            tn = std::max({tn, cp_a[c] + 1, cp_b[c] + 1});
        }
        b->tot_n = tn; b->tot_m = tm; b->tot_j = tj; b->tot_h = th; b->tot_obj = to;
        b->laid_out = true;
        b->uploaded = false;
        for (auto& g : b->host_graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            if (g.graph) cudaGraphDestroy(g.graph);
        }
        b->host_graphs.clear();
    });
}

// The tile kernel's bus inputs for stages [s0, s1): acopf_interleave_kernel on st.
static void launch_interleave(acopf_batch* b, const EvalParams& P, int s0, int s1, cudaStream_t st) {
    if (!P.xi) return;
    for (int a = s0; a < s1; a += 65535) {
        const dim3 grid((unsigned)std::max(1, (b->max_nb + BLOCK * IL_BUSES - 1) / (BLOCK * IL_BUSES)),
                        (unsigned)std::min(65535, s1 - a));
        acopf_interleave_kernel<<<grid, BLOCK, 0, st>>>(P, a);
        cuda_check(cudaGetLastError(), "acopf_interleave_kernel launch");
        b->launches++;
    }
}

// The bus-side work of one evaluation on st: for full evaluations with the
// stage-lane path, the transposition pre-pass, the SL kernel and the tile kernel
// for the (tile, stage) pairs SL does not cover; else the interleave pre-pass
// (large networks) and the tile kernel over every item.
static void launch_bus_work(acopf_batch* b, const EvalParams& P, cudaStream_t st) {
    if (P.what == ACOPF_ALL && b->sl_on) {
        const SLParams& Q = b->slp;
        acopf_sl_transpose_kernel<<<dim3(64, (unsigned)Q.n_groups), 256, 0, st>>>(P, Q);
        cuda_check(cudaGetLastError(), "acopf_sl_transpose_kernel launch");
        acopf_sl_kernel<<<Q.n_items, 32, b->sl_smem, st>>>(P, Q);
        cuda_check(cudaGetLastError(), "acopf_sl_kernel launch");
        b->launches += 2;
        if (b->n_res_items > 0) {
            EvalParams R = P;
            R.bus_items = static_cast<const DBusItem*>(b->d_res_items.p);
            R.bus_recs = static_cast<const DRec*>(b->d_res_recs.p);
            R.n_bus_items = b->n_res_items;
            R.xi = nullptr;                   // direct gathers for the few leftover pairs
            acopf_tile_kernel<ACOPF_ALL><<<R.n_bus_items, TILE_THREADS, b->smem, st>>>(R, 0);
            cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
            b->launches++;
        }
        return;
    }
    if (P.xi && b->il_chunks.size() > 1) {
        // chunk c on stream c % 2: its interleave pre-pass, then its tile kernel; the
        // pre-pass of chunk c + 1 (HBM streaming) overlaps chunk c's tile kernel (L1-bound)
        cuda_check(cudaEventRecord(b->ev_il, st), "event record");
        for (int k = 0; k < 2; ++k) cuda_check(cudaStreamWaitEvent(b->pipe_streams[k], b->ev_il, 0), "stream wait");
        for (size_t c = 0; c < b->il_chunks.size(); ++c) {
            const auto& pc = b->il_chunks[c];
            cudaStream_t cs = b->pipe_streams[c & 1];
            launch_interleave(b, P, pc.s0, pc.s1, cs);
            if (pc.bus_count == 0) continue;
            if (P.what == ACOPF_ALL)
                acopf_tile_kernel<ACOPF_ALL><<<pc.bus_count, TILE_THREADS, b->smem, cs>>>(P, pc.bus_first);
            else acopf_tile_kernel<0u><<<pc.bus_count, TILE_THREADS, b->smem, cs>>>(P, pc.bus_first);
            cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
            b->launches++;
        }
        for (int k = 0; k < 2; ++k) {
            cuda_check(cudaEventRecord(b->ev_ilj[k], b->pipe_streams[k]), "event record");
            cuda_check(cudaStreamWaitEvent(st, b->ev_ilj[k], 0), "stream wait");
        }
        return;
    }
    launch_interleave(b, P, 0, (int)b->stages.size(), st);
    if (P.what == ACOPF_ALL) acopf_tile_kernel<ACOPF_ALL><<<P.n_bus_items, TILE_THREADS, b->smem, st>>>(P, 0);
    else acopf_tile_kernel<0u><<<P.n_bus_items, TILE_THREADS, b->smem, st>>>(P, 0);
    cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
    b->launches++;
}

int acopf_batch_eval(acopf_batch* b, const double* x, double obj_factor, const double* mult, uint32_t what,
                     double* obj, double* grad, double* cons, double* jval, double* hval, void* stream) {
    return guard([&] {
        if (!b->laid_out) throw std::runtime_error("acopf_batch_set_layout was not called");
        if (!b->uploaded) upload(b);
        if ((what & (ACOPF_CONS | ACOPF_JAC | ACOPF_HESS | ACOPF_GRAD)) && !x) throw std::runtime_error("x is NULL");
        if ((what & ACOPF_OBJ) && (!obj || !x)) throw std::runtime_error("obj/x is NULL");
        if ((what & ACOPF_GRAD) && !grad) throw std::runtime_error("grad is NULL");
        if ((what & ACOPF_CONS) && !cons) throw std::runtime_error("cons is NULL");
        if ((what & ACOPF_JAC) && !jval) throw std::runtime_error("jval is NULL");
        if ((what & ACOPF_HESS) && (!hval || !mult)) throw std::runtime_error("hval/mult is NULL");
        cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
        EvalParams P = b->params;
        P.x = x; P.mult = mult; P.obj_factor = obj_factor; P.what = what;
        P.obj = obj; P.grad = grad; P.cons = cons; P.jval = jval; P.hval = hval;
        // NULL = the legacy default stream (CUDA's convention, and torch's default stream)
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const bool bus = (what & (ACOPF_CONS | ACOPF_JAC | ACOPF_HESS)) && P.n_bus_items > 0;
        static const bool no_aux = getenv("ACOPF_EXP_NO_AUX") != nullptr;   // development aid: tile kernel alone
        const bool aux = !no_aux && (what & (ACOPF_OBJ | ACOPF_GRAD | ACOPF_HESS | ACOPF_CONS | ACOPF_JAC)) && P.n_aux_items > 0;
        // the generator/coupling items run as the last blocks of the tile kernel's own grid (one
        // launch, no fork / join) when they are a small share of it: measured cfg3 -5%; with
        // many aux items (cfg1/2/4) their 128-thread blocks in the tail cost 2-4% instead
        const char* fe = getenv("ACOPF_FUSED_AUX");      // 0 / 1 force it (development aid)
        const bool fuse_ok = fe ? atoi(fe) != 0 : (int64_t)P.n_aux_items * 100 <= (int64_t)P.n_bus_items * 15;
        if (fuse_ok && aux && bus && !(what == ACOPF_ALL && b->sl_on) && !(P.xi && b->il_chunks.size() > 1)) {
            P.aux_in_tile = 1;
            P.n_bus_launch = P.n_bus_items;
            launch_interleave(b, P, 0, (int)b->stages.size(), st);
            const int grid = P.n_bus_items + P.n_aux_items;
            if (what == ACOPF_ALL) acopf_tile_kernel<ACOPF_ALL><<<grid, TILE_THREADS, b->smem, st>>>(P, 0);
            else acopf_tile_kernel<0u><<<grid, TILE_THREADS, b->smem, st>>>(P, 0);
            cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
            b->launches++;
            return;
        }
        // the generator/coupling kernel runs concurrently on a forked stream
        const bool fork = aux && bus;
        if (fork) {
            cuda_check(cudaEventRecord(b->ev_fork, st), "event record");
            cuda_check(cudaStreamWaitEvent(b->aux_stream, b->ev_fork, 0), "stream wait");
        }
        if (aux) {
            acopf_aux_kernel<<<P.n_aux_items, BLOCK, b->aux_smem, fork ? b->aux_stream : st>>>(P, 0);
            cuda_check(cudaGetLastError(), ("acopf_aux_kernel launch (" + std::to_string(b->aux_smem) + " B shared)").c_str());
            b->launches++;
            if (P.obj_mode == 1 && (what & ACOPF_OBJ)) {
                acopf_objsum_kernel<<<1, BLOCK, 0, fork ? b->aux_stream : st>>>(P);
                cuda_check(cudaGetLastError(), "acopf_objsum_kernel launch");
                b->launches++;
            }
        }
        if (bus) launch_bus_work(b, P, st);
        if (fork) {
            cuda_check(cudaEventRecord(b->ev_join, b->aux_stream), "event record");
            cuda_check(cudaStreamWaitEvent(st, b->ev_join, 0), "stream wait");
        }
    });
}

int acopf_batch_flows(acopf_batch* b, const double* x, double* flows, double* inj, void* stream) {
    return guard([&] {
        if (!b->laid_out) throw std::runtime_error("acopf_batch_set_layout was not called");
        if (!b->uploaded) upload(b);
        if (!x || !flows || !inj) throw std::runtime_error("x/flows/inj is NULL");
        cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
        EvalParams P = b->params;
        P.x = x; P.mult = nullptr; P.obj_factor = 0.0; P.what = W_FLOWS;
        P.obj = P.grad = P.cons = P.jval = P.hval = nullptr;
        P.flows = flows; P.inj = inj;
        cudaStream_t st = static_cast<cudaStream_t>(stream);     // NULL = legacy default stream
        if (P.n_bus_items > 0) {
            launch_interleave(b, P, 0, (int)b->stages.size(), st);
            acopf_tile_kernel<0u><<<P.n_bus_items, TILE_THREADS, b->smem, st>>>(P, 0);
            cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
            b->launches++;
        }
    });
}

int acopf_batch_eval_host(acopf_batch* b, const double* x, int64_t nx, double obj_factor, const double* mult,
                          int64_t nm, uint32_t what, double* obj, int64_t nobj, double* grad, int64_t ngrad,
                          double* cons, int64_t ncons, double* jval, int64_t nj, double* hval, int64_t nh,
                          void* stream) {
    return guard([&] {
        if (!b->laid_out) throw std::runtime_error("acopf_batch_set_layout was not called");
        // every requested output needs a host buffer of at least the layout's size;
        // every evaluation reads x, the Hessian also the multipliers
        auto need = [&](bool on, const void* p, int64_t have, int64_t want, const char* name) {
            if (!on) return;
            if (!p) throw std::runtime_error(std::string(name) + " is NULL");
            if (have < want)
                throw std::runtime_error(std::string(name) + " has " + std::to_string(have) + " doubles, the layout needs " +
                                         std::to_string(want));
        };
        need(what & ACOPF_ALL, x, nx, b->tot_n, "x");
        need(what & ACOPF_OBJ, obj, nobj, b->tot_obj, "obj");
        need(what & ACOPF_GRAD, grad, ngrad, b->tot_n, "grad");
        need(what & ACOPF_CONS, cons, ncons, b->tot_m, "cons");
        need(what & ACOPF_JAC, jval, nj, b->tot_j, "jval");
        need(what & ACOPF_HESS, hval, nh, b->tot_h, "hval");
        need(what & ACOPF_HESS, mult, nm, b->tot_m, "mult");
        cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
        auto ensure = [&](DevBuf& d, int64_t n) -> double* {
            size_t bytes = sizeof(double) * (size_t)std::max<int64_t>(n, 1);
            if (d.n < bytes) {
                if (d.p) cudaFree(d.p);
                d.p = nullptr;
                d.alloc(bytes);
            }
            return static_cast<double*>(d.p);
        };
        double* dx = ensure(b->h_x, nx);
        double* dm = ensure(b->h_m, nm);
        double* dobj = ensure(b->h_obj, nobj);
        double* dg = ensure(b->h_g, ngrad);
        double* dc = ensure(b->h_c, ncons);
        double* dj = ensure(b->h_j, nj);
        double* dh = ensure(b->h_h, nh);
        if (!b->uploaded) upload(b);
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : b->stream;
        if (b->pipe.size() > 1 && x && nx) {
            // chunk c: H2D of its inputs, its kernels, D2H of its outputs, on stream c % 3;
            // copies of one chunk overlap the kernels and copies of the others.  Composite
            // layouts then run the coupling rows and the stage-order objective (they read every
            // chunk's x / objective terms) and copy out the coupling regions.
            const EvalParams base = b->params;
            EvalParams P = base;
            P.x = dx; P.mult = mult ? dm : nullptr; P.obj_factor = obj_factor; P.what = what;
            P.obj = dobj; P.grad = dg; P.cons = dc; P.jval = dj; P.hval = dh;
            const bool comp = b->pipe_mode == 2;
            cudaEvent_t start;
            cuda_check(cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event");
            cuda_check(cudaEventRecord(start, st), "event record");
            const int S = (int)b->stages.size();
            // start of stage s in region k (s == S: the end of the last stage's block)
            auto rlo = [&](int s, int k) -> int64_t {
                if (s < S) return b->off6[6 * s + k];
                const StageInfo& L = b->stages[S - 1];
                const int64_t sz[6] = {L.n, L.m_eq, L.m_ineq, L.nnz_jeq, L.nnz_jin, L.nnz_h};
                return b->off6[6 * (S - 1) + k] + sz[k];
            };
            auto lo = [&](int s, int k, int64_t total) -> int64_t { return s >= S ? total : b->off6[6 * s + k]; };
            auto m_lo = [&](int s) -> int64_t { return s >= S ? nm : b->off6[6 * s + 1]; };
            auto h2d = [&](double* d, const double* h, int64_t a, int64_t e, cudaStream_t cs, const char* w) {
                if (e > a) cuda_check(cudaMemcpyAsync(d + a, h + a, 8 * (e - a), cudaMemcpyHostToDevice, cs), w);
            };
            auto d2h = [&](double* h, const double* d, int64_t a, int64_t e, cudaStream_t cs, const char* w) {
                if (e > a) cuda_check(cudaMemcpyAsync(h + a, d + a, 8 * (e - a), cudaMemcpyDeviceToHost, cs), w);
            };
            for (size_t c = 0; c < b->pipe.size(); ++c) {
                const auto& pc = b->pipe[c];
                cudaStream_t cs = b->pipe_streams[c % 3];
                cuda_check(cudaStreamWaitEvent(cs, start, 0), "stream wait");
                int64_t x0, x1, r0[2], r1[2], j0[2], j1[2], h0, h1;
                if (comp) {
                    x0 = rlo(pc.s0, 0); x1 = rlo(pc.s1, 0);
                    r0[0] = rlo(pc.s0, 1); r1[0] = rlo(pc.s1, 1); r0[1] = rlo(pc.s0, 2); r1[1] = rlo(pc.s1, 2);
                    j0[0] = rlo(pc.s0, 3); j1[0] = rlo(pc.s1, 3); j0[1] = rlo(pc.s0, 4); j1[1] = rlo(pc.s1, 4);
                    h0 = rlo(pc.s0, 5); h1 = rlo(pc.s1, 5);
                } else {
                    x0 = lo(pc.s0, 0, nx); x1 = lo(pc.s1, 0, nx);
                    r0[0] = m_lo(pc.s0); r1[0] = m_lo(pc.s1); r0[1] = r1[1] = 0;
                    j0[0] = lo(pc.s0, 3, nj); j1[0] = lo(pc.s1, 3, nj); j0[1] = j1[1] = 0;
                    h0 = lo(pc.s0, 5, nh); h1 = lo(pc.s1, 5, nh);
                }
                h2d(dx, x, x0, x1, cs, "H2D x");
                if (mult && nm)
                    for (int q = 0; q < 2; ++q) h2d(dm, mult, r0[q], r1[q], cs, "H2D mult");
                if (pc.aux_count) {
                    acopf_aux_kernel<<<pc.aux_count, BLOCK, b->aux_smem, cs>>>(P, pc.aux_first);
                    cuda_check(cudaGetLastError(), ("acopf_aux_kernel launch (" + std::to_string(b->aux_smem) + " B shared)").c_str());
                    b->launches++;
                }
                if (pc.bus_count && (what & (ACOPF_CONS | ACOPF_JAC | ACOPF_HESS))) {
                    launch_interleave(b, P, pc.s0, pc.s1, cs);
                    if (what == ACOPF_ALL) acopf_tile_kernel<ACOPF_ALL><<<pc.bus_count, TILE_THREADS, b->smem, cs>>>(P, pc.bus_first);
                    else acopf_tile_kernel<0u><<<pc.bus_count, TILE_THREADS, b->smem, cs>>>(P, pc.bus_first);
                    cuda_check(cudaGetLastError(), "acopf_tile_kernel launch");
                    b->launches++;
                }
                if ((what & ACOPF_OBJ) && obj && b->obj_mode != 1) d2h(obj, dobj, pc.s0, pc.s1, cs, "D2H obj");
                if ((what & ACOPF_GRAD) && grad) d2h(grad, dg, x0, x1, cs, "D2H grad");
                for (int q = 0; q < 2; ++q) {
                    if ((what & ACOPF_CONS) && cons) d2h(cons, dc, r0[q], r1[q], cs, "D2H cons");
                    if ((what & ACOPF_JAC) && jval) d2h(jval, dj, j0[q], j1[q], cs, "D2H jac");
                }
                if ((what & ACOPF_HESS) && hval) d2h(hval, dh, h0, h1, cs, "D2H hess");
            }
            // join the pipeline back into the caller's stream
            for (int k = 0; k < 3 && k < (int)b->pipe.size(); ++k) {
                cudaEvent_t done;
                cuda_check(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
                cuda_check(cudaEventRecord(done, b->pipe_streams[k]), "event record");
                cuda_check(cudaStreamWaitEvent(st, done, 0), "stream wait");
                cudaEventDestroy(done);
            }
            if (comp) {
                h2d(dx, x, rlo(S, 0), nx, st, "H2D x (halo)");     // values past the stage blocks (sharded halo)
                const int n_cp = P.n_aux_items - b->n_gen_items;
                if (n_cp > 0 && (what & (ACOPF_CONS | ACOPF_JAC))) {
                    acopf_aux_kernel<<<n_cp, BLOCK, b->aux_smem, st>>>(P, b->n_gen_items);
                    cuda_check(cudaGetLastError(), "acopf_aux_kernel (coupling) launch");
                    b->launches++;
                }
                if (b->obj_mode == 1 && (what & ACOPF_OBJ)) {
                    acopf_objsum_kernel<<<1, BLOCK, 0, st>>>(P);
                    cuda_check(cudaGetLastError(), "acopf_objsum_kernel launch");
                    b->launches++;
                    if (obj) d2h(obj, dobj, 0, 1, st, "D2H obj");
                }
                // the coupling regions: pins after the eq blocks, boxes after the ineq blocks
                if ((what & ACOPF_CONS) && cons) {
                    d2h(cons, dc, rlo(S, 1), rlo(0, 2), st, "D2H cons (pins)");
                    d2h(cons, dc, rlo(S, 2), ncons, st, "D2H cons (boxes)");
                }
                if ((what & ACOPF_JAC) && jval) {
                    d2h(jval, dj, rlo(S, 3), rlo(0, 4), st, "D2H jac (pins)");
                    d2h(jval, dj, rlo(S, 4), nj, st, "D2H jac (boxes)");
                }
            }
            cudaEventDestroy(start);
            cuda_check(cudaStreamSynchronize(st), "stream sync");
            return;
        }
        // the copies and kernels of one evaluation; slot k of `hp` / `dp` / `nb` / `dir` is
        // x, mult, obj, grad, cons, jac, hess
        const void* hp[7] = {x, mult, obj, grad, cons, jval, hval};
        const void* dp[7] = {dx, dm, dobj, dg, dc, dj, dh};
        const int64_t sz[7] = {nx, nm, nobj, ngrad, ncons, nj, nh};
        const bool on[7] = {x && nx > 0, mult && nm > 0, (what & ACOPF_OBJ) && obj, (what & ACOPF_GRAD) && grad,
                            (what & ACOPF_CONS) && cons, (what & ACOPF_JAC) && jval, (what & ACOPF_HESS) && hval};
        auto issue = [&]() {
            for (int k = 0; k < 2; ++k)
                if (on[k]) cuda_check(cudaMemcpyAsync(const_cast<void*>(dp[k]), hp[k], 8 * sz[k], cudaMemcpyHostToDevice, st), "H2D");
            if (acopf_batch_eval(b, dx, obj_factor, mult ? dm : nullptr, what, dobj, dg, dc, dj, dh, st) != 0)
                throw std::runtime_error(g_err);
            for (int k = 2; k < 7; ++k)
                if (on[k]) cuda_check(cudaMemcpyAsync(const_cast<void*>(hp[k]), dp[k], 8 * sz[k], cudaMemcpyDeviceToHost, st), "D2H");
        };
        static const bool graphs_env = !getenv("ACOPF_HOST_GRAPHS") || atoi(getenv("ACOPF_HOST_GRAPHS")) != 0;
        bool use_graph = graphs_env && !b->host_graphs_off && st == b->stream;
        for (int k = 0; k < 7 && use_graph; ++k) {      // graph copies need pinned host memory
            if (!on[k]) continue;
            cudaPointerAttributes a{};
            if (cudaPointerGetAttributes(&a, hp[k]) != cudaSuccess || a.type != cudaMemoryTypeHost) {
                cudaGetLastError();
                use_graph = false;
            }
        }
        if (!use_graph) {
            issue();
            cuda_check(cudaStreamSynchronize(st), "stream sync");
            return;
        }
        acopf_batch::HostGraph* g = nullptr;
        for (auto& h : b->host_graphs) {
            bool same = h.what == what && h.mult == (mult != nullptr) && h.obj_factor == obj_factor;
            for (int k = 0; k < 7 && same; ++k) same = h.sz[k] == (on[k] ? sz[k] : 0) && h.dev[k] == (on[k] ? dp[k] : nullptr);
            if (same) { g = &h; break; }
        }
        if (!g && ++b->host_graph_captures > 32) {
            b->host_graphs_off = true;
            issue();
            cuda_check(cudaStreamSynchronize(st), "stream sync");
            return;
        }
        if (!g) {
            if (b->host_graphs.size() >= 16) {     // bounded cache (e.g. a varying obj_factor)
                for (auto& o : b->host_graphs) {
                    if (o.exec) cudaGraphExecDestroy(o.exec);
                    if (o.graph) cudaGraphDestroy(o.graph);
                }
                b->host_graphs.clear();
            }
            acopf_batch::HostGraph h;
            h.what = what; h.mult = mult != nullptr; h.obj_factor = obj_factor;
            for (int k = 0; k < 7; ++k) { h.sz[k] = on[k] ? sz[k] : 0; h.dev[k] = on[k] ? dp[k] : nullptr; h.host[k] = on[k] ? hp[k] : nullptr; }
            const int64_t l0 = b->launches;
            cudaGraph_t graph = nullptr;
            bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                try { issue(); } catch (...) { ok = false; }
                ok = cudaStreamEndCapture(st, &graph) == cudaSuccess && ok;
            }
            h.n_launches = b->launches - l0;
            b->launches = l0;
            if (ok) {       // the memcpy nodes, by their device ends
                size_t n = 0;
                ok = cudaGraphGetNodes(graph, nullptr, &n) == cudaSuccess;
                std::vector<cudaGraphNode_t> nodes(n);
                if (ok && n) ok = cudaGraphGetNodes(graph, nodes.data(), &n) == cudaSuccess;
                for (size_t i = 0; i < n && ok; ++i) {
                    cudaGraphNodeType t;
                    if (cudaGraphNodeGetType(nodes[i], &t) != cudaSuccess) { ok = false; break; }
                    if (t != cudaGraphNodeTypeMemcpy) continue;
                    cudaMemcpy3DParms mp{};
                    if (cudaGraphMemcpyNodeGetParams(nodes[i], &mp) != cudaSuccess) { ok = false; break; }
                    for (int k = 0; k < 7; ++k)
                        if (on[k] && (k < 2 ? mp.dstPtr.ptr : mp.srcPtr.ptr) == dp[k]) { h.node[k] = nodes[i]; h.parm[k] = mp; }
                }
                for (int k = 0; k < 7 && ok; ++k) ok = !on[k] || h.node[k] != nullptr;
                if (ok) ok = cudaGraphInstantiate(&h.exec, graph, 0) == cudaSuccess;
            }
            cudaGetLastError();
            if (!ok) {          // capture not possible here: plain issue from now on
                if (h.exec) cudaGraphExecDestroy(h.exec);
                if (graph) cudaGraphDestroy(graph);
                b->host_graphs_off = true;
                issue();
                cuda_check(cudaStreamSynchronize(st), "stream sync");
                return;
            }
            h.graph = graph;
            b->host_graphs.push_back(h);
            g = &b->host_graphs.back();
        }
        bool patched = true;
        for (int k = 0; k < 7 && patched; ++k) {   // patch the host ends that moved
            if (!on[k] || g->host[k] == hp[k]) continue;
            cudaMemcpy3DParms mp = g->parm[k];
            if (k < 2) mp.srcPtr.ptr = const_cast<void*>(hp[k]);
            else mp.dstPtr.ptr = const_cast<void*>(hp[k]);
            const cudaError_t ue = cudaGraphExecMemcpyNodeSetParams(g->exec, g->node[k], &mp);
            if (ue != cudaSuccess) {
                if (getenv("ACOPF_DEBUG_GRAPHS"))
                    fprintf(stderr, "acopf: graph copy update k=%d: %s; plain copies from now on\n", k, cudaGetErrorString(ue));
                cudaGetLastError();
                patched = false;
                break;
            }
            g->host[k] = hp[k];
        }
        if (!patched) {        // e.g. host memory from another allocator: the plain sequence
            b->host_graphs_off = true;
            issue();
            cuda_check(cudaStreamSynchronize(st), "stream sync");
            return;
        }
        cuda_check(cudaGraphLaunch(g->exec, st), "cudaGraphLaunch");
        b->launches += g->n_launches;
        cuda_check(cudaStreamSynchronize(st), "stream sync");
    });
}

// Stage-local pattern rows, in stage row order.
static void stage_rows(const acopf_batch* b, int s, int which,
                       std::vector<int64_t>& rowlen, std::vector<int32_t>& cols) {
    const StageInfo& st = b->stages[s];
    const Topo& T = *b->topos[st.topo];
    rowlen.clear();
    cols.clear();
    const int ntile = (int)st.table.size();
    int seg0 = which == 0 ? 0 : 2;
    for (int seg = seg0; seg < seg0 + 2; ++seg) {
        for (int t = 0; t < ntile; ++t) {
            const TileTable& tt = b->tables[st.table[t]];
            int64_t e0 = 0;
            for (int q = 0; q < seg; ++q) e0 += tt.L[q];
            for (int r = 0; r < tt.nB; ++r) {
                int len = tt.rowlen[seg * tt.nB + r];
                rowlen.push_back(len);
                cols.insert(cols.end(), tt.cols.begin() + e0, tt.cols.begin() + e0 + len);
                e0 += len;
            }
        }
    }
    if (which == 0) {
        std::vector<int> c;
        for (int r = 0; r < T.nr; ++r) {
            if (std::binary_search(st.removed_rated.begin(), st.removed_rated.end(), r)) continue;
            flow_row_cols(T, T.rated_branch[r], c);
            for (int rep = 0; rep < 2; ++rep) {
                rowlen.push_back((int64_t)c.size());
                cols.insert(cols.end(), c.begin(), c.end());
            }
        }
    } else {
        for (int g = 0; g < T.ng; ++g) { rowlen.push_back(1); cols.push_back(2 * T.nb + g); }
        for (int g = 0; g < T.ng; ++g) rowlen.push_back(0);
    }
}

int acopf_batch_pattern(const acopf_batch* b, int32_t stage, int32_t which, int64_t n_rows, int64_t* indptr,
                        int32_t* indices) {
    return guard([&] {
        if (which != 0 && which != 1) throw std::runtime_error("which must be 0 (J) or 1 (H)");
        std::vector<int64_t> rowlen;
        std::vector<int32_t> cols;
        if (stage >= 0) {
            if (stage >= (int)b->stages.size()) throw std::runtime_error("stage out of range");
            stage_rows(b, stage, which, rowlen, cols);
            if ((int64_t)rowlen.size() != n_rows) throw std::runtime_error("n_rows does not match the stage");
            indptr[0] = 0;
            for (int64_t r = 0; r < n_rows; ++r) indptr[r + 1] = indptr[r] + rowlen[r];
            std::copy(cols.begin(), cols.end(), indices);
            return;
        }
        if (!b->laid_out) throw std::runtime_error("acopf_batch_set_layout was not called");
        // whole laid-out batch: place every row at its offset, then check the rows tile the data
        std::vector<int64_t> start(n_rows, -1), len(n_rows, 0);
        for (size_t s = 0; s < b->stages.size(); ++s) {
            const StageInfo& st = b->stages[s];
            const int64_t* o = &b->off6[6 * s];
            stage_rows(b, (int)s, which, rowlen, cols);
            int64_t pos = 0;
            for (size_t r = 0; r < rowlen.size(); ++r) {
                int64_t grow, gstart;
                if (which == 0) {
                    bool eq = (int64_t)r < st.m_eq;
                    grow = eq ? o[1] + (int64_t)r : o[2] + ((int64_t)r - st.m_eq);
                    gstart = eq ? o[3] + pos : o[4] + (pos - st.nnz_jeq);
                } else {
                    grow = o[0] + (int64_t)r;
                    gstart = o[5] + pos;
                }
                if (grow < 0 || grow >= n_rows) throw std::runtime_error("row outside n_rows");
                start[grow] = gstart;
                len[grow] = rowlen[r];
                for (int64_t e = 0; e < rowlen[r]; ++e) indices[gstart + e] = (int32_t)(o[0] + cols[pos + e]);
                pos += rowlen[r];
            }
        }
        if (which == 0) {
            for (size_t c = 0; c < b->cp_row.size(); ++c) {
                int64_t r = b->cp_row[c], p = b->cp_jpos[c];
                start[r] = p;
                len[r] = 2;
                int64_t lo = std::min(b->cp_a[c], b->cp_b[c]), hi = std::max(b->cp_a[c], b->cp_b[c]);
                indices[p] = (int32_t)lo;
                indices[p + 1] = (int32_t)hi;
            }
        }
        indptr[0] = 0;
        for (int64_t r = 0; r < n_rows; ++r) {
            if (len[r] > 0 && start[r] != indptr[r]) throw std::runtime_error("layout rows are not contiguous in row order");
            indptr[r + 1] = indptr[r] + len[r];
        }
    });
}

int64_t acopf_batch_launches(const acopf_batch* b) { return b ? b->launches : 0; }

int acopf_batch_verify(const acopf_batch* b, int64_t* stats) {
    return guard([&] {
        int64_t ntiles = 0, nends = 0, area = 0, pads = 0, smem = 0, rounds = 0, lane_terms = 0, chain = 0;
        int64_t cost[3] = {0, 0, 0};
        for (size_t ti = 0; ti < b->topos.size(); ++ti) {
            ntiles += (int64_t)b->base_table[ti].size();
            for (int id : b->base_table[ti]) nends += (int64_t)b->tables[id].ends.size();
        }
        for (size_t i = 0; i < b->tables.size(); ++i) {
            const TileTable& tt = b->tables[i];
            const std::string err = verify_tile(tt);
            if (!err.empty()) throw std::runtime_error("table " + std::to_string(i) + ": " + err);
            std::vector<uint8_t> blob;
            tt.serialise(*b->topos[tt.topo], blob);
            area += tt.nArea;
            pads += (int64_t)tt.nega.size();
            tile_store_cost(tt, cost);
            for (size_t r = 0; r < tt.sround.size() / 4; ++r) {
                ++rounds;
                lane_terms += (int64_t)tt.sround[4 * r + 1] * tt.sround[4 * r + 3];
                chain += tt.sround[4 * r + 1];
            }
            smem = std::max<int64_t>(smem, (int64_t)tile_smem_bytes((int)blob.size(), tt.nArea));
        }
        if (stats) {
            stats[0] = (int64_t)b->tables.size(); stats[1] = ntiles; stats[2] = nends;
            stats[3] = area; stats[4] = pads; stats[5] = smem;
            stats[6] = rounds; stats[7] = lane_terms; stats[8] = chain;
            stats[9] = cost[0]; stats[10] = cost[1]; stats[11] = cost[2];
        }
    });
}

int acopf_nccl_unique_id(void* id128) {
    return guard([&] {
        if (!id128) throw std::runtime_error("id buffer is NULL");
        ncclUniqueId id;
        nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof id);
    });
}

int acopf_multi_create(acopf_batch* b, int32_t rank, int32_t world, const int64_t* x_lo, const int64_t* x_hi,
                       const int64_t* need_ptr, const int64_t* need_idx, int64_t halo_dst0,
                       const int32_t* obj_counts, const void* nccl_id, acopf_multi** out) {
    return guard([&] {
        if (!b || !out || world < 1 || rank < 0 || rank >= world) throw std::runtime_error("bad arguments");
        if (!b->laid_out) throw std::runtime_error("acopf_batch_set_layout was not called");
        if (b->obj_mode != ACOPF_OBJ_TERMS) throw std::runtime_error("a sharded batch needs ACOPF_OBJ_TERMS");
        std::unique_ptr<acopf_multi> M(new acopf_multi());
        M->b = b;
        M->rank = rank;
        M->world = world;
        M->halo_dst0 = halo_dst0;
        // exports: every global index some other rank needs that lies in this rank's x range
        const int64_t lo = x_lo[rank], hi = x_hi[rank];
        std::vector<int64_t> ex;
        for (int r = 0; r < world; ++r) {
            if (r == rank) continue;
            for (int64_t i = need_ptr[r]; i < need_ptr[r + 1]; ++i)
                if (need_idx[i] >= lo && need_idx[i] < hi) ex.push_back(need_idx[i]);
        }
        std::sort(ex.begin(), ex.end());
        ex.erase(std::unique(ex.begin(), ex.end()), ex.end());
        // every rank's export list (derived from the same inputs), for the gathered layout
        std::vector<std::vector<int64_t>> exports(world);
        for (int q = 0; q < world; ++q) {
            for (int r = 0; r < world; ++r) {
                if (r == q) continue;
                for (int64_t i = need_ptr[r]; i < need_ptr[r + 1]; ++i)
                    if (need_idx[i] >= x_lo[q] && need_idx[i] < x_hi[q]) exports[q].push_back(need_idx[i]);
            }
            std::sort(exports[q].begin(), exports[q].end());
            exports[q].erase(std::unique(exports[q].begin(), exports[q].end()), exports[q].end());
            M->export_max = std::max<int64_t>(M->export_max, (int64_t)exports[q].size());
        }
        for (int64_t g : ex) M->export_idx.push_back(g - lo);
        // halo: this rank's needs, each read from its owner's slot in the gathered buffer
        for (int64_t i = need_ptr[rank]; i < need_ptr[rank + 1]; ++i) {
            const int64_t g = need_idx[i];
            int owner = -1;
            for (int q = 0; q < world && owner < 0; ++q)
                if (g >= x_lo[q] && g < x_hi[q]) owner = q;
            if (owner < 0 || owner == rank) throw std::runtime_error("halo index not owned by another rank");
            const auto& e = exports[owner];
            const int64_t j = (int64_t)(std::lower_bound(e.begin(), e.end(), g) - e.begin());
            M->halo_src.push_back((int64_t)owner * M->export_max + j);
        }
        M->obj_counts.assign(obj_counts, obj_counts + world);
        for (int32_t c : M->obj_counts) M->obj_max = std::max<int>(M->obj_max, c);
        if (M->obj_counts[rank] != (int)b->stages.size())
            throw std::runtime_error("obj_counts[rank] must equal this rank's stage count");
        if (nccl_id) {            // device side: communicator and buffers (collective over all ranks)
            cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof id);
            nccl_check(nccl().CommInitRank(&M->comm, world, id, rank), "ncclCommInitRank");
            M->d_export.upload(M->export_idx);
            M->d_halo_src.upload(M->halo_src);
            M->d_counts.upload(M->obj_counts);
            M->d_send.alloc(sizeof(double) * (size_t)M->export_max);
            M->d_recv.alloc(sizeof(double) * (size_t)M->export_max * world);
            M->d_obj_send.alloc(sizeof(double) * (size_t)M->obj_max);
            M->d_obj_recv.alloc(sizeof(double) * (size_t)M->obj_max * world);
            cuda_check(cudaStreamCreateWithFlags(&M->halo_stream, cudaStreamNonBlocking), "stream");
            for (cudaEvent_t* e : {&M->ev_fork, &M->ev_halo, &M->ev_gen})
                cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        }
        *out = M.release();
    });
}

int acopf_multi_plan(const acopf_multi* m, int64_t* sizes3, int64_t* export_idx, int64_t* halo_src) {
    return guard([&] {
        if (sizes3) { sizes3[0] = (int64_t)m->export_idx.size(); sizes3[1] = m->export_max; sizes3[2] = (int64_t)m->halo_src.size(); }
        if (export_idx) std::copy(m->export_idx.begin(), m->export_idx.end(), export_idx);
        if (halo_src) std::copy(m->halo_src.begin(), m->halo_src.end(), halo_src);
    });
}

int acopf_multi_destroy(acopf_multi* m) {
    if (m) {
        cudaSetDevice(m->b->device);
        delete m;
    }
    return 0;
}

int acopf_batch_eval_multi(acopf_multi* m, double* x, double obj_factor, const double* mult, uint32_t what,
                           double* obj, double* grad, double* cons, double* jval, double* hval, void* stream) {
    return guard([&] {
        if (!m->comm) throw std::runtime_error("multi handle made without a NCCL id (plan only)");
        acopf_batch* b = m->b;
        if (!b->uploaded) upload(b);
        if ((what & ACOPF_ALL) && !x) throw std::runtime_error("x is NULL");
        if ((what & ACOPF_OBJ) && !obj) throw std::runtime_error("obj is NULL");
        if ((what & ACOPF_GRAD) && !grad) throw std::runtime_error("grad is NULL");
        if ((what & ACOPF_CONS) && !cons) throw std::runtime_error("cons is NULL");
        if ((what & ACOPF_JAC) && !jval) throw std::runtime_error("jval is NULL");
        if ((what & ACOPF_HESS) && (!hval || !mult)) throw std::runtime_error("hval/mult is NULL");
        cuda_check(cudaSetDevice(b->device), "cudaSetDevice");
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        EvalParams P = b->params;
        P.x = x; P.mult = mult; P.obj_factor = obj_factor; P.what = what;
        P.obj = static_cast<double*>(m->d_obj_send.p);      // this rank's w_s f_s, padded to obj_max
        P.grad = grad; P.cons = cons; P.jval = jval; P.hval = hval;
        cuda_check(cudaEventRecord(m->ev_fork, st), "event record");
        // halo chain on its own stream: pack -> NCCL all-gather -> unpack -> coupling rows;
        // it overlaps the tile kernel, which never reads the halo
        const int n_cp_items = P.n_aux_items - b->n_gen_items;
        const bool halo = (what & (ACOPF_CONS | ACOPF_JAC)) != 0;
        if (halo) {
            cudaStream_t hs = m->halo_stream;
            cuda_check(cudaStreamWaitEvent(hs, m->ev_fork, 0), "stream wait");
            const long long ne = (long long)m->export_idx.size(), nh = (long long)m->halo_src.size();
            acopf_halo_pack_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>(1184, (m->export_max + BLOCK - 1) / BLOCK)),
                                     BLOCK, 0, hs>>>(x, static_cast<const long long*>(m->d_export.p), ne, m->export_max,
                                                     static_cast<double*>(m->d_send.p));
            cuda_check(cudaGetLastError(), "acopf_halo_pack_kernel launch");
            b->launches++;
            nccl_check(nccl().AllGather(m->d_send.p, m->d_recv.p, (size_t)m->export_max, ncclDouble, m->comm, hs),
                       "ncclAllGather(halo)");
            if (nh > 0) {
                acopf_halo_unpack_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>(1184, (nh + BLOCK - 1) / BLOCK)),
                                           BLOCK, 0, hs>>>(x, m->halo_dst0, static_cast<const long long*>(m->d_halo_src.p),
                                                           nh, static_cast<const double*>(m->d_recv.p));
                cuda_check(cudaGetLastError(), "acopf_halo_unpack_kernel launch");
                b->launches++;
            }
            if (n_cp_items > 0) {
                acopf_aux_kernel<<<n_cp_items, BLOCK, b->aux_smem, hs>>>(P, b->n_gen_items);
                cuda_check(cudaGetLastError(), "acopf_aux_kernel (coupling) launch");
                b->launches++;
            }
            cuda_check(cudaEventRecord(m->ev_halo, hs), "event record");
        }
        // generator chunks (gradient, PG Hessian diagonal, w_s f_s) beside the tile kernel;
        // the objective all-gather is issued by every rank whenever the objective is asked
        // (collectives must match across ranks, even for a rank without generator items)
        const bool gen = (what & (ACOPF_OBJ | ACOPF_GRAD | ACOPF_HESS)) && (b->n_gen_items > 0 || (what & ACOPF_OBJ));
        if (gen) {
            cuda_check(cudaStreamWaitEvent(b->aux_stream, m->ev_fork, 0), "stream wait");
            if (b->n_gen_items > 0) {
                acopf_aux_kernel<<<b->n_gen_items, BLOCK, b->aux_smem, b->aux_stream>>>(P, 0);
                cuda_check(cudaGetLastError(), "acopf_aux_kernel (generators) launch");
                b->launches++;
            }
            if (what & ACOPF_OBJ) {
                // every rank's terms, then the stage-order sum (bit-identical to one GPU)
                nccl_check(nccl().AllGather(m->d_obj_send.p, m->d_obj_recv.p, (size_t)m->obj_max, ncclDouble, m->comm,
                                            b->aux_stream), "ncclAllGather(objective)");
                acopf_objsum_multi_kernel<<<1, BLOCK, 0, b->aux_stream>>>(static_cast<const double*>(m->d_obj_recv.p),
                                                                          static_cast<const int*>(m->d_counts.p),
                                                                          m->world, m->obj_max, obj);
                cuda_check(cudaGetLastError(), "acopf_objsum_multi_kernel launch");
                b->launches++;
            }
            cuda_check(cudaEventRecord(m->ev_gen, b->aux_stream), "event record");
        }
        if ((what & (ACOPF_CONS | ACOPF_JAC | ACOPF_HESS)) && P.n_bus_items > 0) launch_bus_work(b, P, st);
        if (halo) cuda_check(cudaStreamWaitEvent(st, m->ev_halo, 0), "stream wait");
        if (gen) cuda_check(cudaStreamWaitEvent(st, m->ev_gen, 0), "stream wait");
    });
}

int acopf_kkt_assemble(int64_t nf, int64_t me, double* K, const int64_t* h_ptr, const int32_t* h_col,
                       const int64_t* h_vi, const double* hval, const double* dx, const int64_t* jt_ptr,
                       const int32_t* jt_row, const int64_t* jt_vi, const int64_t* ji_ptr, const int32_t* ji_col,
                       const int64_t* ji_vi, const double* jval, const double* ds, const int64_t* je_ptr,
                       const int32_t* je_col, const int64_t* je_vi, const double* sc_e, const double* sc_i,
                       double reg, double delta, void* stream) {
    return guard([&] {
        if (nf < 0 || me < 0 || !K) throw std::runtime_error("bad arguments");
        KKTParams Q{};
        Q.nf = nf; Q.me = me; Q.dim = nf + me; Q.K = K;
        Q.h_ptr = h_ptr; Q.h_col = h_col; Q.h_vi = h_vi; Q.hval = hval; Q.dx = dx;
        Q.jt_ptr = jt_ptr; Q.jt_row = jt_row; Q.jt_vi = jt_vi;
        Q.ji_ptr = ji_ptr; Q.ji_col = ji_col; Q.ji_vi = ji_vi; Q.jval = jval; Q.ds = ds;
        Q.je_ptr = je_ptr; Q.je_col = je_col; Q.je_vi = je_vi; Q.sc_e = sc_e; Q.sc_i = sc_i;
        Q.reg = reg; Q.delta = delta;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (nf > 0) {
            acopf_kkt_hfull_kernel<<<(unsigned)((nf + 127) / 128), 128, 0, st>>>(Q);
            cuda_check(cudaGetLastError(), "acopf_kkt_hfull_kernel launch");
            const unsigned gx = (unsigned)std::min<int64_t>(64, (nf + 255) / 256);
            acopf_kkt_finish_kernel<<<dim3(gx, (unsigned)std::min<int64_t>(nf, 65535)), 256, 0, st>>>(Q);
            cuda_check(cudaGetLastError(), "acopf_kkt_finish_kernel launch");
        }
        const int64_t nd = std::max(nf, me);
        if (nd > 0) {
            acopf_kkt_diag_je_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, st>>>(Q);
            cuda_check(cudaGetLastError(), "acopf_kkt_diag_je_kernel launch");
        }
    });
}

int acopf_graph_islands(int32_t nbus, const uint8_t* alive, int64_t nedge, const int32_t* ea, const int32_t* eb,
                        const uint8_t* edge_live, int32_t* n_islands, int32_t* label) {
    return guard([&] {
        std::vector<int32_t> parent(nbus);
        std::iota(parent.begin(), parent.end(), 0);
        auto find = [&](int32_t v) {
            while (parent[v] != v) { parent[v] = parent[parent[v]]; v = parent[v]; }
            return v;
        };
        for (int64_t k = 0; k < nedge; ++k) {
            if (edge_live && !edge_live[k]) continue;
            const int32_t a = ea[k], b = eb[k];
            if (a < 0 || a >= nbus || b < 0 || b >= nbus) throw std::runtime_error("edge endpoint out of range");
            if (!alive[a] || !alive[b]) continue;
            const int32_t ra = find(a), rb = find(b);
            if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
        }
        // labels in order of first bus (the order of check_connectivity's DFS roots)
        std::vector<int32_t> lab(nbus, -1);
        int32_t count = 0;
        for (int32_t v = 0; v < nbus; ++v) {
            if (!alive[v]) continue;
            const int32_t r = find(v);
            if (lab[r] < 0) lab[r] = count++;
            if (label) label[v] = lab[r];
        }
        if (label)
            for (int32_t v = 0; v < nbus; ++v) if (!alive[v]) label[v] = -1;
        *n_islands = count;
    });
}

int acopf_graph_bridges(int32_t nbus, int64_t nedge, const int32_t* ea, const int32_t* eb, const uint8_t* edge_live,
                        uint8_t* is_bridge) {
    return guard([&] {
        // iterative Tarjan over the live multigraph: a parallel twin is a back edge
        std::vector<int64_t> ptr(nbus + 1, 0), adj_e;
        std::vector<int32_t> adj_v;
        for (int64_t k = 0; k < nedge; ++k) {
            is_bridge[k] = 0;
            if (edge_live && !edge_live[k]) continue;
            if (ea[k] < 0 || ea[k] >= nbus || eb[k] < 0 || eb[k] >= nbus) throw std::runtime_error("edge endpoint out of range");
            ptr[ea[k] + 1]++;
            ptr[eb[k] + 1]++;
        }
        for (int32_t v = 0; v < nbus; ++v) ptr[v + 1] += ptr[v];
        adj_e.resize(ptr[nbus]);
        adj_v.resize(ptr[nbus]);
        std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
        for (int64_t k = 0; k < nedge; ++k) {
            if (edge_live && !edge_live[k]) continue;
            adj_v[fill[ea[k]]] = eb[k]; adj_e[fill[ea[k]]++] = k;
            adj_v[fill[eb[k]]] = ea[k]; adj_e[fill[eb[k]]++] = k;
        }
        std::vector<int32_t> disc(nbus, -1), low(nbus, 0);
        std::vector<int64_t> it(nbus, 0), via(nbus, -1);
        std::vector<int32_t> stack;
        int32_t t = 0;
        for (int32_t root = 0; root < nbus; ++root) {
            if (disc[root] >= 0 || ptr[root] == ptr[root + 1]) continue;
            disc[root] = low[root] = t++;
            it[root] = ptr[root];
            via[root] = -1;
            stack.push_back(root);
            while (!stack.empty()) {
                const int32_t u = stack.back();
                bool pushed = false;
                while (it[u] < ptr[u + 1]) {
                    const int64_t j = it[u]++;
                    const int32_t v = adj_v[j];
                    const int64_t k = adj_e[j];
                    if (k == via[u]) continue;
                    if (disc[v] < 0) {
                        disc[v] = low[v] = t++;
                        it[v] = ptr[v];
                        via[v] = k;
                        stack.push_back(v);
                        pushed = true;
                        break;
                    }
                    low[u] = std::min(low[u], disc[v]);
                }
                if (pushed) continue;
                stack.pop_back();
                if (!stack.empty()) {
                    const int32_t p = stack.back();
                    low[p] = std::min(low[p], low[u]);
                    if (low[u] > disc[p]) is_bridge[via[u]] = 1;
                }
            }
        }
    });
}

int acopf_copy_runs(int64_t n, double* dst, const int64_t* dst_off, const double* src, const int64_t* src_off,
                    const int64_t* len) {
    return guard([&] {
        int64_t total = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (len[i] < 0 || dst_off[i] < 0 || src_off[i] < 0) throw std::runtime_error("negative run");
            total += len[i];
        }
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const int nt = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)hw, 16, total / (1 << 20) + 1}));
        std::atomic<int64_t> next{0};
        auto work = [&] {
            for (int64_t i; (i = next.fetch_add(1)) < n;)
                if (len[i]) std::memcpy(dst + dst_off[i], src + src_off[i], sizeof(double) * (size_t)len[i]);
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
    });
}

int acopf_format_matrix(const char* section, int64_t rows, const int64_t* row_ptr, const double* values,
                        char* out, int64_t cap, int64_t* len) {
    return guard([&] {
        if (!section || rows < 0 || (rows > 0 && (!row_ptr || !values))) throw std::runtime_error("bad arguments");
        std::string s;
        s.reserve((size_t)std::max<int64_t>(64, rows > 0 ? 12 * (row_ptr[rows] - row_ptr[0]) + 4 * rows : 64));
        fmt_matrix(section, rows, row_ptr, values, s);
        if (len) *len = (int64_t)s.size();
        if (out) {
            if ((int64_t)s.size() > cap) throw std::runtime_error("output buffer too small");
            std::memcpy(out, s.data(), s.size());
        }
    });
}

int acopf_canonical_order(int64_t n, const int32_t* cols, int32_t* perm) {
    return guard([&] {
        std::vector<std::pair<int, Sym>> coo(n);
        for (int64_t i = 0; i < n; ++i) coo[i] = {cols[i], Sym{0, (int)i, 0}};
        Row row;
        canonicalise(coo, row);
        for (size_t t = 0; t < row.terms.size(); ++t) perm[t] = row.terms[t].a;
    });
}

}  // extern "C"

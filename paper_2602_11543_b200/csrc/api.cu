// C-ABI implementation: one spes_ctx per node/GPU. Host orchestration in C++,
// device work in kernels.cu / gemm.cu, collectives through NCCL.
// Reference interfaces each entry point replaces are listed in include/spes_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spes_b200.h"
#include "glibc_expf.h"
#include "kernels.h"
#include "wire.hpp"
#include "tmap.hpp"

using spes_dev::GemmGroup;
using spes_k::bf16;

namespace {

thread_local std::string g_last_error;

struct SpesError : std::runtime_error {
    spes_status code;
    SpesError(spes_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(spes_status c, const std::string& m) { throw SpesError(c, m); }

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(SPES_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void ckn(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(SPES_NCCL_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}

template <class F>
spes_status guard(F&& f) {
    try {
        f();
        return SPES_OK;
    } catch (const SpesError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const spes_wire::ProtocolError& e) {  // "[Code] message"
        g_last_error = e.what();
        return SPES_PROTOCOL_ERROR;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return SPES_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return SPES_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return SPES_LOGIC_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SPES_RUNTIME_ERROR;
    }
}

// ---- layout (enumerate_blocks, proj/include/spes/model.hpp:95-111) ----
struct Layout {
    int64_t V, d, f;
    int L, M, k;
    int64_t off_emb() const { return 0; }
    int64_t off_head() const { return V * d; }
    int64_t off_norm(int l) const { return 2 * V * d + static_cast<int64_t>(l) * (d + d * M); }
    int64_t off_router(int l) const { return off_norm(l) + d; }
    int64_t psi() const { return 2 * V * d + static_cast<int64_t>(L) * (d + d * M); }
    int64_t per_expert() const { return 3 * d * f; }
    int64_t off_expert(int l, int j) const {
        return psi() + (static_cast<int64_t>(l) * M + j) * per_expert();
    }
    int64_t total() const { return off_expert(L, 0); }
};

Layout layout_of(const spes_model_cfg* c) {
    return Layout{c->vocab, c->hidden, c->intermediate, c->layers, c->experts_total,
                  c->experts_active};
}

// ModelConfig::validate (model.hpp:33-40) + the B200 routing limits. Hidden, intermediate
// and vocab sizes are free: the device layout pads them to the tcgen05 tile (device_cfg).
void validate_cfg(const spes_model_cfg* c) {
    if (!c) fail(SPES_INVALID_ARGUMENT, "model config: null");
    if (c->vocab < 1 || c->hidden < 1 || c->intermediate < 1 || c->layers < 1)
        throw std::invalid_argument("model config: all dims must be >= 1");
    if (c->experts_active < 1 || c->experts_active > c->experts_total)
        throw std::invalid_argument("model config: need 1 <= k <= M");
    if (c->coeff_ce < 0 || c->coeff_lb < 0 || c->coeff_moe_z < 0 || c->coeff_z < 0)
        throw std::invalid_argument("model config: loss coefficients must be >= 0");
    if (c->tied_head) throw std::logic_error("tied head not implemented");
    if (c->experts_total > 64 || c->experts_active > 8)
        fail(SPES_INVALID_ARGUMENT, "B200 path: experts_total <= 64 and experts_active <= 8");
}

int bn_for(int64_t n) { return (n % 256 == 0) ? 256 : 128; }

// The device model: hidden, intermediate and vocab rounded up to the 128-wide tcgen05 tile.
// Padded rows / columns of every block are zeros and stay zeros (their gradients are zero,
// so AdamW / SGD / sync / merge keep them at zero); the rmsnorm mean divides by the true
// hidden size and the softmax-CE masks the padded vocabulary columns, so the padded model
// computes the caller's model exactly (parameter I/O converts between the layouts).
spes_model_cfg device_cfg(const spes_model_cfg* c) {
    spes_model_cfg p = *c;
    p.hidden = (c->hidden + 127) / 128 * 128;
    p.intermediate = (c->intermediate + 127) / 128 * 128;
    p.vocab = (c->vocab + 127) / 128 * 128;
    return p;
}

// Copy between the caller's layout (enumerate_blocks of its config, `u`) and the padded
// device layout (`p`, zero-filled by the caller when to_dev): every block is a row-major
// matrix whose rows and columns both may be padded.
void convert_layout(const Layout& U, const Layout& D, const float* src, float* dst, bool to_dev) {
    auto block = [&](int64_t uo, int64_t po, int64_t ur, int64_t uc, int64_t pc) {
        for (int64_t r = 0; r < ur; ++r) {
            const float* a = to_dev ? src + uo + r * uc : src + po + r * pc;
            float* b = to_dev ? dst + po + r * pc : dst + uo + r * uc;
            std::memcpy(b, a, sizeof(float) * uc);
        }
    };
    block(U.off_emb(), D.off_emb(), U.V, U.d, D.d);     // emb [V x d]
    block(U.off_head(), D.off_head(), U.d, U.V, D.V);   // head [d x V]
    for (int l = 0; l < U.L; ++l) {
        block(U.off_norm(l), D.off_norm(l), 1, U.d, D.d);        // gain [d]
        block(U.off_router(l), D.off_router(l), U.d, U.M, D.M);  // router [d x M]
    }
    for (int l = 0; l < U.L; ++l)
        for (int j = 0; j < U.M; ++j) {
            const int64_t uo = U.off_expert(l, j), po = D.off_expert(l, j);
            block(uo, po, U.d, U.f, D.f);                                      // wg [d x f]
            block(uo + U.d * U.f, po + D.d * D.f, U.d, U.f, D.f);              // wu [d x f]
            block(uo + 2 * U.d * U.f, po + 2 * D.d * D.f, U.f, U.d, D.d);      // wd [f x d]
        }
}
int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

struct DevMem {
    std::vector<void*> ptrs;
    template <class T>
    T* alloc(int64_t n) {
        void* p = nullptr;
        const size_t bytes = static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T);
        ck(cudaMalloc(&p, bytes), "cudaMalloc");
        ck(cudaMemset(p, 0, bytes), "cudaMemset");
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    void release() {
        for (void* p : ptrs) cudaFree(p);
        ptrs.clear();
    }
    ~DevMem() { release(); }
};

struct LayerBufs {
    float *logits, *probs, *topk_w, *lse_r, *inv_rms, *denom, *y, *row_w, *lb_coeff;
    int32_t *topk_idx, *chunk_counts, *counts, *pad_off, *slot_row, *row_token, *tiles;
    GemmGroup* groups;
    bf16 *xp, *gu, *hact;  // routed rows (expert-major dispatch), GEMM outputs
    bf16* normed_bf;       // router-normalized h (dispatch source; router-gradient operand)
    CUtensorMap a_normed_mn;  // normed_bf [tokens x d] as the MN-major A of g_router
    int64_t* grad_off;  // device [M]
    CUtensorMap a_xp, a_hact, a_xp_mn, a_hact_mn;  // *_mn: [tokens x features] as MN-major
    CUtensorMap b_w1_mn, b_w2_mn, b_w2, b_w1;  // *_mn: row-major weights as MN-major B
};

}  // namespace

struct spes_ctx {
    spes_model_cfg cfg;  // the caller's model
    Layout lay;          // device layout (hidden / intermediate / vocab padded to 128)
    Layout ulay;         // the caller's layout (enumerate_blocks of cfg)
    bool padded = false;
    int node = 0, n_nodes = 1, device = 0;
    int expf_variant = 1;
    cudaStream_t stream = nullptr;
    // low-priority side stream: the owned experts' AdamW runs there as soon as their dW
    // GEMMs finish, under the router / norm / embedding backward on the main stream
    cudaStream_t side = nullptr;
    bool overlap_opt = true;
    bool early_wd = true;  // wd's AdamW starts right after dW_down (else with wg|wu)
    cudaEvent_t ev_join = nullptr;
    cudaEvent_t ev_fork[5] = {}, ev_ready[5] = {};  // side-stream hand-offs within a step
    std::vector<int64_t> layer_lo, layer_hi;  // owned experts' compact range per layer
    ncclComm_t comm = nullptr;
    // peers' parameter vectors mapped over NVLink (CUDA IPC), for the owner-set means
    std::vector<float*> peer_params;
    bool p2p_tried = false, p2p_ok = false;
    // fused expert exchange (sync_exchange): per-layer "means done" flags of this node
    // (exported by IPC with the parameters), the peers' flags, the cached task list
    uint32_t* sync_flags = nullptr;
    std::vector<uint32_t*> peer_flags;
    uint32_t** peer_flags_dev = nullptr;
    uint32_t sync_epoch = 0;
    spes_k::SyncTask* sync_tasks = nullptr;
    int n_sync_tasks = -1;  // -1: task list to (re)build
    int sync_max_src = 1;
    int* sync_ctr = nullptr;
    int* sync_layer_total = nullptr;
    double sync_mean_bytes = 0, sync_pull_bytes = 0;
    int32_t* barrier_buf = nullptr;
    int64_t launches = 0;

    // ownership
    std::vector<std::vector<int>> node_experts;  // node -> sorted experts
    std::vector<std::vector<int>> owners;        // expert -> ascending nodes
    std::vector<uint8_t> owned;                  // this node's mask [M]
    std::vector<int64_t> grad_off_host;          // [L*M] compact offset or -1
    int64_t G = 0;                               // compact trainable size
    // fused optimizer: owned experts' AdamW runs in the dW GEMM epilogues (their gradients
    // are never materialized); the standalone pass covers psi only. Off (default): the
    // gradients are materialized and one standalone pass updates everything. Both give
    // identical bits; the fused epilogue is issue/latency-bound at ~3.7 TB/s with the 8
    // epilogue warps that fit next to the MMA ring, so it does not beat the separate pass yet.
    bool fused_opt = false;
    // dSwiGLU epilogue of this context (SPES_DSWIGLU_TMA at creation; gemm_dswiglu): 4 =
    // 32-column pieces staged by TMA and written back in place, 3 buffers, 5 operand stages
    // (dH cfg2 641 -> 831 TFLOP/s, cfg5 1112 -> 1182); 0 direct loads; 1 / 2 64-column pieces
    // through the transpose slots (cost operand stages; only used for d <= 2048); 3 in place
    // with 2 buffers
    int dswiglu_variant = 4;
    // inner optimizer (LocalRoundConfig::inner, trainer.hpp:116-121): AdamW, or SGD
    // (theta -= lr * g, no moments; always the standalone pass)
    bool inner_sgd = false;
    spes_k::AdamScalars cur_adam{};  // this step's AdamW scalars (set before backward)
    spes_k::AdamMaps* adam_maps = nullptr;  // [L] TMA views for the staged fused optimizer
    // DiLoCo baseline: this rank's slice of the round-start global model,
    // its fp64 Nesterov buffer, and the exchange buffers (N x slice each)
    // device corpus: sequences x (S+1) tokens resident in HBM
    int32_t* corpus = nullptr;
    int64_t corpus_rows = 0, corpus_seq = 0;
    int64_t* d_rows = nullptr;
    int64_t d_rows_cap = 0;
    float *outer_theta = nullptr, *outer_recv = nullptr, *outer_gather = nullptr;
    double* outer_buf = nullptr;
    int64_t outer_slice = 0;
    bool outer_ready = false;
    spes_k::AdamScalars* d_adam = nullptr;  // device copy read by the optimizer kernels
    // the local step as one CUDA graph per (T, optimizer placement): the launch sequence
    // is host-static (group tables and tile counts live on the device), so it is captured
    // on the second step of a shape and replayed; profiling runs eagerly
    bool use_graph = true;
    cudaGraphExec_t step_graph = nullptr;
    int64_t graph_T = -1, graph_seen_T = -1;
    int graph_fused = -1;
    int64_t graph_launches = 0;
    std::vector<spes_k::AdamSeg> segs_host;

    DevMem persistent;  // params, shadows, optimizer state
    float* params = nullptr;
    bf16 *w1 = nullptr, *w2 = nullptr, *headB = nullptr;  // bf16 GEMM operand copies
    float *grads = nullptr, *m = nullptr, *v = nullptr;
    spes_k::AdamSeg* segs = nullptr;
    spes_k::AdamSeg* all_segs = nullptr;  // head + every expert (shadow refresh)
    int n_all_segs = 0;
    int64_t all_segs_total = 0;
    int64_t* grad_off_dev = nullptr;  // [L*M]
    int64_t adam_step = 0;

    // activations (sized for T_pad)
    DevMem act;
    int64_t T = 0, T_pad = 0, R_cap = 0, B = 0, S = 0;
    bool use_pairs = false;  // cta_group::2 GEMMs (256-row tiles)
    // layer 0's input h0 = emb[inputs] is never materialized: its consumers read the
    // (L2-resident) embedding rows through the token index
    bool virtual_h0 = true;
    int tr = 128;            // GEMM tile rows == expert row padding
    std::vector<float*> h;  // L+1 buffers [T_pad x d]
    std::vector<LayerBufs> layers;
    int32_t *tokens = nullptr, *inputs = nullptr, *targets = nullptr, *err = nullptr;
    bf16 *dyw = nullptr, *dgu = nullptr;
    float *dot_part = nullptr;
    double* loss_part = nullptr;
    int32_t* eg_scratch = nullptr;  // embedding-gradient bucketing (2V + 1 + T)
    // router weight gradient on the tensor cores (g_router = normed^T glog, MN-major pair
    // GEMM over the tokens, split K, then summed in split order into the gradient); set
    // at creation (M > 16)
    bool router_tc = false;
    bf16* glog_bf = nullptr;  // [T_pad x 128] bf16 glog, experts zero-padded to 128 columns
    CUtensorMap b_glog_mn;
    float* rg_part = nullptr;  // [rg_split][d][128]
    GemmGroup* rg_groups = nullptr;
    int32_t* rg_tiles = nullptr;
    int rg_split = 1, rg_max = 0;
    float *dxp = nullptr, *gw_part = nullptr, *glog = nullptr, *gnormed = nullptr, *gh = nullptr,
          *nr_partial = nullptr;
    bf16 *hL = nullptr, *dlog_bf = nullptr;
    float *head_logits = nullptr, *dlogits = nullptr, *diff = nullptr, *lse_head = nullptr;
    float *lse_all = nullptr, *probs_all = nullptr, *coeff_all = nullptr;
    double* d_losses = nullptr;
    GemmGroup* head_groups = nullptr;  // [2 + head_split]: fwd, dX, dW K-splits
    CUtensorMap* gu_maps = nullptr;    // [L] per layer's GU as {64 x 128} boxes (device memory)
    CUtensorMap* dsw_maps = nullptr;   // [L][2] GU {32 x 128} + dGU {32 x 32}, 64B swizzle
    int32_t* head_tiles = nullptr;     // [3]
    int head_max[3] = {0, 0, 0};
    int head_split = 1;
    float* head_dw_part = nullptr;
    CUtensorMap a_dyw, a_dgu, b_dgu_mn, b_dyw_mn, a_hL, b_headB_mn, a_dlog, b_headB, a_hL_mn,
        b_dlog_mn;
    int max_tiles[6] = {0, 0, 0, 0, 0, 0};

    // host staging
    int32_t* h_tokens = nullptr;
    int64_t h_tokens_cap = 0;
    double* h_losses = nullptr;
    // pinned staging of the merge's small host<->device transfers (async, no bounce copies)
    struct MergePin {
        double sim[64 * 64];
        int32_t peers[64 * 64];
        double coef[64];
        int64_t eo[64], vo[64];
        double disp[148 * 8];
    };
    MergePin* h_merge = nullptr;

    // sync / merge scratch
    DevMem scratch;
    float* psi_stage = nullptr;
    float* expert_stage = nullptr;
    int64_t expert_stage_cap = 0;
    double *gram_partial = nullptr, *sim = nullptr, *coef = nullptr, *disp_partial = nullptr;
    int32_t* peers_dev = nullptr;
    int64_t* layer_expert_offs = nullptr;  // [M] scratch
    int gram_chunks = 0;

    // live per-kernel-family timing with CUDA events on the context's stream
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> pending;  // (family, start event index)
    std::vector<std::string> fam_names;
    std::vector<double> fam_ms;
    std::vector<int64_t> fam_n;
};

namespace {

// Kernel launches are counted into the calling context for the duration of one API call.
// The thread-local pointer is restored when the call returns, so it never outlives the
// call: a destroyed context must not be written through by a later kernel-level call (that
// dangling increment once corrupted unrelated host memory between tests).
struct CounterScope {
    int64_t* prev;
    explicit CounterScope(spes_ctx* c) : prev(spes_k::g_launch_counter) {
        spes_k::g_launch_counter = &c->launches;
    }
    ~CounterScope() { spes_k::g_launch_counter = prev; }
    CounterScope(const CounterScope&) = delete;
    CounterScope& operator=(const CounterScope&) = delete;
};

void drop_graph(spes_ctx* c) {
    if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
    c->step_graph = nullptr;
    c->graph_T = c->graph_seen_T = -1;
}

// Sync plan: the primary owner of expert e computes its owner-set
// mean and distributes it. Primary = e / (M/N) when N | M and that node owns e (the
// contiguous balanced layout -> one in-place all-gather per layer), else the lowest
// owner (-> grouped broadcasts). Experts without owners keep their global value.
void sync_plan(int M, int N, const std::vector<std::vector<int>>& owners,
               std::vector<int>& primary, bool& balanced) {
    const int s_bal = (M % N == 0) ? M / N : 0;
    primary.assign(M, -1);
    balanced = s_bal > 0;
    for (int e = 0; e < M; ++e) {
        const auto& O = owners[e];
        if (O.empty()) {
            balanced = false;
            continue;
        }
        int p = O.front();
        if (s_bal && std::find(O.begin(), O.end(), e / s_bal) != O.end()) p = e / s_bal;
        primary[e] = p;
        if (!s_bal || p != e / s_bal) balanced = false;
    }
}

// Brackets the launches of one kernel family with CUDA events when profiling is on.
struct Prof {
    spes_ctx* c;
    int fam = -1;
    size_t i = 0;
    Prof(spes_ctx* ctx, const char* name) : c(ctx) {
        if (!c->prof) return;
        auto it = std::find(c->fam_names.begin(), c->fam_names.end(), name);
        if (it == c->fam_names.end()) {
            c->fam_names.push_back(name);
            c->fam_ms.push_back(0.0);
            c->fam_n.push_back(0);
            fam = static_cast<int>(c->fam_names.size()) - 1;
        } else {
            fam = static_cast<int>(it - c->fam_names.begin());
        }
        while (c->ev_pool.size() < c->ev_used + 2) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            c->ev_pool.push_back(e);
        }
        i = c->ev_used;
        c->ev_used += 2;
        cudaEventRecord(c->ev_pool[i], c->stream);
    }
    ~Prof() {
        if (fam < 0) return;
        cudaEventRecord(c->ev_pool[i + 1], c->stream);
        c->pending.push_back({fam, i});
    }
};

void prof_collect(spes_ctx* c) {
    if (c->pending.empty()) return;
    cudaStreamSynchronize(c->stream);
    for (auto& p : c->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev_pool[p.second], c->ev_pool[p.second + 1]);
        c->fam_ms[p.first] += ms;
        c->fam_n[p.first] += 1;
    }
    c->pending.clear();
    c->ev_used = 0;
}

void build_ownership_tables(spes_ctx* c) {
    const Layout& L = c->lay;
    c->owned.assign(L.M, 0);
    for (int e : c->node_experts[c->node]) c->owned[e] = 1;
    c->owners.assign(L.M, {});
    for (int n = 0; n < c->n_nodes; ++n)
        for (int e : c->node_experts[n]) c->owners[e].push_back(n);
    // compact trainable layout: psi, then owned experts (layer-major, ascending). The
    // segments also tell the optimizer which bf16 operand copy each element feeds
    // (kind 2: head -> headB, kind 1: expert -> W1/W2 slot).
    c->grad_off_host.assign(static_cast<size_t>(L.L) * L.M, -1);
    c->segs_host.clear();
    c->segs_host.push_back({0, 0, L.V * L.d, 0, 0});                          // emb
    c->segs_host.push_back({L.off_head(), L.off_head(), L.V * L.d, 2, 0});     // head
    c->segs_host.push_back({2 * L.V * L.d, 2 * L.V * L.d, L.psi() - 2 * L.V * L.d, 0, 0});
    int64_t off = L.psi();
    c->layer_lo.assign(L.L, 0);
    c->layer_hi.assign(L.L, 0);
    for (int l = 0; l < L.L; ++l) {
        c->layer_lo[l] = off;
        for (int j = 0; j < L.M; ++j)
            if (c->owned[j]) {
                c->grad_off_host[static_cast<size_t>(l) * L.M + j] = off;
                c->segs_host.push_back({L.off_expert(l, j), off, L.per_expert(), 1, l * L.M + j});
                off += L.per_expert();
            }
        c->layer_hi[l] = off;
    }
    c->G = off;
    // (re)allocate grads / moments
    if (c->grads) {
        cudaFree(c->grads);
        cudaFree(c->m);
        cudaFree(c->v);
        cudaFree(c->segs);
        auto& P = c->persistent.ptrs;
        P.erase(std::remove_if(P.begin(), P.end(),
                               [&](void* p) {
                                   return p == c->grads || p == c->m || p == c->v || p == c->segs;
                               }),
                P.end());
    }
    c->grads = c->persistent.alloc<float>(c->G);
    c->m = c->persistent.alloc<float>(c->G);
    c->v = c->persistent.alloc<float>(c->G);
    c->segs = c->persistent.alloc<spes_k::AdamSeg>(static_cast<int64_t>(c->segs_host.size()));
    ck(cudaMemcpy(c->segs, c->segs_host.data(), sizeof(spes_k::AdamSeg) * c->segs_host.size(),
                  cudaMemcpyHostToDevice),
       "segs");
    ck(cudaMemcpy(c->grad_off_dev, c->grad_off_host.data(), 8 * c->grad_off_host.size(),
                  cudaMemcpyHostToDevice),
       "grad_off");
    c->adam_step = 0;
    // TMA views of every layer's expert parameters and owned experts' moments (fused
    // optimizer, pair kernel): rows of f (wg / wu) and of d (wd) floats
    {
        std::vector<spes_k::AdamMaps> am(L.L);
        for (int l = 0; l < L.L; ++l) {
            const float* th = c->params + L.off_expert(l, 0);
            const int64_t nown = (c->layer_hi[l] - c->layer_lo[l]) / L.per_expert();
            const int64_t rows_m = std::max<int64_t>(1, 3 * nown);
            using spes_host::make_tmap_f32;
            am[l].th_f = make_tmap_f32(th, 3 * L.d * L.M, L.f, 32, 128);
            am[l].th_d = make_tmap_f32(th, 3 * L.f * L.M, L.d, 32, 128);
            am[l].m_f = make_tmap_f32(c->m + c->layer_lo[l], rows_m * L.d, L.f, 32, 128);
            am[l].v_f = make_tmap_f32(c->v + c->layer_lo[l], rows_m * L.d, L.f, 32, 128);
            am[l].m_d = make_tmap_f32(c->m + c->layer_lo[l], rows_m * L.f, L.d, 32, 128);
            am[l].v_d = make_tmap_f32(c->v + c->layer_lo[l], rows_m * L.f, L.d, 32, 128);
            am[l].th_base = th;
            am[l].mv_base = c->layer_lo[l];
        }
        if (!c->adam_maps) c->adam_maps = c->persistent.alloc<spes_k::AdamMaps>(std::max(1, L.L));
        ck(cudaMemcpy(c->adam_maps, am.data(), sizeof(spes_k::AdamMaps) * L.L,
                      cudaMemcpyHostToDevice),
           "adam maps");
    }
}

// optimizer segment tables: psi segments, then experts of 3df scalars each
spes_k::SegTable train_table(const spes_ctx* c) {
    return spes_k::SegTable{c->segs, 3, c->lay.psi(), c->lay.per_expert()};
}
spes_k::SegTable refresh_table(const spes_ctx* c) {  // head, then every expert
    return spes_k::SegTable{c->all_segs, 1, c->lay.V * c->lay.d, c->lay.per_expert()};
}

spes_k::Shadows shadows_of(const spes_ctx* c) {
    return spes_k::Shadows{c->w1, c->w2, c->headB, c->lay.d, c->lay.f};
}

// Every bf16 operand copy from the fp32 parameters (after load / sync / merge).
void refresh_shadows_all(spes_ctx* c) {
    spes_k::refresh_shadows(c->params, refresh_table(c), c->all_segs_total, shadows_of(c),
                            c->stream);
}

void ensure_activations(spes_ctx* c, int64_t B, int64_t S) {
    const int64_t T = B * S;
    if (T < 1) throw std::invalid_argument("batch: need B*S >= 1");
    if (T == c->T && c->T_pad > 0) {
        // same token count, other batch shape: the buffers fit (tokens holds 2T >= B(S+1)
        // ints) but the captured step splits inputs / targets with the old S
        if (B != c->B || S != c->S) drop_graph(c);
        c->B = B;
        c->S = S;
        return;
    }
    c->B = B;
    c->S = S;
    const Layout& L = c->lay;
    drop_graph(c);  // buffers move
    c->act.release();
    c->T = T;
    // cta_group::2 pair tiles (256 rows) whenever every GEMM M dimension allows it
    c->use_pairs = (L.d % 256 == 0) && (L.f % 256 == 0);
    c->tr = c->use_pairs ? 256 : 128;
    const int64_t tr = c->tr;
    const int bdiv = c->use_pairs ? 2 : 1;  // K-major B box rows per CTA = BN / bdiv
    c->T_pad = rup(T, tr);
    c->R_cap = rup(T * L.k + static_cast<int64_t>(L.M) * tr, tr);
    const int64_t Tp = c->T_pad, R = c->R_cap, d = L.d, f = L.f, V = L.V, M = L.M, k = L.k;
    DevMem& A = c->act;
    c->h.assign(L.L + 1, nullptr);
    for (auto& p : c->h) p = A.alloc<float>(Tp * d);
    c->tokens = A.alloc<int32_t>(2 * T);  // B(S+1) = T + B <= 2T for every shape of this T
    c->inputs = A.alloc<int32_t>(Tp);
    c->eg_scratch = A.alloc<int32_t>(2 * L.V + 1 + Tp);
    c->targets = A.alloc<int32_t>(Tp);
    c->err = A.alloc<int32_t>(1);
    c->layers.assign(L.L, LayerBufs{});
    const int64_t nchunks = (T + 255) / 256;
    c->lse_all = A.alloc<float>(L.L * Tp);
    c->probs_all = A.alloc<float>(L.L * Tp * M);
    c->coeff_all = A.alloc<float>(L.L * M);
    for (int l = 0; l < L.L; ++l) {
        LayerBufs& Y = c->layers[l];
        Y.logits = A.alloc<float>(Tp * M);
        Y.probs = c->probs_all + l * Tp * M;
        Y.topk_w = A.alloc<float>(Tp * k);
        Y.topk_idx = A.alloc<int32_t>(Tp * k);
        Y.lse_r = c->lse_all + l * Tp;
        Y.inv_rms = A.alloc<float>(Tp);
        Y.denom = A.alloc<float>(Tp);
        Y.chunk_counts = A.alloc<int32_t>(nchunks * M);
        Y.counts = A.alloc<int32_t>(M);
        Y.pad_off = A.alloc<int32_t>(M + 1);
        Y.lb_coeff = c->coeff_all + l * M;
        Y.slot_row = A.alloc<int32_t>(Tp * k);
        Y.row_token = A.alloc<int32_t>(R);
        Y.row_w = A.alloc<float>(R);
        Y.groups = A.alloc<GemmGroup>(6 * M);
        Y.tiles = A.alloc<int32_t>(6);
        Y.xp = A.alloc<bf16>(R * d);
        Y.gu = A.alloc<bf16>(R * 2 * f);
        Y.hact = A.alloc<bf16>(R * f);
        Y.y = A.alloc<float>(R * d);
        Y.normed_bf = A.alloc<bf16>(Tp * d);
        // padding rows stay zero (finite operands for the router-gradient GEMM)
        ck(cudaMemsetAsync(Y.normed_bf, 0, sizeof(bf16) * Tp * d, c->stream), "normed_bf");
        Y.grad_off = c->grad_off_dev + static_cast<int64_t>(l) * M;
        using spes_host::make_tmap_bf16;
        Y.a_normed_mn = make_tmap_bf16(Y.normed_bf, Tp, d, 64);
        Y.a_xp = make_tmap_bf16(Y.xp, R, d, 128);
        Y.a_hact = make_tmap_bf16(Y.hact, R, f, 128);
        Y.a_xp_mn = make_tmap_bf16(Y.xp, R, d, 64);
        Y.a_hact_mn = make_tmap_bf16(Y.hact, R, f, 64);
        Y.b_w1_mn = make_tmap_bf16(c->w1 + static_cast<int64_t>(l) * M * d * 2 * f, M * d, 2 * f, 64);
        Y.b_w2_mn = make_tmap_bf16(c->w2 + static_cast<int64_t>(l) * M * f * d, M * f, d, 64);
        Y.b_w2 = make_tmap_bf16(c->w2 + static_cast<int64_t>(l) * M * f * d, M * f, d,
                                bn_for(f) / bdiv);
        Y.b_w1 = make_tmap_bf16(c->w1 + static_cast<int64_t>(l) * M * d * 2 * f, M * d, 2 * f,
                                bn_for(d) / bdiv);
    }
    {  // the dSwiGLU epilogue stages its factor rows from GU by TMA: maps in device memory
        std::vector<CUtensorMap> gm(L.L);
        for (int l = 0; l < L.L; ++l)
            gm[l] = spes_host::make_tmap_bf16(c->layers[l].gu, R, 2 * f, 128);
        c->gu_maps = A.alloc<CUtensorMap>(L.L);
        ck(cudaMemcpy(c->gu_maps, gm.data(), sizeof(CUtensorMap) * L.L, cudaMemcpyHostToDevice),
           "gu maps");
    }
    c->dyw = A.alloc<bf16>(R * d);
    c->dgu = A.alloc<bf16>(R * 2 * f);
    {  // the in-place variant: 32-column factor pieces and the dGU stores
        std::vector<CUtensorMap> dm(2 * L.L);
        for (int l = 0; l < L.L; ++l) {
            dm[2 * l] = spes_host::make_tmap_bf16_sw64(c->layers[l].gu, R, 2 * f, 128);
            dm[2 * l + 1] = spes_host::make_tmap_bf16_sw64(c->dgu, R, 2 * f, 32);
        }
        c->dsw_maps = A.alloc<CUtensorMap>(2 * L.L);
        ck(cudaMemcpy(c->dsw_maps, dm.data(), sizeof(CUtensorMap) * 2 * L.L,
                      cudaMemcpyHostToDevice),
           "dswiglu maps");
    }
    c->dxp = A.alloc<float>(R * d);
    c->gw_part = A.alloc<float>(R);
    c->dot_part = A.alloc<float>(Tp * (d / 128));
    c->loss_part = A.alloc<double>((Tp / 256 + 1) * (2 + 2 * L.L));
    c->glog = A.alloc<float>(Tp * M);
    c->gnormed = A.alloc<float>(Tp * d);
    c->gh = A.alloc<float>(Tp * d);
    c->glog_bf = A.alloc<bf16>(Tp * 128);
    ck(cudaMemsetAsync(c->glog_bf, 0, sizeof(bf16) * Tp * 128, c->stream), "glog_bf");
    c->b_glog_mn = spes_host::make_tmap_bf16(c->glog_bf, Tp, 128, 64);
    {  // g_router: (d / tr) output tiles of 256 x 128, K (tokens) split to cover the SMs
        const int64_t tiles = d / tr;
        int64_t ns = std::max<int64_t>(1, (2 * 148 / bdiv + tiles - 1) / tiles);
        while (ns > 1 && (Tp % (64 * ns) != 0 || Tp / ns < 512)) --ns;
        c->rg_split = static_cast<int>(ns);
        c->rg_part = A.alloc<float>(ns * d * 128);
        c->rg_groups = A.alloc<GemmGroup>(ns);
        c->rg_tiles = A.alloc<int32_t>(1);
        std::vector<GemmGroup> rg(ns);
        int32_t ts = 0;
        for (int64_t sp = 0; sp < ns; ++sp) {
            GemmGroup& g = rg[sp];
            g.k0 = static_cast<int32_t>(sp * (Tp / ns));
            g.bk0 = g.k0;
            g.k_len = static_cast<int32_t>(Tp / ns);
            g.m_tiles = static_cast<int32_t>(d / tr);
            g.n_tiles = 1;
            g.out0 = c->rg_part + sp * d * 128;
            g.ldo = 128;
            g.tile_start = ts;
            ts += g.m_tiles;
        }
        c->rg_max = ts;
        ck(cudaMemcpy(c->rg_groups, rg.data(), sizeof(GemmGroup) * ns, cudaMemcpyHostToDevice),
           "router-gradient groups");
        ck(cudaMemcpy(c->rg_tiles, &ts, sizeof(ts), cudaMemcpyHostToDevice), "router-gradient tiles");
    }
    c->nr_partial = A.alloc<float>(spes_k::kNormRouterChunks * d * (M + 1));
    c->hL = A.alloc<bf16>(Tp * d);
    ck(cudaMemsetAsync(c->hL, 0, sizeof(bf16) * Tp * d, c->stream), "hL");  // padding rows
    c->head_logits = A.alloc<float>(Tp * V);
    c->dlog_bf = A.alloc<bf16>(Tp * V);
    c->diff = A.alloc<float>(Tp);
    c->lse_head = A.alloc<float>(Tp);
    c->d_losses = A.alloc<double>(8);
    c->d_adam = A.alloc<spes_k::AdamScalars>(1);
    // head dW = hL^T dlogits has only (d/128)*(V/BN) output tiles: split K (tokens)
    // so the grid covers the SMs; partials are summed in split order (deterministic).
    {
        const int64_t tiles = (d / tr) * (V / bn_for(V));
        int64_t ns = std::max<int64_t>(1, (2 * 148 / bdiv + tiles - 1) / tiles);
        while (ns > 1 && (Tp % (64 * ns) != 0 || Tp / ns < 512)) --ns;
        c->head_split = static_cast<int>(ns);
    }
    c->head_groups = A.alloc<GemmGroup>(2 + c->head_split);
    c->head_tiles = A.alloc<int32_t>(3);
    c->head_dw_part = c->head_split > 1 ? A.alloc<float>(c->head_split * d * V) : nullptr;
    using spes_host::make_tmap_bf16;
    c->a_dyw = make_tmap_bf16(c->dyw, R, d, 128);
    c->a_dgu = make_tmap_bf16(c->dgu, R, 2 * f, 128);
    c->b_dgu_mn = make_tmap_bf16(c->dgu, R, 2 * f, 64);
    c->b_dyw_mn = make_tmap_bf16(c->dyw, R, d, 64);
    c->a_hL = make_tmap_bf16(c->hL, Tp, d, 128);
    c->b_headB_mn = make_tmap_bf16(c->headB, d, V, 64);
    c->a_dlog = make_tmap_bf16(c->dlog_bf, Tp, V, 128);
    c->b_headB = make_tmap_bf16(c->headB, d, V, bn_for(d) / bdiv);
    c->a_hL_mn = make_tmap_bf16(c->hL, Tp, d, 64);
    c->b_dlog_mn = make_tmap_bf16(c->dlog_bf, Tp, V, 64);
    // head GEMM groups (static for a given T_pad)
    std::vector<GemmGroup> hg(2 + c->head_split);
    hg[0].k_len = static_cast<int32_t>(d);
    hg[0].m_tiles = static_cast<int32_t>(Tp / tr);
    hg[0].n_tiles = static_cast<int32_t>(V / bn_for(V));
    hg[0].out0 = c->head_logits;
    hg[0].ldo = V;
    hg[1].k_len = static_cast<int32_t>(V);
    hg[1].m_tiles = static_cast<int32_t>(Tp / tr);
    hg[1].n_tiles = static_cast<int32_t>(d / bn_for(d));
    hg[1].out0 = c->gh;
    hg[1].ldo = d;
    const int nsplit = c->head_split;
    int32_t ts = 0;
    for (int sp = 0; sp < nsplit; ++sp) {
        GemmGroup& g = hg[2 + sp];
        g.k0 = static_cast<int32_t>(sp * (Tp / nsplit));
        g.bk0 = g.k0;
        g.k_len = static_cast<int32_t>(Tp / nsplit);
        g.m_tiles = static_cast<int32_t>(d / tr);
        g.n_tiles = static_cast<int32_t>(V / bn_for(V));
        g.out0 = nsplit > 1 ? c->head_dw_part + sp * d * V
                       : c->grads + L.off_head();  // psi is first in the compact layout
        g.ldo = V;
        g.tile_start = ts;
        ts += g.m_tiles * g.n_tiles;
    }
    int32_t ht[3];
    for (int i = 0; i < 2; ++i) {
        ht[i] = hg[i].m_tiles * hg[i].n_tiles;
        c->head_max[i] = ht[i];
    }
    ht[2] = ts;
    c->head_max[2] = ts;
    ck(cudaMemcpy(c->head_groups, hg.data(), sizeof(GemmGroup) * hg.size(), cudaMemcpyHostToDevice),
       "head groups");
    ck(cudaMemcpy(c->head_tiles, ht, sizeof(ht), cudaMemcpyHostToDevice), "head tiles");
    // upper bounds of routed GEMM tile counts
    const int64_t mt_max = (T * k) / tr + M;
    c->max_tiles[0] = static_cast<int>(mt_max * (2 * f / 256));
    c->max_tiles[1] = static_cast<int>(mt_max * (d / bn_for(d)));
    c->max_tiles[2] = static_cast<int>(mt_max * (f / bn_for(f)));
    c->max_tiles[3] = static_cast<int>(mt_max * (d / bn_for(d)));
    const int64_t no = static_cast<int64_t>(std::count(c->owned.begin(), c->owned.end(), 1));
    c->max_tiles[4] = static_cast<int>(no * (d / tr) * (2 * f / 256));
    c->max_tiles[5] = static_cast<int>(no * (f / tr) * (d / bn_for(d)));
}

// gradient seeds of the reverse tape (model.hpp:365-372): float arithmetic as the reference
struct Seeds {
    float inv_T, inv_L, c_ce, c_lb, c_mz, c_z, g_lbsum, g_mzsum, g_s2, g_ssum, g_s;
};
Seeds seeds_for(const spes_ctx* c) {
    Seeds s;
    volatile float one = 1.f;
    s.inv_T = one / static_cast<float>(c->T);
    s.inv_L = one / static_cast<float>(c->lay.L);
    s.c_ce = static_cast<float>(c->cfg.coeff_ce);
    s.c_lb = static_cast<float>(c->cfg.coeff_lb);
    s.c_mz = static_cast<float>(c->cfg.coeff_moe_z);
    s.c_z = static_cast<float>(c->cfg.coeff_z);
    const float g_z = s.c_z * one, g_mz = s.c_mz * one, g_lb = s.c_lb * one, g_ce = s.c_ce * one;
    s.g_lbsum = s.inv_L * g_lb;
    s.g_mzsum = s.inv_L * g_mz;
    s.g_s2 = s.inv_T * g_z;
    s.g_ssum = s.inv_T * g_ce;
    s.g_s = s.inv_T * s.g_mzsum;
    return s;
}

// Off-critical-path work on the low-priority side stream (not while profiling: the
// per-family event timings need one serial stream).
bool use_side(const spes_ctx* c) { return c->overlap_opt && !c->prof; }
// owned experts' optimizer step inside the dW GEMM epilogues (AdamW only)
bool fused(const spes_ctx* c) { return c->fused_opt && !c->inner_sgd; }
// owned experts' AdamW there, right after their dW GEMMs
bool split_opt(const spes_ctx* c) {
    return use_side(c) && !fused(c) && c->G > c->lay.psi();
}

void forward_backward(spes_ctx* c) {
    const Layout& L = c->lay;
    cudaStream_t st = c->stream;
    const int64_t T = c->T, Tp = c->T_pad, R = c->R_cap, d = L.d, f = L.f, V = L.V;
    const int M = L.M, k = L.k;
    const Seeds sd = seeds_for(c);
    float* P = c->params;
    spes_k::gemm_set_pair_mode(c->use_pairs);
    // input rows of layer l: layer 0 reads emb[inputs[t]] in place (virtual_h0)
    auto hsrc = [&](int l) -> const float* {
        return (l == 0 && c->virtual_h0) ? P + L.off_emb() : c->h[l];
    };
    auto hmap = [&](int l) -> const int32_t* { return (l == 0 && c->virtual_h0) ? c->inputs : nullptr; };
    // side-stream hand-offs: fork(i) starts side work after everything enqueued on st so
    // far; ready(i) marks it done; need(i) makes st wait for it. Serial when profiling.
    const bool side = use_side(c);
    cudaStream_t ss = side ? c->side : st;
    auto fork = [&](int i) {
        if (!side) return;
        ck(cudaEventRecord(c->ev_fork[i], st), "event");
        ck(cudaStreamWaitEvent(ss, c->ev_fork[i], 0), "wait");
    };
    auto ready = [&](int i) {
        if (side) ck(cudaEventRecord(c->ev_ready[i], ss), "event");
    };
    auto need = [&](int i) {
        if (side) ck(cudaStreamWaitEvent(st, c->ev_ready[i], 0), "wait");
    };
#define PROF(name) Prof _prof_##__LINE__(c, name)
    {
        PROF("embed_gather");
        spes_k::embed_gather(P + L.off_emb(), c->tokens, c->B, c->S, d, c->ulay.V,
                             c->virtual_h0 ? nullptr : c->h[0], c->inputs,
                             c->targets, c->err, st);
    }
    bool eg_planned = false;
    {  // token bucketing for the embedding gradient: only needs the inputs
        PROF("embed_grad");
        fork(0);
        eg_planned = spes_k::embed_grad_plan(c->inputs, T, V, c->eg_scratch, ss);
        ready(0);
    }
    for (int l = 0; l < L.L; ++l) {
        LayerBufs& Y = c->layers[l];
        {
            PROF("router_fwd");
            spes_k::router_forward(hsrc(l), hmap(l), P + L.off_norm(l), P + L.off_router(l), T, d,
                                   c->ulay.d, M, k,
                                   c->cfg.renormalize_after_topk, c->cfg.rms_eps, c->expf_variant,
                                   nullptr, Y.normed_bf, Y.logits, Y.probs, Y.topk_idx,
                                   Y.topk_w, Y.lse_r, Y.inv_rms, Y.denom, st);
        }
        {
            PROF("route_plan");
            spes_k::RoutePlan rp{Y.chunk_counts, Y.counts, Y.pad_off, Y.lb_coeff, Y.slot_row,
                                 Y.row_token, Y.row_w, Y.groups, Y.tiles};
            spes_k::GroupBases gb{Y.gu, Y.y, c->dgu, c->dxp, c->grads, Y.grad_off, d, f,
                                  bn_for(d), bn_for(f), bn_for(d), bn_for(d), c->tr,
                                  P + L.off_expert(l, 0), l * M, fused(c) ? 1 : 0};
            spes_k::route_plan(Y.topk_idx, Y.topk_w, T, M, k, R, rp, gb, st);
        }
        {
            PROF("permute");  // TMA-staged row scatter (dispatch)
            spes_k::permute_rows_tma(Y.normed_bf, d, Y.slot_row, Y.row_token, Y.pad_off + M, T, k,
                                     Y.xp, st);
        }
        {
            PROF("gemm_fwd_gate_up");
            spes_k::gemm_swiglu(Y.a_xp, Y.b_w1_mn, Y.groups + 0 * M, M, Y.tiles + 0, c->max_tiles[0],
                                Y.hact, f, st);
        }
        {
            PROF("gemm_fwd_down");
            spes_k::gemm_store_f32(bn_for(d), spes_k::GemmMajor::KMN, Y.a_hact, Y.b_w2_mn,
                                   Y.groups + 1 * M, M, Y.tiles + 1,
                                   c->max_tiles[1], st);
        }
        {
            PROF("combine_fwd");
            spes_k::combine_forward(hsrc(l), hmap(l), Y.y, Y.slot_row, Y.topk_idx, Y.topk_w, T, d, k,
                                    l + 1 == L.L ? nullptr : c->h[l + 1],
                                    l + 1 == L.L ? c->hL : nullptr, st);
        }
    }
    {
        PROF("head_fwd");
        if (V == 256 && c->ulay.V == V) {  // softmax-CE in the GEMM epilogue: no fp32 logits
            spes_k::gemm_head_ce(c->a_hL, c->b_headB_mn, c->head_groups + 0, 1, c->head_tiles + 0,
                                 c->head_max[0], c->targets, T, sd.g_s2, sd.g_ssum, c->dlog_bf, c->diff, c->lse_head, st);
        } else {
            spes_k::gemm_store_f32(bn_for(V), spes_k::GemmMajor::KMN, c->a_hL, c->b_headB_mn,
                                   c->head_groups + 0, 1, c->head_tiles + 0, c->head_max[0], st);
        }
    }
    {
        PROF("head_ce_losses");
        if (V != 256 || c->ulay.V != V)
            spes_k::head_ce(c->head_logits, c->targets, T, Tp, V, c->ulay.V, sd.g_s2,
                            sd.g_ssum, c->dlog_bf, c->diff, c->lse_head, st);
        fork(1);  // loss scalars: read by the host and by the optimizer's finite-loss guard
        spes_k::losses_reduce(c->diff, c->lse_head, c->lse_all, c->probs_all, c->coeff_all, T, Tp,
                              L.L, M, sd.inv_T, sd.inv_L, sd.c_ce, sd.c_lb, sd.c_mz, sd.c_z,
                              c->err, c->loss_part, c->d_losses, ss);
        ready(1);
    }
    // ---- backward ----
    {
        PROF("head_bwd");
        spes_k::gemm_store_f32(bn_for(d), spes_k::GemmMajor::KK, c->a_dlog, c->b_headB,
                               c->head_groups + 1, 1,
                               c->head_tiles + 1, c->head_max[1], st);
        spes_k::gemm_store_f32(bn_for(V), spes_k::GemmMajor::MNMN, c->a_hL_mn, c->b_dlog_mn,
                               c->head_groups + 2,
                               c->head_split, c->head_tiles + 2, c->head_max[2], st);
        if (c->head_split > 1)
            spes_k::splitk_reduce(c->head_dw_part, c->head_split, d * V,
                                  c->grads + L.off_head(), st);
    }
    for (int l = L.L - 1; l >= 0; --l) {
        LayerBufs& Y = c->layers[l];
        {
            PROF("combine_bwd");
            // token-ordered rows once the upstream gradient (T x d fp32) outgrows L2's
            // reach (cfg5: 0.69 -> 0.80 of HBM); expert-major rows otherwise (cfg2: 0.74
            // token-ordered 0.62)
            const bool tok_order = 4 * T * d > (int64_t(64) << 20);
            spes_k::combine_backward(c->gh, Y.y, Y.row_token, Y.row_w, Y.pad_off + M, R, d, c->dyw,
                                     c->gw_part, st, tok_order ? Y.slot_row : nullptr, Y.topk_w,
                                     T, k);
        }
        {  // the router's per-token scalar chain only needs the gate-weight gradients: it
           // runs beside the expert GEMMs
            PROF("router_bwd");
            fork(2);
            spes_k::router_scalar_backward(Y.probs, Y.lse_r, Y.denom, Y.topk_idx, Y.slot_row,
                                           c->gw_part, Y.lb_coeff, T, M, k,
                                           c->cfg.renormalize_after_topk, sd.g_lbsum, sd.g_s,
                                           c->glog, c->router_tc ? c->glog_bf : nullptr, ss);
            ready(2);
        }
        const bool unfused_dw = c->max_tiles[4] > 0 && !fused(c);
        // owned experts' AdamW for the weights of this layer whose gradients are final and
        // whose bf16 operand copies the remaining GEMMs no longer read: wd (sub = 2) after
        // dW_down (dH read W2 before), wg|wu (sub = 0) after dW_gu (dX read W1 before)
        auto expert_adamw = [&](int sub, int ev) {
            if (!split_opt(c)) return;
            const int64_t df = d * f, per = 3 * df;
            const int nown = static_cast<int>((c->layer_hi[l] - c->layer_lo[l]) / per);
            if (!c->early_wd && sub == 2) return;
            const int64_t off = sub == 2 ? 2 * df : 0;
            const int64_t len = sub == 2 ? df : (c->early_wd ? 2 * df : per);
            if (nown == 0) return;
            fork(ev);
            const int seg0 = 3 + static_cast<int>((c->layer_lo[l] - c->lay.psi()) / per);
            spes_k::adamw_pieces(c->params, c->grads, c->m, c->v, train_table(c), seg0, nown, off,
                                 len, c->d_adam, shadows_of(c), c->d_losses, ss);
        };
        {
            PROF("gemm_bwd_dh");
            spes_k::gemm_dswiglu(bn_for(f), c->a_dyw, Y.b_w2, Y.groups + 2 * M, M, Y.tiles + 2,
                                 c->max_tiles[2], Y.gu, f,
                                 d <= 2048 ? c->gu_maps + l : nullptr, c->dsw_maps + 2 * l,
                                 c->dswiglu_variant, st);
        }
        if (unfused_dw) {
            {
                PROF("gemm_bwd_dw_down");
                spes_k::gemm_store_f32(bn_for(d), spes_k::GemmMajor::MNMN, Y.a_hact_mn,
                                       c->b_dyw_mn, Y.groups + 5 * M, M,
                                       Y.tiles + 5, c->max_tiles[5], st);
            }
            expert_adamw(2, 3);
        }
        {
            PROF("gemm_bwd_dx");
            spes_k::gemm_store_f32(bn_for(d), spes_k::GemmMajor::KK, c->a_dgu, Y.b_w1,
                                   Y.groups + 3 * M, M, Y.tiles + 3,
                                   c->max_tiles[3], st);
        }
        if (c->max_tiles[4] > 0 && fused(c)) {
            need(1);  // the epilogues' finite-loss guard reads the loss scalars
            // owned experts: dW and MaskedAdamW in one pass (no gradient materialized)
            const spes_k::Shadows sh = shadows_of(c);
            const spes_k::AdamEpi ae{c->d_adam, c->m, c->v, sh.w1, sh.w2, d, f, c->d_losses};
            {
                PROF("gemm_bwd_dw_gate_up+adamw");
                spes_k::gemm_adamw_w1(Y.a_xp_mn, c->b_dgu_mn, Y.groups + 4 * M, M, Y.tiles + 4,
                                      c->max_tiles[4], ae, st, c->adam_maps, M);
            }
            {
                PROF("gemm_bwd_dw_down+adamw");
                spes_k::gemm_adamw_w2(bn_for(d), Y.a_hact_mn, c->b_dyw_mn, Y.groups + 5 * M, M,
                                      Y.tiles + 5, c->max_tiles[5], ae, st, c->adam_maps, M);
            }
        } else if (unfused_dw) {
            {
                PROF("gemm_bwd_dw_gate_up");
                spes_k::gemm_grad_w1(Y.a_xp_mn, c->b_dgu_mn, Y.groups + 4 * M, M, Y.tiles + 4,
                                     c->max_tiles[4], st);
            }
            expert_adamw(0, 4);
        }
        {
            PROF("router_bwd");
            need(2);  // glog (and, earlier on the side stream, the loss scalars)
            spes_k::normed_grad(hsrc(l), hmap(l), P + L.off_norm(l), P + L.off_router(l),
                                Y.slot_row, c->dxp, T, d, M, k, c->glog, c->gnormed, c->dot_part,
                                st);
        }
        {
            PROF("norm_router_grads");  // + rmsnorm backward into gh
            spes_k::norm_router_grads(hsrc(l), hmap(l), P + L.off_norm(l), c->gnormed, c->glog,
                                      Y.inv_rms, T, d, c->ulay.d, c->router_tc ? 0 : M,
                                      c->nr_partial, c->grads + L.off_norm(l),
                                      c->grads + L.off_router(l), c->dot_part, c->gh, st);
        }
        if (c->router_tc) {
            PROF("router_grad_gemm");  // g_router = normed^T glog (bf16 operands, fp32 sums)
            spes_k::gemm_store_f32(128, spes_k::GemmMajor::MNMN, Y.a_normed_mn, c->b_glog_mn,
                                   c->rg_groups, c->rg_split, c->rg_tiles, c->rg_max, st);
            spes_k::router_grad_reduce(c->rg_part, c->rg_split, d, M, c->grads + L.off_router(l),
                                       st);
        }
    }
    {
        PROF("embed_grad");
        if (eg_planned) need(0);
        spes_k::embed_grad_apply(c->inputs, c->gh, T, d, V, c->grads + L.off_emb(), c->eg_scratch,
                                 st);
    }
}

// MaskedAdamW::step scalars (trainer.hpp:68-84): bias corrections in double, cast to float.
// Called before the backward so the fused dW epilogues can apply the step.
void optimizer_begin(spes_ctx* c, const spes_adamw_cfg* o) {
    if (c->inner_sgd) {  // trainer.hpp:197-204: float(lr), no optimizer state
        c->cur_adam = spes_k::AdamScalars{};
        c->cur_adam.lr = static_cast<float>(o->lr);
        c->cur_adam.sgd = 1;
        ck(cudaMemcpyAsync(c->d_adam, &c->cur_adam, sizeof(c->cur_adam), cudaMemcpyHostToDevice,
                           c->stream),
           "sgd scalars");
        return;
    }
    c->adam_step += 1;
    const float bc1 = 1.f - static_cast<float>(std::pow(o->beta1, static_cast<double>(c->adam_step)));
    const float bc2 = 1.f - static_cast<float>(std::pow(o->beta2, static_cast<double>(c->adam_step)));
    const float b1 = static_cast<float>(o->beta1), b2 = static_cast<float>(o->beta2);
    volatile float one = 1.f;
    const float omb1 = one - b1, omb2 = one - b2;
    c->cur_adam = spes_k::AdamScalars{static_cast<float>(o->lr), b1, b2, omb1, omb2,
                                      static_cast<float>(o->eps),
                                      static_cast<float>(o->weight_decay), bc1, bc2};
    ck(cudaMemcpyAsync(c->d_adam, &c->cur_adam, sizeof(c->cur_adam), cudaMemcpyHostToDevice,
                       c->stream),
       "adam scalars");
}

// The rest of the step: psi (and, unfused and not split off, the owned experts) after
// the backward; then the side stream joins.
void optimizer_finish(spes_ctx* c) {
    PROF("adamw");
    const bool split = split_opt(c);
    // psi: the table's 3 leading segments; then the owned experts
    const int nseg = fused(c) || split ? 3 : static_cast<int>(c->segs_host.size());
    spes_k::adamw(c->params, c->grads, c->m, c->v, train_table(c), 0, nseg, c->d_adam,
                  shadows_of(c), c->d_losses, c->stream);
    if (use_side(c)) {  // everything enqueued on the side stream this step
        ck(cudaEventRecord(c->ev_join, c->side), "event");
        ck(cudaStreamWaitEvent(c->stream, c->ev_join, 0), "wait");
    }
}

void validate_tokens(const spes_ctx* c, const int32_t* tokens, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= c->ulay.V)
            throw std::out_of_range("batch: token id out of vocabulary");
}

void upload_tokens(spes_ctx* c, const int32_t* tokens, int64_t n) {
    if (n > c->h_tokens_cap) {
        if (c->h_tokens) cudaFreeHost(c->h_tokens);
        ck(cudaMallocHost(&c->h_tokens, sizeof(int32_t) * n), "cudaMallocHost");
        c->h_tokens_cap = n;
    }
    std::memcpy(c->h_tokens, tokens, sizeof(int32_t) * n);
    ck(cudaMemcpyAsync(c->tokens, c->h_tokens, sizeof(int32_t) * n, cudaMemcpyHostToDevice,
                       c->stream),
       "H2D tokens");
}

// The device status word (c->err): bit 0 an out-of-vocabulary token id (set by the token
// split), bit 1 a non-finite loss (set by the loss reduction). It is sticky: once set, no
// later step applies an update (spes_dev::loss_ok) until the host reports and clears it,
// which ends the round with the reference's exception (model.hpp:280-281: out_of_range
// before any update; trainer.hpp:166-167: runtime_error, no update).
void raise_status(spes_ctx* c, int32_t st, const std::string& where) {
    if (!st) return;
    ck(cudaMemsetAsync(c->err, 0, 4, c->stream), "clear status");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (st & 1) throw std::out_of_range("batch: token id out of vocabulary" + where);
    throw std::runtime_error("local_round: non-finite loss" + where);
}

// losses of the last step (one D2H with its status word); reports a bad step
void read_losses(spes_ctx* c, spes_losses* out) {
    ck(cudaMemcpyAsync(c->h_losses, c->d_losses, sizeof(double) * 6, cudaMemcpyDeviceToHost,
                       c->stream),
       "D2H losses");
    ck(cudaStreamSynchronize(c->stream), "step");
    out->total = c->h_losses[0];
    out->ce = c->h_losses[1];
    out->lb = c->h_losses[2];
    out->moe_z = c->h_losses[3];
    out->z = c->h_losses[4];
}

// Steps run without reading their losses (device tokens, losses == NULL) are checked when
// the round ends: at the next sync, round start or parameter read.
void check_status(spes_ctx* c, const char* where) {
    if (c->T == 0 || !c->err) return;
    int32_t st = 0;
    ck(cudaMemcpyAsync(&st, c->err, 4, cudaMemcpyDeviceToHost, c->stream), "D2H status");
    ck(cudaStreamSynchronize(c->stream), "sync");
    raise_status(c, st, where);
}

void local_step_impl(spes_ctx* c, int64_t B, int64_t S, const spes_adamw_cfg* opt,
                     spes_losses* losses) {
    optimizer_begin(c, opt);
    // forward + backward (fused: owned experts updated unless the loss is non-finite) and
    // the optimizer pass (device-side non-finite check), eagerly or as a replayed graph
    const bool graph = c->use_graph && !c->prof;
    if (graph && c->step_graph && c->graph_T == c->T && c->graph_fused == (fused(c) ? 1 : 0)) {
        ck(cudaGraphLaunch(c->step_graph, c->stream), "graph launch");
        c->launches += c->graph_launches;
    } else if (graph && c->graph_seen_T == c->T) {  // second step of this shape: capture
        drop_graph(c);
        const int64_t before = c->launches;
        ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "capture");
        forward_backward(c);
        optimizer_finish(c);
        cudaGraph_t g = nullptr;
        ck(cudaStreamEndCapture(c->stream, &g), "end capture");
        ck(cudaGraphInstantiate(&c->step_graph, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        c->graph_launches = c->launches - before;
        c->launches = before + c->graph_launches;
        c->graph_T = c->T;
        c->graph_fused = fused(c) ? 1 : 0;
        ck(cudaGraphLaunch(c->step_graph, c->stream), "graph launch");
    } else {
        forward_backward(c);
        optimizer_finish(c);
        c->graph_seen_T = c->T;
    }
    if (losses) {
        read_losses(c, losses);
        const int32_t st = static_cast<int32_t>(c->h_losses[5]);
        if (st) {  // no update was applied (this step, or any since the bad one)
            if (!c->inner_sgd) c->adam_step -= 1;
            raise_status(c, st, "");
        }
    }
    (void)B;
    (void)S;
}

}  // namespace

// ============================ C ABI ============================
extern "C" {

const char* spes_last_error(void) { return g_last_error.c_str(); }

spes_status spes_validate_cfg(const spes_model_cfg* cfg) {
    return guard([&] { validate_cfg(cfg); });
}

int64_t spes_param_count(const spes_model_cfg* cfg) { return layout_of(cfg).total(); }

spes_status spes_block_offsets(const spes_model_cfg* cfg, int64_t* offsets, int32_t* n_out) {
    return guard([&] {
        Layout L = layout_of(cfg);
        std::vector<int64_t> o;
        o.push_back(L.off_emb());
        o.push_back(L.off_head());
        for (int l = 0; l < L.L; ++l) {
            o.push_back(L.off_norm(l));
            o.push_back(L.off_router(l));
        }
        for (int l = 0; l < L.L; ++l)
            for (int j = 0; j < L.M; ++j)
                for (int w = 0; w < 3; ++w) o.push_back(L.off_expert(l, j) + w * L.d * L.f);
        if (offsets) std::copy(o.begin(), o.end(), offsets);
        if (n_out) *n_out = static_cast<int32_t>(o.size());
    });
}

spes_status spes_param_partition(const spes_model_cfg* cfg, int32_t n, int32_t* node_offsets,
                                 int32_t* experts) {
    return guard([&] {
        const int m = cfg->experts_total;
        if (n < 1 || n > m) throw std::invalid_argument("partition: need 1 <= N <= M (no empty nodes)");
        int base = m / n, extra = m % n, next = 0;
        node_offsets[0] = 0;
        for (int i = 0; i < n; ++i) {
            int take = base + (i < extra ? 1 : 0);
            for (int j = 0; j < take; ++j) experts[next] = next, ++next;
            node_offsets[i + 1] = next;
        }
    });
}

double spes_lr_at(double peak, double min_frac, int64_t warmup, int64_t total, int64_t step) {
    if (warmup > 0 && step < warmup) return peak * static_cast<double>(step + 1) / static_cast<double>(warmup);
    double lo = peak * min_frac;
    int64_t span = total - warmup;
    if (span <= 0) return peak;
    double progress = static_cast<double>(step - warmup) / static_cast<double>(span);
    progress = std::min(1.0, std::max(0.0, progress));
    return lo + (peak - lo) * 0.5 * (1.0 + std::cos(M_PI * progress));
}

spes_status spes_sync_plan(int32_t experts_total, int32_t n_nodes, const int32_t* node_offsets,
                           const int32_t* experts, int32_t* primary_out, int32_t* balanced_out) {
    return guard([&] {
        if (n_nodes < 1 || experts_total < 1) throw std::invalid_argument("sync_plan: bad sizes");
        std::vector<std::vector<int>> owners(experts_total);
        for (int n = 0; n < n_nodes; ++n)
            for (int q = node_offsets[n]; q < node_offsets[n + 1]; ++q) {
                if (experts[q] < 0 || experts[q] >= experts_total)
                    throw std::invalid_argument("ownership: expert id out of range");
                owners[experts[q]].push_back(n);
            }
        std::vector<int> primary;
        bool balanced = false;
        sync_plan(experts_total, n_nodes, owners, primary, balanced);
        std::copy(primary.begin(), primary.end(), primary_out);
        *balanced_out = balanced ? 1 : 0;
    });
}

int32_t spes_merge_at(const spes_merge_sched* s, int32_t round) {
    return s->warmup_rounds > 0 && round < s->warmup_rounds && s->interval > 0 &&
           round % s->interval == 0;
}

spes_status spes_alpha_at(const spes_merge_sched* s, int32_t round, double* alpha) {
    return guard([&] {
        if (round < 0) throw std::invalid_argument("alpha_at: negative round");
        if (s->warmup_rounds <= 0) {
            *alpha = 0.0;
            return;
        }
        double frac = 1.0 - static_cast<double>(round) / static_cast<double>(s->warmup_rounds);
        *alpha = s->alpha0 * std::max(0.0, frac);
    });
}

spes_status spes_nccl_unique_id(void* out128) {
    return guard([&] {
        ncclUniqueId id;
        ckn(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out128, &id, sizeof(id));
    });
}

spes_status spes_create(const spes_model_cfg* cfg, int32_t node, int32_t n_nodes,
                        int32_t cuda_device, const void* nccl_id, spes_ctx** out) {
    return guard([&] {
        validate_cfg(cfg);
        if (n_nodes < 1 || node < 0 || node >= n_nodes)
            throw std::invalid_argument("worker: node id out of range");
        if (n_nodes > 1 && !nccl_id) throw std::invalid_argument("nccl id required when n_nodes > 1");
        auto c = std::make_unique<spes_ctx>();
        c->cfg = *cfg;
        const spes_model_cfg dcfg = device_cfg(cfg);
        c->lay = layout_of(&dcfg);
        c->ulay = layout_of(cfg);
        c->padded = c->lay.total() != c->ulay.total();
        c->node = node;
        c->n_nodes = n_nodes;
        c->device = cuda_device;
        ck(cudaSetDevice(cuda_device), "cudaSetDevice");
        CounterScope counter_scope(c.get());
        int prio_lo = 0, prio_hi = 0;
        ck(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priorities");
        ck(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi), "stream");
        ck(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, prio_lo), "stream");
        ck(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming), "event");
        for (int i = 0; i < 5; ++i) {
            ck(cudaEventCreateWithFlags(&c->ev_fork[i], cudaEventDisableTiming), "event");
            ck(cudaEventCreateWithFlags(&c->ev_ready[i], cudaEventDisableTiming), "event");
        }
        if (const char* e = std::getenv("SPES_OPT_OVERLAP")) c->overlap_opt = std::atoi(e) != 0;
        if (const char* e = std::getenv("SPES_FUSED_OPT")) c->fused_opt = std::atoi(e) != 0;
        if (const char* e = std::getenv("SPES_EARLY_WD")) c->early_wd = std::atoi(e) != 0;
        if (const char* e = std::getenv("SPES_STEP_GRAPH")) c->use_graph = std::atoi(e) != 0;
        // the CUDA-core kernel re-streams h once per 16 experts: above 16 the tensor-core
        // GEMM wins (cfg5 norm+router gradients 182 -> 66 ms per round), at 16 it does not
        // (cfg2 3.2 -> 4.1 ms)
        c->router_tc = c->lay.M > 16;
        if (const char* e = std::getenv("SPES_ROUTER_TC")) c->router_tc = std::atoi(e) != 0;
        if (const char* e = std::getenv("SPES_DSWIGLU_TMA"))  // 0 direct, else the variant (1-4)
            c->dswiglu_variant = std::max(0, std::min(4, std::atoi(e)));
        if (const char* e = std::getenv("SPES_ADAM_BG")) {  // "threads,tiles,per_sm,u"
            int th = 64, ti = 16, ps = 0, u = 2;
            if (std::sscanf(e, "%d,%d,%d,%d", &th, &ti, &ps, &u) >= 1 && th >= 32 && th <= 256 &&
                th % 32 == 0)
                spes_k::adamw_background_shape(th, ti < 1 ? 1 : ti, ps < 0 ? 0 : ps, u);
        }
        c->expf_variant = spes_expf::host_variant_from(&expf);
        spes_k::gemm_prepare(cuda_device);
        const Layout& L = c->lay;
        DevMem& P = c->persistent;
        c->params = P.alloc<float>(L.total());
        const int64_t slots = static_cast<int64_t>(L.L) * L.M;
        c->w1 = P.alloc<bf16>(slots * L.d * 2 * L.f);
        c->w2 = P.alloc<bf16>(slots * L.f * L.d);
        c->headB = P.alloc<bf16>(L.d * L.V);
        c->grad_off_dev = P.alloc<int64_t>(slots);
        {  // refresh table: head + every expert, indexed contiguously
            std::vector<spes_k::AdamSeg> all;
            int64_t off = 0;
            all.push_back({L.off_head(), off, L.V * L.d, 2, 0});
            off += L.V * L.d;
            for (int l = 0; l < L.L; ++l)
                for (int j = 0; j < L.M; ++j) {
                    all.push_back({L.off_expert(l, j), off, L.per_expert(), 1, l * L.M + j});
                    off += L.per_expert();
                }
            c->n_all_segs = static_cast<int>(all.size());
            c->all_segs_total = off;
            c->all_segs = P.alloc<spes_k::AdamSeg>(static_cast<int64_t>(all.size()));
            ck(cudaMemcpy(c->all_segs, all.data(), sizeof(spes_k::AdamSeg) * all.size(),
                          cudaMemcpyHostToDevice),
               "all segs");
        }
        ck(cudaMallocHost(&c->h_losses, sizeof(double) * 8), "pinned losses");
        // default ownership: param_partition (model.hpp:466-477) when N <= M, else all
        c->node_experts.assign(n_nodes, {});
        if (n_nodes <= L.M) {
            int base = L.M / n_nodes, extra = L.M % n_nodes, next = 0;
            for (int i = 0; i < n_nodes; ++i) {
                int take = base + (i < extra ? 1 : 0);
                for (int j = 0; j < take; ++j) c->node_experts[i].push_back(next++);
            }
        } else {
            throw std::invalid_argument("partition: need 1 <= N <= M (no empty nodes)");
        }
        build_ownership_tables(c.get());
        if (n_nodes > 1) {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            ckn(ncclCommInitRank(&c->comm, n_nodes, id, node), "ncclCommInitRank");
        }
        *out = c.release();
    });
}

void spes_destroy(spes_ctx* c) {
    if (c) drop_graph(c);
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->side) cudaStreamSynchronize(c->side);  // normally joined into stream at step end
    if (spes_k::g_launch_counter == &c->launches) spes_k::g_launch_counter = nullptr;
    for (float* p : c->peer_params)
        if (p) cudaIpcCloseMemHandle(p);
    for (size_t n = 0; n < c->peer_flags.size(); ++n)
        if (c->peer_flags[n] && static_cast<int>(n) != c->node) cudaIpcCloseMemHandle(c->peer_flags[n]);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->h_tokens) cudaFreeHost(c->h_tokens);
    if (c->h_losses) cudaFreeHost(c->h_losses);
    if (c->h_merge) cudaFreeHost(c->h_merge);
    c->act.release();
    c->scratch.release();
    c->persistent.release();
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->side) cudaStreamDestroy(c->side);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (int i = 0; i < 5; ++i) {
        if (c->ev_fork[i]) cudaEventDestroy(c->ev_fork[i]);
        if (c->ev_ready[i]) cudaEventDestroy(c->ev_ready[i]);
    }
    if (c->corpus) cudaFree(c->corpus);
    if (c->d_rows) cudaFree(c->d_rows);
    if (c->sync_tasks) cudaFree(c->sync_tasks);
    delete c;
}

spes_status spes_set_ownership(spes_ctx* c, const int32_t* node_offsets, const int32_t* experts) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        std::vector<std::vector<int>> ne(c->n_nodes);
        for (int n = 0; n < c->n_nodes; ++n) {
            for (int q = node_offsets[n]; q < node_offsets[n + 1]; ++q) {
                const int e = experts[q];
                if (e < 0 || e >= c->lay.M)
                    throw std::invalid_argument("ownership: expert id out of range");
                if (!ne[n].empty() && e <= ne[n].back())
                    throw std::invalid_argument("ownership: experts must be sorted and distinct");
                ne[n].push_back(e);
            }
        }
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->node_experts = ne;
        build_ownership_tables(c);
        c->n_sync_tasks = -1;  // the exchange plan follows the ownership map
        // activation buffers embed grad offsets / tile bounds: rebuild on next step
        c->act.release();
        c->T = c->T_pad = 0;
    });
}

// the caller's parameter vector (enumerate_blocks layout, host) -> the device model
void upload_user_params(spes_ctx* c, const float* host) {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    CounterScope counter_scope(c);
    if (!c->padded) {
        ck(cudaMemcpyAsync(c->params, host, sizeof(float) * c->lay.total(), cudaMemcpyHostToDevice,
                           c->stream),
           "H2D params");
    } else {
        std::vector<float> dev(static_cast<size_t>(c->lay.total()), 0.f);
        convert_layout(c->ulay, c->lay, host, dev.data(), true);
        ck(cudaMemcpyAsync(c->params, dev.data(), sizeof(float) * dev.size(),
                           cudaMemcpyHostToDevice, c->stream),
           "H2D params");
        ck(cudaStreamSynchronize(c->stream), "sync");
    }
    refresh_shadows_all(c);
    ck(cudaStreamSynchronize(c->stream), "sync");
}
// the device model -> the caller's layout (host)
void download_user_params(spes_ctx* c, float* host) {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    if (!c->padded) {
        ck(cudaMemcpyAsync(host, c->params, sizeof(float) * c->lay.total(), cudaMemcpyDeviceToHost,
                           c->stream),
           "D2H params");
        ck(cudaStreamSynchronize(c->stream), "sync");
        return;
    }
    std::vector<float> dev(static_cast<size_t>(c->lay.total()));
    ck(cudaMemcpyAsync(dev.data(), c->params, sizeof(float) * dev.size(), cudaMemcpyDeviceToHost,
                       c->stream),
       "D2H params");
    ck(cudaStreamSynchronize(c->stream), "sync");
    convert_layout(c->ulay, c->lay, dev.data(), host, false);
}

spes_status spes_load_params(spes_ctx* c, const float* host, int64_t n) {
    return guard([&] {
        if (n != c->ulay.total()) throw std::invalid_argument("load_params: size mismatch");
        upload_user_params(c, host);
    });
}

// ---- upcycling (model.hpp:415-460), host side: upcycle.cpp ----
extern "C++" {
namespace spes_upcycle {
void upcycle(int64_t V, int64_t d, int64_t f, int L, const float* dense, int m, double noise_frac,
             double noise_std, uint64_t seed, float* out);
}
}

spes_status spes_upcycle_from_dense(const spes_model_cfg* dense_cfg, const float* dense_params,
                                    int32_t m, double noise_frac, double noise_std, uint64_t seed,
                                    spes_model_cfg* out_cfg, float* out_params) {
    return guard([&] {
        if (dense_cfg->experts_total != 1)
            throw std::invalid_argument("upcycle: source must have a single expert");
        if (m < 2) throw std::invalid_argument("upcycle: need M >= 2");
        if (dense_cfg->tied_head) throw std::logic_error("tied head not implemented");
        spes_model_cfg oc = *dense_cfg;
        oc.experts_total = m;
        oc.renormalize_after_topk = 1;
        spes_upcycle::upcycle(dense_cfg->vocab, dense_cfg->hidden, dense_cfg->intermediate,
                              dense_cfg->layers, dense_params, m, noise_frac, noise_std, seed,
                              out_params);
        if (out_cfg) *out_cfg = oc;
    });
}

// ---- wire / checkpoint format (proj/src/wire.cpp:96-176, 212-236) ----
namespace {
std::vector<spes_wire::Block> wire_blocks(const spes_model_cfg* cfg) {
    // ModelConfig::validate (model.hpp:33-40) only: the codec has no tiling constraints
    if (cfg->vocab < 1 || cfg->hidden < 1 || cfg->intermediate < 1 || cfg->layers < 1)
        throw std::invalid_argument("model config: all dims must be >= 1");
    if (cfg->experts_active < 1 || cfg->experts_active > cfg->experts_total)
        throw std::invalid_argument("model config: need 1 <= k <= M");
    if (cfg->tied_head) throw std::logic_error("tied head not implemented");
    return spes_wire::model_blocks(cfg->vocab, cfg->hidden, cfg->intermediate, cfg->layers,
                                   cfg->experts_total);
}
// device parameters <-> a host copy (pinned staging would not pay off for a one-shot export)
std::vector<float> params_to_host(spes_ctx* c) {
    std::vector<float> h(static_cast<size_t>(c->ulay.total()));
    download_user_params(c, h.data());
    return h;
}
void params_from_host(spes_ctx* c, const std::vector<float>& h) { upload_user_params(c, h.data()); }
}  // namespace

int64_t spes_model_payload_bytes(const spes_model_cfg* cfg) {
    try {
        return spes_wire::payload_bytes(wire_blocks(cfg));
    } catch (...) {
        return -1;
    }
}

spes_status spes_encode_model_host(const spes_model_cfg* cfg, const float* params, uint8_t* out,
                                   int64_t cap) {
    return guard([&] {
        const auto blocks = wire_blocks(cfg);
        if (cap < spes_wire::payload_bytes(blocks))
            throw std::invalid_argument("encode_model: output buffer too small");
        spes_wire::encode_model(blocks, params, out);
    });
}

spes_status spes_decode_model_host(const spes_model_cfg* cfg, const uint8_t* payload, int64_t len,
                                   float* params) {
    return guard([&] {
        const auto blocks = wire_blocks(cfg);
        const auto& last = blocks.back();
        std::vector<float> tmp(static_cast<size_t>(last.offset + last.numel));
        spes_wire::decode_model(blocks, payload, len, tmp.data());  // all-or-nothing
        std::memcpy(params, tmp.data(), sizeof(float) * tmp.size());
    });
}

spes_status spes_encode_model(spes_ctx* c, uint8_t* out, int64_t cap) {
    return guard([&] {
        const auto blocks = wire_blocks(&c->cfg);
        if (cap < spes_wire::payload_bytes(blocks))
            throw std::invalid_argument("encode_model: output buffer too small");
        const auto h = params_to_host(c);
        spes_wire::encode_model(blocks, h.data(), out);
    });
}

spes_status spes_decode_model(spes_ctx* c, const uint8_t* payload, int64_t len) {
    return guard([&] {
        const auto blocks = wire_blocks(&c->cfg);
        std::vector<float> h(static_cast<size_t>(c->ulay.total()));
        spes_wire::decode_model(blocks, payload, len, h.data());
        params_from_host(c, h);
    });
}

spes_status spes_write_checkpoint(spes_ctx* c, const char* path, uint64_t round) {
    return guard([&] {
        const auto blocks = wire_blocks(&c->cfg);
        const auto h = params_to_host(c);
        spes_wire::write_checkpoint(path, blocks, h.data(), round);
    });
}

spes_status spes_read_checkpoint(spes_ctx* c, const char* path, uint64_t* round) {
    return guard([&] {
        const auto blocks = wire_blocks(&c->cfg);
        std::vector<float> h(static_cast<size_t>(c->ulay.total()));
        const uint64_t r = spes_wire::read_checkpoint(path, blocks, h.data());
        params_from_host(c, h);
        if (round) *round = r;
    });
}

spes_status spes_load_params_device(spes_ctx* c, const float* dev, int64_t n) {
    return guard([&] {
        if (n != c->ulay.total()) throw std::invalid_argument("load_params: size mismatch");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (c->padded) {  // through the host conversion (padded layouts are small models)
            std::vector<float> h(static_cast<size_t>(n));
            ck(cudaMemcpy(h.data(), dev, sizeof(float) * n, cudaMemcpyDeviceToHost), "D2H params");
            upload_user_params(c, h.data());
            return;
        }
        ck(cudaMemcpyAsync(c->params, dev, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->stream),
           "D2D params");
        refresh_shadows_all(c);
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

spes_status spes_read_params(spes_ctx* c, float* host, int64_t n) {
    return guard([&] {
        if (n != c->ulay.total()) throw std::invalid_argument("read_params: size mismatch");
        download_user_params(c, host);
    });
}

spes_status spes_round_begin(spes_ctx* c, int32_t carry_state) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        check_status(c, " (unreported step of the previous round)");
        if (!carry_state) {
            // fresh MaskedAdamW (trainer.hpp:151-156): zero moments, step 0
            ck(cudaMemsetAsync(c->m, 0, sizeof(float) * c->G, c->stream), "m");
            ck(cudaMemsetAsync(c->v, 0, sizeof(float) * c->G, c->stream), "v");
            c->adam_step = 0;
        }
    });
}

spes_status spes_local_step(spes_ctx* c, const int32_t* tokens, int64_t B, int64_t S,
                            const spes_adamw_cfg* opt, spes_losses* losses) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (B < 1 || S < 1) throw std::invalid_argument("batch: need B, S >= 1");
        validate_tokens(c, tokens, B * (S + 1));
        ensure_activations(c, B, S);
        upload_tokens(c, tokens, B * (S + 1));
        local_step_impl(c, B, S, opt, losses);
    });
}

spes_status spes_local_step_device(spes_ctx* c, const int32_t* d_tokens, int64_t B, int64_t S,
                                   const spes_adamw_cfg* opt, spes_losses* losses) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (B < 1 || S < 1) throw std::invalid_argument("batch: need B, S >= 1");
        ensure_activations(c, B, S);
        ck(cudaMemcpyAsync(c->tokens, d_tokens, sizeof(int32_t) * B * (S + 1),
                           cudaMemcpyDeviceToDevice, c->stream),
           "D2D tokens");
        local_step_impl(c, B, S, opt, losses);  // losses == NULL: reported at round end
    });
}

spes_status spes_local_round(spes_ctx* c, const int32_t* tokens, int64_t B, int64_t S, int32_t H,
                             const double* lr, const spes_adamw_cfg* opt, int32_t carry_state,
                             spes_losses* per_step) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (H < 1) throw std::invalid_argument("local_round: need H >= 1");
        if (B < 1 || S < 1) throw std::invalid_argument("batch: need B, S >= 1");
        const int64_t per = B * (S + 1);
        if (!carry_state) {
            ck(cudaMemsetAsync(c->m, 0, sizeof(float) * c->G, c->stream), "m");
            ck(cudaMemsetAsync(c->v, 0, sizeof(float) * c->G, c->stream), "v");
            c->adam_step = 0;
        }
        ensure_activations(c, B, S);
        for (int h = 0; h < H; ++h) {
            const int32_t* tk = tokens + static_cast<int64_t>(h) * per;
            validate_tokens(c, tk, per);
            upload_tokens(c, tk, per);
            spes_adamw_cfg o = *opt;
            if (lr) o.lr = lr[h];
            spes_losses tmp;
            spes_losses* lo = per_step ? &per_step[h] : &tmp;
            try {
                local_step_impl(c, B, S, &o, lo);
            } catch (const std::runtime_error& e) {
                if (dynamic_cast<const SpesError*>(&e)) throw;
                throw std::runtime_error(std::string(e.what()) + " at step " + std::to_string(h));
            }
        }
    });
}

// ---- CommLedger (protocol.hpp:29-52) ----
extern "C++" {
namespace spes_ledger {
struct Entry {
    int32_t node, round;
    uint64_t up, down;
};
std::vector<Entry> expected(int64_t V, int64_t d, int64_t f, int L, int M, int nodes,
                            const std::vector<std::vector<int>>& owned, int rounds, bool diloco,
                            uint64_t totals[4]);
struct RoundRow {
    int32_t round;
    double mean_total, mean_ce, mean_lb, mean_moe_z, mean_z, merge_displacement_sq;
    uint64_t bytes_up, bytes_down;
};
std::string metrics_csv(const RoundRow* rows, int n, int64_t tokens_per_round,
                        const double* wall_ms, int n_wall);
}
}

spes_status spes_metrics_csv(const spes_round_metrics* rows, int32_t n, int64_t tokens_per_round,
                             const double* wall_ms, char* out, int64_t cap, int64_t* len) {
    return guard([&] {
        if (n < 0) throw std::invalid_argument("metrics: negative row count");
        std::vector<spes_ledger::RoundRow> r(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i)
            r[i] = {rows[i].round, rows[i].mean_total, rows[i].mean_ce, rows[i].mean_lb,
                    rows[i].mean_moe_z, rows[i].mean_z, rows[i].merge_displacement_sq,
                    rows[i].bytes_up, rows[i].bytes_down};
        const std::string t = spes_ledger::metrics_csv(r.data(), n, tokens_per_round, wall_ms,
                                                       wall_ms ? n : 0);
        *len = static_cast<int64_t>(t.size());
        if (out && cap > 0) std::memcpy(out, t.data(), std::min<size_t>(t.size(), static_cast<size_t>(cap)));
    });
}

spes_status spes_comm_ledger(const spes_model_cfg* cfg, int32_t n_nodes,
                             const int32_t* node_offsets, const int32_t* experts, int32_t rounds,
                             int32_t diloco, spes_ledger_entry* entries, int32_t cap,
                             int32_t* n_entries, uint64_t* totals) {
    return guard([&] {  // host bookkeeping: the model's shape only, no tcgen05 tiling limits
        if (cfg->vocab < 1 || cfg->hidden < 1 || cfg->intermediate < 1 || cfg->layers < 1 ||
            cfg->experts_total < 1)
            throw std::invalid_argument("config: all dimensions must be positive");
        const int M = cfg->experts_total;
        if (n_nodes < 1 || n_nodes > M)
            throw std::invalid_argument("partition: need 1 <= N <= M (no empty nodes)");
        std::vector<std::vector<int>> owned(static_cast<size_t>(n_nodes));
        if (node_offsets) {
            for (int n = 0; n < n_nodes; ++n)
                for (int q = node_offsets[n]; q < node_offsets[n + 1]; ++q) owned[n].push_back(experts[q]);
        } else {  // param_partition (model.hpp:466-477)
            const int base = M / n_nodes, extra = M % n_nodes;
            int next = 0;
            for (int n = 0; n < n_nodes; ++n)
                for (int j = 0; j < base + (n < extra ? 1 : 0); ++j) owned[n].push_back(next++);
        }
        const auto e = spes_ledger::expected(cfg->vocab, cfg->hidden, cfg->intermediate,
                                             cfg->layers, M, n_nodes, owned, rounds, diloco != 0,
                                             totals);
        for (size_t i = 0; i < e.size() && static_cast<int32_t>(i) < cap; ++i)
            entries[i] = spes_ledger_entry{e[i].node, e[i].round, e[i].up, e[i].down};
        *n_entries = static_cast<int32_t>(e.size());
    });
}

// ---- device corpus and batch streams (corpus.cpp) ----
extern "C++" {
namespace spes_corpus {
struct BatchStream;
void gen_corpus(int64_t vocab, int64_t seq, int sources, int64_t sequences, uint64_t seed,
                double skew, int32_t* tokens, int32_t* source_id);
void shard_corpus(const int32_t* source_id, int64_t n, int nodes, int by_source, uint64_t seed,
                  int64_t* order, int64_t* offsets);
BatchStream* stream_create(const int64_t* shard, int64_t n, int64_t batch, uint64_t seed);
void stream_next(BatchStream* s, int64_t* rows);
void stream_destroy(BatchStream* s);
void prepare_device_corpus(int64_t vocab, int64_t seq, int sources, int64_t sequences,
                           uint64_t seed, double skew, std::vector<double>& cum,
                           uint64_t* state, int* pos);
}
}
struct spes_batch_stream {
    spes_corpus::BatchStream* s;
};

spes_status spes_gen_corpus(int64_t vocab, int64_t seq, int32_t sources, int64_t sequences,
                            uint64_t seed, double skew, int32_t* tokens, int32_t* source_id) {
    return guard([&] {
        spes_corpus::gen_corpus(vocab, seq, sources, sequences, seed, skew, tokens, source_id);
    });
}

spes_status spes_shard_corpus(const int32_t* source_id, int64_t sequences, int32_t nodes,
                              int32_t by_source, uint64_t seed, int64_t* order,
                              int64_t* node_offsets) {
    return guard([&] {
        spes_corpus::shard_corpus(source_id, sequences, nodes, by_source, seed, order, node_offsets);
    });
}

spes_status spes_batch_stream_create(const int64_t* shard, int64_t n, int64_t batch, uint64_t seed,
                                     spes_batch_stream** out) {
    return guard([&] {
        *out = new spes_batch_stream{spes_corpus::stream_create(shard, n, batch, seed)};
    });
}

spes_status spes_batch_stream_next(spes_batch_stream* s, int64_t* rows) {
    return guard([&] { spes_corpus::stream_next(s->s, rows); });
}

void spes_batch_stream_destroy(spes_batch_stream* s) {
    if (!s) return;
    spes_corpus::stream_destroy(s->s);
    delete s;
}

spes_status spes_corpus_load(spes_ctx* c, const int32_t* tokens, int64_t sequences, int64_t seq) {
    return guard([&] {
        if (sequences < 1 || seq < 1) throw std::invalid_argument("corpus: need sequences, S >= 1");
        validate_tokens(c, tokens, sequences * (seq + 1));  // once, not per step
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (c->corpus) cudaFree(c->corpus);
        c->corpus = nullptr;
        ck(cudaMalloc(&c->corpus, sizeof(int32_t) * sequences * (seq + 1)), "corpus alloc");
        ck(cudaMemcpy(c->corpus, tokens, sizeof(int32_t) * sequences * (seq + 1),
                      cudaMemcpyHostToDevice),
           "corpus H2D");
        c->corpus_rows = sequences;
        c->corpus_seq = seq;
    });
}

spes_status spes_corpus_generate(spes_ctx* c, int64_t vocab, int64_t seq, int32_t sources,
                                 int64_t sequences, uint64_t seed, double skew,
                                 int32_t* tokens_out, int32_t* source_id_out) {
    return guard([&] {
        if (vocab > c->ulay.V)
            throw std::invalid_argument("corpus: vocabulary larger than the model's");
        std::vector<double> cum;
        uint64_t state[312];
        int pos = 0;
        spes_corpus::prepare_device_corpus(vocab, seq, sources, sequences, seed, skew, cum, state,
                                           &pos);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int64_t n = sequences * (seq + 1);
        if (c->corpus) cudaFree(c->corpus);
        c->corpus = nullptr;
        c->corpus_rows = 0;
        ck(cudaMalloc(&c->corpus, sizeof(int32_t) * n), "corpus alloc");
        double *d_cum = nullptr, *d_u = nullptr;
        uint64_t* d_state = nullptr;
        auto release = [&] {
            cudaFree(d_cum);
            cudaFree(d_u);
            cudaFree(d_state);
        };
        try {
            ck(cudaMalloc(&d_cum, sizeof(double) * cum.size()), "corpus tables");
            ck(cudaMalloc(&d_u, sizeof(double) * n), "corpus draws");
            ck(cudaMalloc(&d_state, sizeof(state)), "engine state");
            ck(cudaMemcpyAsync(d_cum, cum.data(), sizeof(double) * cum.size(),
                               cudaMemcpyHostToDevice, c->stream),
               "H2D tables");
            ck(cudaMemcpyAsync(d_state, state, sizeof(state), cudaMemcpyHostToDevice, c->stream),
               "H2D state");
            spes_k::corpus_draws(d_state, pos, n, d_u, c->stream);
            spes_k::corpus_chains(d_cum, d_u, sequences, seq, static_cast<int>(vocab), sources,
                                  c->corpus, c->stream);
            ck(cudaGetLastError(), "corpus kernels");
            if (tokens_out)
                ck(cudaMemcpyAsync(tokens_out, c->corpus, sizeof(int32_t) * n,
                                   cudaMemcpyDeviceToHost, c->stream),
                   "D2H corpus");
            ck(cudaStreamSynchronize(c->stream), "corpus generation");
        } catch (...) {
            release();
            throw;
        }
        release();
        if (source_id_out)
            for (int64_t r = 0; r < sequences; ++r) source_id_out[r] = static_cast<int32_t>(r % sources);
        c->corpus_rows = sequences;
        c->corpus_seq = seq;
    });
}

namespace {
void gather_corpus_rows(spes_ctx* c, const int64_t* rows, int64_t B) {
    if (!c->corpus) throw std::logic_error("local_step_rows: no corpus loaded (spes_corpus_load)");
    for (int64_t b = 0; b < B; ++b)
        if (rows[b] < 0 || rows[b] >= c->corpus_rows)
            throw std::out_of_range("batch: corpus row out of range");
    if (B > c->d_rows_cap) {
        if (c->d_rows) cudaFree(c->d_rows);
        ck(cudaMalloc(&c->d_rows, sizeof(int64_t) * B), "rows alloc");
        c->d_rows_cap = B;
    }
    // pageable source: staged by the driver, safe to reuse right after the call
    ck(cudaMemcpyAsync(c->d_rows, rows, sizeof(int64_t) * B, cudaMemcpyHostToDevice, c->stream),
       "H2D rows");
    spes_k::corpus_gather(c->corpus, c->d_rows, B, c->corpus_seq + 1, c->tokens, c->stream);
}
}  // namespace

spes_status spes_local_step_rows(spes_ctx* c, const int64_t* rows, int64_t B,
                                 const spes_adamw_cfg* opt, spes_losses* losses) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (B < 1) throw std::invalid_argument("batch: need B >= 1");
        ensure_activations(c, B, c->corpus_seq);
        gather_corpus_rows(c, rows, B);
        local_step_impl(c, B, c->corpus_seq, opt, losses);
    });
}

spes_status spes_local_round_rows(spes_ctx* c, const int64_t* rows, int64_t B, int32_t H,
                                  const double* lr, const spes_adamw_cfg* opt, int32_t carry_state,
                                  spes_losses* per_step) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (H < 1) throw std::invalid_argument("local_round: need H >= 1");
        if (B < 1) throw std::invalid_argument("batch: need B >= 1");
        if (!carry_state) {
            ck(cudaMemsetAsync(c->m, 0, sizeof(float) * c->G, c->stream), "m");
            ck(cudaMemsetAsync(c->v, 0, sizeof(float) * c->G, c->stream), "v");
            c->adam_step = 0;
        }
        ensure_activations(c, B, c->corpus_seq);
        for (int h = 0; h < H; ++h) {
            gather_corpus_rows(c, rows + static_cast<int64_t>(h) * B, B);
            spes_adamw_cfg o = *opt;
            if (lr) o.lr = lr[h];
            spes_losses tmp;
            spes_losses* lo = per_step ? &per_step[h] : &tmp;
            try {
                local_step_impl(c, B, c->corpus_seq, &o, lo);
            } catch (const std::runtime_error& e) {
                if (dynamic_cast<const SpesError*>(&e)) throw;
                throw std::runtime_error(std::string(e.what()) + " at step " + std::to_string(h));
            }
        }
    });
}

// ---- DiLoCo baseline: full-model outer sync (protocol.cpp:199-213, trainer.hpp:228-271) ----
// Slicing: the flat parameter vector in N equal slices of outer_slice floats (the last one
// padded); rank r owns slice r. Exchange = grouped send/recv (each rank receives its slice
// from every node, node order), fp64 outer step on the slice, then all-gather.
spes_status spes_outer_begin(spes_ctx* c) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int64_t P = c->lay.total(), N = c->n_nodes;
        const int64_t sl = rup((P + N - 1) / N, 4);
        if (sl != c->outer_slice) {
            c->outer_theta = c->persistent.alloc<float>(sl);
            c->outer_buf = c->persistent.alloc<double>(sl);
            c->outer_recv = c->persistent.alloc<float>(sl * N);
            c->outer_gather = c->persistent.alloc<float>(sl * N);
            c->outer_slice = sl;
        }
        const int64_t lo = std::min<int64_t>(P, sl * c->node), n = std::min<int64_t>(P, lo + sl) - lo;
        ck(cudaMemsetAsync(c->outer_theta, 0, sizeof(float) * sl, c->stream), "theta");
        ck(cudaMemcpyAsync(c->outer_theta, c->params + lo, sizeof(float) * n, cudaMemcpyDeviceToDevice,
                           c->stream),
           "theta snapshot");
        ck(cudaMemsetAsync(c->outer_buf, 0, sizeof(double) * sl, c->stream), "nesterov");
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->outer_ready = true;
    });
}

spes_status spes_outer_sync(spes_ctx* c, int32_t kind, double lr, double momentum,
                            spes_sync_stats* stats) {
    return guard([&] {
        if (!c->outer_ready)
            throw std::logic_error("outer_sync: call spes_outer_begin on the round-start model first");
        if (kind != 0 && kind != 1) throw std::invalid_argument("outer_sync: kind is 0 (SGD) or 1 (Nesterov)");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        cudaStream_t st = c->stream;
        const int64_t P = c->lay.total(), sl = c->outer_slice;
        const int N = c->n_nodes, me = c->node;
        auto range = [&](int r) {
            const int64_t lo = std::min<int64_t>(P, sl * r);
            return std::make_pair(lo, std::min<int64_t>(P, lo + sl) - lo);
        };
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        ck(cudaEventRecord(e0, st), "event");
        const auto [mlo, mn] = range(me);
        // recv[i] = node i's local values of my slice (node order)
        ck(cudaMemcpyAsync(c->outer_recv + static_cast<int64_t>(me) * sl, c->params + mlo,
                           sizeof(float) * mn, cudaMemcpyDeviceToDevice, st),
           "own slice");
        if (N > 1) {
            ckn(ncclGroupStart(), "group");
            for (int p = 0; p < N; ++p) {
                if (p == me) continue;
                const auto [plo, pn] = range(p);
                if (pn > 0) ckn(ncclSend(c->params + plo, pn, ncclFloat, p, c->comm, st), "send");
                if (mn > 0)
                    ckn(ncclRecv(c->outer_recv + static_cast<int64_t>(p) * sl, mn, ncclFloat, p, c->comm, st),
                        "recv");
            }
            ckn(ncclGroupEnd(), "group end");
        }
        spes_k::outer_step(c->outer_theta, c->outer_recv, N, mn, sl, kind, lr, momentum, c->outer_buf,
                           c->outer_gather + static_cast<int64_t>(me) * sl, st);
        if (N > 1)
            ckn(ncclAllGather(c->outer_gather + static_cast<int64_t>(me) * sl, c->outer_gather, sl,
                              ncclFloat, c->comm, st),
                "allgather model");
        ck(cudaMemcpyAsync(c->params, c->outer_gather, sizeof(float) * P, cudaMemcpyDeviceToDevice, st),
           "new global");
        refresh_shadows_all(c);
        ck(cudaEventRecord(e1, st), "event");
        ck(cudaStreamSynchronize(st), "outer sync");
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, e0, e1), "event time");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (stats) {
            stats->psi_bytes_in = 0;
            stats->expert_bytes_in = 4.0 * (static_cast<double>(mn) * (N - 1) + static_cast<double>(P - mn));
            stats->ms = ms;
        }
    });
}

// ---- sync (Server::aggregate, protocol.cpp:197-251) ----
// Map every peer's parameter vector (collective, once): IPC handles travel by an NCCL
// all-gather; a second all-gather of the per-rank outcome keeps the choice between the
// NVLink peer-read path and the NCCL send/recv path identical on all ranks.
static void open_peer_params(spes_ctx* c) {
    if (c->p2p_tried) return;
    c->p2p_tried = true;
    const int N = c->n_nodes, me = c->node;
    if (const char* e = std::getenv("SPES_SYNC_P2P"))
        if (std::atoi(e) == 0) return;  // all ranks see the same environment
    struct Rec {
        cudaIpcMemHandle_t h, hf;
        int32_t ok;
        int32_t pad[15];
    };
    if (!c->sync_flags) c->sync_flags = c->persistent.alloc<uint32_t>(c->lay.L);
    Rec mine{};
    mine.ok = cudaIpcGetMemHandle(&mine.h, c->params) == cudaSuccess &&
                      cudaIpcGetMemHandle(&mine.hf, c->sync_flags) == cudaSuccess
                  ? 1
                  : 0;
    cudaGetLastError();
    Rec* d = nullptr;
    ck(cudaMalloc(&d, sizeof(Rec) * N), "cudaMalloc");
    ck(cudaMemcpy(d + me, &mine, sizeof(Rec), cudaMemcpyHostToDevice), "H2D");
    ckn(ncclAllGather(d + me, d, sizeof(Rec), ncclUint8, c->comm, c->stream), "allgather ipc");
    std::vector<Rec> all(N);
    ck(cudaMemcpyAsync(all.data(), d, sizeof(Rec) * N, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    int32_t ok = 1;
    std::vector<float*> peers(N, nullptr);
    std::vector<uint32_t*> pflags(N, nullptr);
    pflags[me] = c->sync_flags;
    for (int n = 0; n < N; ++n) {
        if (!all[n].ok) ok = 0;
        if (n == me || !ok) continue;
        void* p = nullptr;
        void* pf = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[n].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&pf, all[n].hf, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            if (p) cudaIpcCloseMemHandle(p);
            ok = 0;
            continue;
        }
        peers[n] = static_cast<float*>(p);
        pflags[n] = static_cast<uint32_t*>(pf);
    }
    // agree: every rank must have opened every peer
    int32_t* flags = reinterpret_cast<int32_t*>(d);
    ck(cudaMemcpy(flags + me, &ok, 4, cudaMemcpyHostToDevice), "H2D");
    ckn(ncclAllGather(flags + me, flags, 1, ncclInt32, c->comm, c->stream), "allgather ok");
    std::vector<int32_t> oks(N);
    ck(cudaMemcpyAsync(oks.data(), flags, 4 * N, cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    cudaFree(d);
    bool all_ok = true;
    for (int32_t v : oks) all_ok = all_ok && v;
    if (!all_ok) {
        for (int n = 0; n < N; ++n) {
            if (n == me) continue;
            if (peers[n]) cudaIpcCloseMemHandle(peers[n]);
            if (pflags[n]) cudaIpcCloseMemHandle(pflags[n]);
        }
        return;
    }
    c->peer_params = peers;
    c->peer_flags = pflags;
    c->peer_flags_dev = c->persistent.alloc<uint32_t*>(N);
    ck(cudaMemcpy(c->peer_flags_dev, pflags.data(), sizeof(uint32_t*) * N, cudaMemcpyHostToDevice),
       "peer flags");
    c->p2p_ok = true;
}

// Task list of the fused expert exchange (kernels.cu sync_exchange_k): chunks of every
// owner-set mean this node is primary for (owners ascending; copies of
// co-owners read from their mapped parameters) and of every expert it pulls from a
// primary. Built once per ownership map (pointers do not move).
static void build_sync_tasks(spes_ctx* c, const std::vector<int>& primary) {
    const Layout& L = c->lay;
    const int me = c->node;
    // chunk = 2^lg scalars: about 32 chunks per expert within [64 Ki, 1 Mi] (cfg2: 128 Ki,
    // cfg5: 512 Ki; 2^17..2^20 measured within 3% at cfg5 N=4); order 1: layers interleaved
    int lg = 16, order = 1;
    while (lg < 20 && (int64_t(1) << (lg + 1)) * 32 <= c->lay.per_expert()) ++lg;
    if (const char* e = std::getenv("SPES_SYNC_CHUNK")) lg = std::max(12, std::min(24, std::atoi(e)));
    if (const char* e = std::getenv("SPES_SYNC_ORDER")) order = std::atoi(e);
    const int64_t per = L.per_expert(), chunk = int64_t(1) << lg;
    std::vector<std::vector<spes_k::SyncTask>> means(L.L), pulls(L.L);
    std::vector<int> layer_total(L.L, 0);
    c->sync_mean_bytes = c->sync_pull_bytes = 0;
    c->sync_max_src = 1;
    for (int l = 0; l < L.L; ++l)
        for (int e = 0; e < L.M; ++e) {
            const auto& O = c->owners[e];
            const int64_t off = L.off_expert(l, e);
            const bool mean = O.size() >= 2 && primary[e] == me;
            const bool pull = primary[e] >= 0 && primary[e] != me;
            if (!mean && !pull) continue;
            if (mean && static_cast<int>(O.size()) > spes_k::SYNC_MAX_SRC)
                throw std::invalid_argument("sync: more than 8 owners of one expert");
            for (int64_t o0 = 0; o0 < per; o0 += chunk) {
                spes_k::SyncTask t{};
                t.dst = c->params + off + o0;
                t.off = o0;
                t.n4 = std::min(chunk, per - o0) / 4;
                t.slot = l * L.M + e;
                t.layer = l;
                if (mean) {
                    t.nsrc = static_cast<int32_t>(O.size());
                    t.primary = -1;
                    for (size_t q = 0; q < O.size(); ++q)
                        t.src[q] = (O[q] == me ? c->params : c->peer_params[O[q]]) + off + o0;
                    means[l].push_back(t);
                    layer_total[l] += 1;
                } else {
                    t.nsrc = 0;
                    t.primary = primary[e];
                    t.src[0] = c->peer_params[primary[e]] + off + o0;
                    pulls[l].push_back(t);
                }
            }
            if (mean) c->sync_mean_bytes += 4.0 * per * (O.size() - 1);
            if (mean) c->sync_max_src = std::max(c->sync_max_src, static_cast<int>(O.size()));
            if (pull) c->sync_pull_bytes += 4.0 * per;
        }
    // a layer's pulls round-robin over the primaries, starting after this node: every node
    // pulls from every primary at the same time instead of all nodes draining one primary's
    // NVLink egress after another (the (layer, expert) order made the primaries hot spots)
    for (int l = 0; l < L.L; ++l) {
        const int N = c->n_nodes;
        std::vector<std::vector<spes_k::SyncTask>> byp(N);
        for (const auto& t : pulls[l]) byp[(t.primary - me - 1 + 2 * N) % N].push_back(t);
        std::vector<spes_k::SyncTask> rr;
        for (size_t i = 0;; ++i) {
            bool any = false;
            for (int p = 0; p < N; ++p)
                if (i < byp[p].size()) {
                    rr.push_back(byp[p][i]);
                    any = true;
                }
            if (!any) break;
        }
        pulls[l].swap(rr);
    }
    // queue order: means of layers 0 and 1, pulls of layer 0, means of layer 2, pulls of
    // layer 1, ...: a layer's pulls come after every node's means of that layer have had a
    // head start, and the means of later layers still overlap them
    std::vector<spes_k::SyncTask> q;
    if (order == 1) {
        for (int l = 0; l <= L.L; ++l) {
            if (l < L.L) q.insert(q.end(), means[l].begin(), means[l].end());
            if (l >= 1) q.insert(q.end(), pulls[l - 1].begin(), pulls[l - 1].end());
        }
    } else {  // every mean first, then every pull
        for (int l = 0; l < L.L; ++l) q.insert(q.end(), means[l].begin(), means[l].end());
        for (int l = 0; l < L.L; ++l) q.insert(q.end(), pulls[l].begin(), pulls[l].end());
    }
    const int n = static_cast<int>(q.size());
    const auto& means_q = q;
    if (c->sync_tasks) cudaFree(c->sync_tasks);
    ck(cudaMalloc(&c->sync_tasks, sizeof(spes_k::SyncTask) * std::max(n, 1)), "sync tasks");
    if (n > 0)
        ck(cudaMemcpy(c->sync_tasks, means_q.data(), sizeof(spes_k::SyncTask) * n,
                      cudaMemcpyHostToDevice),
           "sync tasks");
    if (!c->sync_ctr) {
        c->sync_ctr = c->persistent.alloc<int>(1 + L.L);
        c->sync_layer_total = c->persistent.alloc<int>(L.L);
    }
    ck(cudaMemcpy(c->sync_layer_total, layer_total.data(), sizeof(int) * L.L,
                  cudaMemcpyHostToDevice),
       "layer totals");
    c->n_sync_tasks = n;
}

spes_status spes_sync(spes_ctx* c, spes_sync_stats* stats) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        const Layout& L = c->lay;
        const int N = c->n_nodes, me = c->node;
        cudaStream_t st = c->stream;
        if (N == 1) {  // one node: the owner-set means are the node's own values
            if (stats) *stats = spes_sync_stats{};
            check_status(c, " (a step of this round)");
            return;
        }
        cudaEvent_t e0, e1;
        ck(cudaEventCreate(&e0), "event");
        ck(cudaEventCreate(&e1), "event");
        // the reported time starts once every node has arrived (a one-word all-reduce), so it
        // measures the exchange itself, not this node waiting for slower nodes' local rounds
        if (!c->barrier_buf) c->barrier_buf = c->persistent.alloc<int32_t>(1);
        ckn(ncclAllReduce(c->barrier_buf, c->barrier_buf, 1, ncclInt32, ncclSum, c->comm, st),
            "barrier");
        ck(cudaEventRecord(e0, st), "event");
        double psi_in = 0, exp_in = 0;
        Prof prof_sync(c, "sync");
        if (N > 1) {
            const int64_t psi = L.psi();
            if (!c->psi_stage) c->psi_stage = c->scratch.alloc<float>(psi * N);
            // psi: every node's copy, then fp64 node-order mean (protocol.cpp:238-243)
            {
                Prof pp(c, "sync_psi");
                ckn(ncclAllGather(c->params, c->psi_stage, psi, ncclFloat, c->comm, st),
                    "allgather psi");
                spes_k::owner_mean_strided(c->psi_stage, N, psi, psi, c->params, st);
            }
            psi_in = 4.0 * psi * (N - 1);
            // experts: primary owner per expert
            std::vector<int> primary;
            bool balanced = false;
            sync_plan(L.M, N, c->owners, primary, balanced);
            const int s_bal = balanced ? L.M / N : 0;
            const int64_t per = L.per_expert();
            open_peer_params(c);
            // staging for co-owner copies received by this primary (NCCL path only)
            int64_t need = 0;
            for (int e = 0; e < L.M; ++e)
                if (primary[e] == me) need += static_cast<int64_t>(c->owners[e].size() - 1) * per * L.L;
            if (!c->p2p_ok && need > c->expert_stage_cap) {
                c->expert_stage = c->scratch.alloc<float>(need);
                c->expert_stage_cap = need;
            }
            std::map<std::pair<int, int>, float*> slot;  // (expert*L + l, owner) -> staging
            int64_t q = 0;
            // phase timers (profiled rounds only)
            auto ph = std::make_unique<Prof>(c, "sync_to_primary");
            if (!c->p2p_ok) {  // co-owner copies to the primary over NCCL
                ckn(ncclGroupStart(), "group");
                for (int l = 0; l < L.L; ++l)
                    for (int e = 0; e < L.M; ++e) {
                        const auto& O = c->owners[e];
                        if (O.size() < 2) continue;
                        float* mine = c->params + L.off_expert(l, e);
                        if (primary[e] == me) {
                            for (int o : O) {
                                if (o == me) continue;
                                float* dst = c->expert_stage + q;
                                q += per;
                                slot[{e * L.L + l, o}] = dst;
                                ckn(ncclRecv(dst, per, ncclFloat, o, c->comm, st), "recv");
                            }
                        } else if (std::find(O.begin(), O.end(), me) != O.end()) {
                            ckn(ncclSend(mine, per, ncclFloat, primary[e], c->comm, st), "send");
                        }
                    }
                ckn(ncclGroupEnd(), "group end");
            }
            ph.reset();
            const spes_k::Shadows shd = shadows_of(c);
            if (c->p2p_ok) {
                // one persistent kernel: owner-set means at the primary (co-owners' copies
                // read in place over NVLink; their local rounds are done, every rank has
                // passed the psi all-gather above) and pulls from the primaries, a layer's
                // pulls gated by its primary's per-layer flag, so means and pulls overlap
                // across layers and nodes. Both write the experts' bf16 operand copies. The
                // barrier after it keeps every rank from starting its next local round (which
                // rewrites the experts it owns) before every pull from it is done.
                ph = std::make_unique<Prof>(c, "sync_exchange");
                if (c->n_sync_tasks < 0) build_sync_tasks(c, primary);
                exp_in += c->sync_mean_bytes + c->sync_pull_bytes;
                c->sync_epoch += 1;
                spes_k::sync_exchange(c->sync_tasks, c->n_sync_tasks, c->sync_max_src, c->sync_ctr,
                                      c->sync_layer_total, L.L, c->sync_flags, c->peer_flags_dev,
                                      c->sync_epoch, shd, st);
                if (!c->barrier_buf) c->barrier_buf = c->persistent.alloc<int32_t>(1);
                ckn(ncclAllReduce(c->barrier_buf, c->barrier_buf, 1, ncclInt32, ncclSum, c->comm, st),
                    "barrier");
            } else {
                ph = std::make_unique<Prof>(c, "sync_owner_mean");
                // owner-set mean at the primary from the staged copies, owners ascending
                for (int l = 0; l < L.L; ++l)
                    for (int e = 0; e < L.M; ++e) {
                        const auto& O = c->owners[e];
                        if (O.size() < 2 || primary[e] != me) continue;
                        std::vector<const float*> srcs;
                        float* mine = c->params + L.off_expert(l, e);
                        for (int o : O) {
                            srcs.push_back(o == me ? mine : slot[{e * L.L + l, o}]);
                            if (o != me) exp_in += 4.0 * per;
                        }
                        spes_k::owner_mean(srcs.data(), static_cast<int>(srcs.size()), per, mine,
                                           st, nullptr, l * L.M + e);
                    }
                ph.reset();
                ph = std::make_unique<Prof>(c, "sync_gather");
            }
            // NCCL path: every node receives every expert from its primary
            if (c->p2p_ok) {
                // done by the exchange above
            } else if (balanced) {
                for (int l = 0; l < L.L; ++l) {
                    float* base = c->params + L.off_expert(l, 0);
                    const int64_t cnt = per * s_bal;
                    ckn(ncclAllGather(base + me * cnt, base, cnt, ncclFloat, c->comm, st), "allgather experts");
                }
            } else {
                ckn(ncclGroupStart(), "group");
                for (int l = 0; l < L.L; ++l)
                    for (int e = 0; e < L.M; ++e) {
                        if (primary[e] < 0) continue;
                        float* p = c->params + L.off_expert(l, e);
                        ckn(ncclBroadcast(p, p, per, ncclFloat, primary[e], c->comm, st), "bcast");
                    }
                ckn(ncclGroupEnd(), "group end");
            }
            if (!c->p2p_ok) {
                int64_t mine_primary = 0;
                for (int e = 0; e < L.M; ++e) mine_primary += primary[e] == me;
                exp_in += 4.0 * per * L.L * (L.M - mine_primary);
            }
            ph.reset();
            ph = std::make_unique<Prof>(c, "sync_refresh_shadows");
            if (c->p2p_ok)  // expert copies were written by the means and the pulls
                spes_k::refresh_shadows(c->params, refresh_table(c), L.V * L.d, shd, st);  // the head leads the refresh table
            else
                refresh_shadows_all(c);
            ph.reset();
        }
        ck(cudaEventRecord(e1, st), "event");
        ck(cudaStreamSynchronize(st), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, e0, e1), "event time");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (stats) {
            stats->psi_bytes_in = psi_in;
            stats->expert_bytes_in = exp_in;
            stats->ms = ms;
        }
        // after the collective, so a bad node never leaves its peers waiting in it (its
        // updates stopped at the bad step; the reference aborts the run at that point)
        check_status(c, " (a step of this round)");
    });
}

// ---- merge (merging.hpp:55-150) ----
namespace {

void layer_sims(spes_ctx* c, int l, int source) {
    const Layout& L = c->lay;
    const int M = L.M;
    const int64_t df = L.d * L.f;
    if (!c->gram_partial) {
        c->gram_chunks = 148 * 2;
        c->gram_partial = c->scratch.alloc<double>(static_cast<int64_t>(c->gram_chunks) * M * (M + 1) / 2);
        c->sim = c->scratch.alloc<double>(static_cast<int64_t>(M) * M);
        c->coef = c->scratch.alloc<double>(M);
        c->disp_partial = c->scratch.alloc<double>(148 * 8);
        c->peers_dev = c->scratch.alloc<int32_t>(M * M);
        c->layer_expert_offs = c->scratch.alloc<int64_t>(2 * M);
    }
    if (!c->h_merge) ck(cudaMallocHost(&c->h_merge, sizeof(spes_ctx::MergePin)), "pinned merge");
    int64_t* vo = c->h_merge->vo;
    for (int j = 0; j < M; ++j) vo[j] = L.off_expert(l, j) + (source == 1 ? df : 0);
    ck(cudaMemcpyAsync(c->layer_expert_offs + M, vo, 8 * M, cudaMemcpyHostToDevice, c->stream), "vo");
    spes_k::gram_partials(c->params, c->layer_expert_offs + M, M, df, df, source == 2 ? 1 : 0,
                          c->gram_partial, c->gram_chunks, c->stream);
    spes_k::gram_finish(c->gram_partial, M, c->gram_chunks, c->sim, c->stream);
}

// Sequential fp64 similarity row (exact reference order), for near-tie resolution.
void exact_sim_row(spes_ctx* c, int l, int source, int j, std::vector<double>& row) {
    const Layout& L = c->lay;
    const int M = L.M;
    const int64_t df = L.d * L.f;
    const int64_t D = source == 2 ? 2 * df : df;
    std::vector<std::vector<float>> w(M, std::vector<float>(D));
    for (int e = 0; e < M; ++e) {
        const int64_t o = L.off_expert(l, e);
        if (source == 0 || source == 2)
            ck(cudaMemcpy(w[e].data(), c->params + o, 4 * df, cudaMemcpyDeviceToHost), "D2H");
        if (source == 1)
            ck(cudaMemcpy(w[e].data(), c->params + o + df, 4 * df, cudaMemcpyDeviceToHost), "D2H");
        if (source == 2)
            ck(cudaMemcpy(w[e].data() + df, c->params + o + df, 4 * df, cudaMemcpyDeviceToHost), "D2H");
    }
    std::vector<double> norm(M);
    for (int e = 0; e < M; ++e) {
        double n2 = 0.0;
        for (int64_t i = 0; i < D; ++i) n2 += static_cast<double>(w[e][i]) * static_cast<double>(w[e][i]);
        norm[e] = std::sqrt(n2);
    }
    row.assign(M, 0.0);
    for (int e = 0; e < M; ++e) {
        double v = 0.0;
        if (norm[j] > 0.0 && norm[e] > 0.0) {
            double dot = 0.0;
            const int a = std::min(j, e), b = std::max(j, e);
            for (int64_t i = 0; i < D; ++i) dot += static_cast<double>(w[a][i]) * static_cast<double>(w[b][i]);
            v = dot / (norm[a] * norm[b]);
        }
        row[e] = v;
    }
}

// select_peers (merging.hpp:85-95): stable descending, K, ascending
std::vector<int> select_peers_host(const double* sim_row, int M, int j, int K) {
    std::vector<int> idx;
    for (int i = 0; i < M; ++i)
        if (i != j) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return sim_row[a] > sim_row[b]; });
    if (static_cast<int>(idx.size()) > K) idx.resize(K);
    std::sort(idx.begin(), idx.end());
    return idx;
}

bool near_tie_at_boundary(const double* sim_row, int M, int j, int K) {
    std::vector<double> v;
    for (int i = 0; i < M; ++i)
        if (i != j) v.push_back(sim_row[i]);
    if (static_cast<int>(v.size()) <= K) return false;
    std::sort(v.begin(), v.end(), std::greater<double>());
    const double a = v[K - 1], b = v[K];
    return std::fabs(a - b) <= 1e-9 * std::max(1.0, std::max(std::fabs(a), std::fabs(b)));
}

}  // namespace

spes_status spes_similarity(spes_ctx* c, int32_t layer, int32_t source, double* sim_out) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (c->lay.M < 2) throw std::invalid_argument("similarity_matrix: need M >= 2");
        if (layer < 0 || layer >= c->lay.L) throw std::out_of_range("similarity: bad layer");
        layer_sims(c, layer, source);
        ck(cudaMemcpyAsync(sim_out, c->sim, 8 * c->lay.M * c->lay.M, cudaMemcpyDeviceToHost, c->stream), "D2H sim");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

spes_status spes_merge(spes_ctx* c, const spes_merge_sched* sched, int32_t round0,
                       spes_merge_event* events, int32_t* peers_out, int32_t* n_events) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        CounterScope counter_scope(c);
        if (n_events) *n_events = 0;
        if (!spes_merge_at(sched, round0)) return;
        double alpha = 0.0;
        {
            spes_status s = spes_alpha_at(sched, round0, &alpha);
            if (s != SPES_OK) throw std::invalid_argument(g_last_error);
        }
        if (alpha <= 0.0) return;
        const Layout& L = c->lay;
        const int M = L.M;
        if (M < 2) throw std::invalid_argument("similarity_matrix: need M >= 2");
        const int K = std::min(sched->peers, M - 1);
        if (K < 1) throw std::invalid_argument("select_peers: need K >= 1");
        std::vector<double> sim(static_cast<size_t>(M) * M);
        for (int l = 0; l < L.L; ++l) {
            {
                Prof prof(c, "merge_similarity");
                layer_sims(c, l, sched->source);
                ck(cudaMemcpyAsync(c->h_merge->sim, c->sim, 8 * M * M, cudaMemcpyDeviceToHost,
                                   c->stream),
                   "D2H sim");
            }
            ck(cudaStreamSynchronize(c->stream), "sync");
            std::memcpy(sim.data(), c->h_merge->sim, 8 * M * M);
            std::vector<int32_t> peers(static_cast<size_t>(M) * K);
            std::vector<double> coef(M);
            for (int j = 0; j < M; ++j) {
                const double* row = sim.data() + static_cast<size_t>(j) * M;
                std::vector<double> exact;
                if (near_tie_at_boundary(row, M, j, K)) {
                    exact_sim_row(c, l, sched->source, j, exact);
                    row = exact.data();
                }
                auto p = select_peers_host(row, M, j, K);
                for (int q = 0; q < K; ++q) peers[static_cast<size_t>(j) * K + q] = p[q];
                coef[j] = alpha / static_cast<double>(p.size());
            }
            auto* hp = c->h_merge;
            for (int j = 0; j < M; ++j) hp->eo[j] = L.off_expert(l, j);
            std::memcpy(hp->peers, peers.data(), 4 * M * K);
            std::memcpy(hp->coef, coef.data(), 8 * M);
            const int nblocks = 148 * 4;
            {
                Prof prof(c, "merge_apply");
                ck(cudaMemcpyAsync(c->peers_dev, hp->peers, 4 * M * K, cudaMemcpyHostToDevice,
                                   c->stream),
                   "peers");
                ck(cudaMemcpyAsync(c->coef, hp->coef, 8 * M, cudaMemcpyHostToDevice, c->stream), "coef");
                ck(cudaMemcpyAsync(c->layer_expert_offs, hp->eo, 8 * M, cudaMemcpyHostToDevice,
                                   c->stream),
                   "eo");
                // the merged experts' bf16 operand copies are written from the same values
                // (no refresh pass over the experts afterwards)
                const spes_k::Shadows shm = shadows_of(c);
                spes_k::merge_apply(c->params, c->layer_expert_offs, M, L.per_expert(), c->peers_dev,
                                    K, c->coef, c->disp_partial, nblocks, c->stream, &shm, l * M);
                ck(cudaMemcpyAsync(hp->disp, c->disp_partial, 8 * nblocks, cudaMemcpyDeviceToHost,
                                   c->stream),
                   "disp");
            }
            ck(cudaStreamSynchronize(c->stream), "sync");
            double disp = 0.0;
            for (int i = 0; i < nblocks; ++i) disp += hp->disp[i];
            if (events) {
                events[l].layer = l;
                events[l].peers_k = K;
                events[l].alpha = alpha;
                events[l].displacement_sq = disp;
            }
            if (peers_out)
                std::memcpy(peers_out + static_cast<size_t>(l) * M * K, peers.data(), 4 * M * K);
        }
        ck(cudaStreamSynchronize(c->stream), "sync");
        if (n_events) *n_events = L.L;
    });
}

spes_status spes_counts(spes_ctx* c, int64_t* opt_state, int64_t* grad_scalars, int64_t* step) {
    return guard([&] {
        // the caller's model's units (|psi| + |Phi_i|, trainer.hpp:186-189)
        const int64_t nown = static_cast<int64_t>(c->node_experts[c->node].size());
        const int64_t Gu = c->ulay.psi() + c->ulay.L * nown * c->ulay.per_expert();
        if (opt_state) *opt_state = c->inner_sgd ? 0 : 2 * Gu;
        if (grad_scalars) *grad_scalars = Gu;
        if (step) *step = c->adam_step;
    });
}

spes_status spes_set_fused_optimizer(spes_ctx* c, int32_t on) {
    return guard([&] {
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->fused_opt = on != 0;  // group tables are rebuilt every step with the mode
    });
}

spes_status spes_set_inner_optimizer(spes_ctx* c, int32_t kind) {
    return guard([&] {
        if (kind != 0 && kind != 1)
            throw std::invalid_argument("inner optimizer: 0 (AdamW) or 1 (SGD)");
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->inner_sgd = kind == 1;
        drop_graph(c);  // the captured step holds the other optimizer placement
    });
}

spes_status spes_set_stream_overlap(spes_ctx* c, int32_t on) {
    return guard([&] {
        ck(cudaStreamSynchronize(c->stream), "sync");
        c->overlap_opt = on != 0;
        drop_graph(c);  // the captured step holds the other stream layout
    });
}

spes_status spes_read_grads(spes_ctx* c, float* host, int64_t n) {
    return guard([&] {
        if (n != c->ulay.total()) throw std::invalid_argument("read_grads: size mismatch");
        if (fused(c) && c->G > c->lay.psi())
            throw std::logic_error(
                "read_grads: owned-expert gradients are fused into the optimizer; call "
                "spes_set_fused_optimizer(ctx, 0) before the step to materialize them");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        std::vector<float> comp(c->G);
        ck(cudaMemcpyAsync(comp.data(), c->grads, 4 * c->G, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
        std::vector<float> full(c->padded ? static_cast<size_t>(c->lay.total()) : 0);
        float* dst = c->padded ? full.data() : host;
        std::memset(dst, 0, 4 * c->lay.total());
        for (const auto& s : c->segs_host)
            std::memcpy(dst + s.param_off, comp.data() + s.comp_off, 4 * s.len);
        if (c->padded) convert_layout(c->ulay, c->lay, full.data(), host, false);
    });
}

spes_status spes_debug_read(spes_ctx* c, const char* name, int32_t layer, void* host,
                            int64_t bytes) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const Layout& L = c->lay;
        const std::string n(name);
        if (c->T == 0 && n != "w1" && n != "w2")
            throw std::logic_error("debug_read: no step has run");
        const int64_t T = c->T, d = L.d, M = L.M, k = L.k;
        const void* src = nullptr;
        int64_t sz = 0;
        auto lay = [&]() -> LayerBufs& {
            if (layer < 0 || layer >= L.L) throw std::out_of_range("debug_read: bad layer");
            return c->layers[layer];
        };
        // [T x d] activations in the caller's hidden width (device rows may be padded)
        const int64_t du = c->ulay.d;
        auto rows_out = [&](const float* dev_rows) {
            if (bytes < 4 * T * du) throw std::invalid_argument("debug_read: buffer too small");
            ck(cudaMemcpy2D(host, 4 * du, dev_rows, 4 * d, 4 * du, T, cudaMemcpyDeviceToHost), "D2H");
        };
        if (n == "h") {
            if (layer < 0 || layer > L.L) throw std::out_of_range("debug_read: bad layer");
            if (layer == 0 && c->virtual_h0) {  // emb[inputs] (never materialized on device)
                if (bytes < 4 * T * du) throw std::invalid_argument("debug_read: buffer too small");
                std::vector<int32_t> in(static_cast<size_t>(T));
                ck(cudaMemcpy(in.data(), c->inputs, 4 * T, cudaMemcpyDeviceToHost), "D2H");
                float* out = static_cast<float*>(host);
                for (int64_t t = 0; t < T; ++t)
                    ck(cudaMemcpy(out + t * du, c->params + L.off_emb() + static_cast<int64_t>(in[t]) * d,
                                  4 * du, cudaMemcpyDeviceToHost),
                       "D2H emb row");
                return;
            }
            if (layer == L.L)
                throw std::invalid_argument(
                    "debug_read: the final hidden state is kept only as the bf16 head operand");
            rows_out(c->h[layer]);
            return;
        } else if (n == "w1" || n == "w2") {  // a layer's bf16 expert operand copies
            if (layer < 0 || layer >= L.L) throw std::out_of_range("debug_read: bad layer");
            const int64_t per_slot = n == "w1" ? L.d * 2 * L.f : L.f * L.d;
            const bf16* base = n == "w1" ? c->w1 : c->w2;
            src = base + per_slot * L.M * layer;
            sz = 2 * per_slot * L.M;
        } else if (n == "normed") {
            throw std::invalid_argument(
                "debug_read: normed is not stored on the training path (recomputed in "
                "backward); spes_kernel_router returns it");
        } else if (n == "logits") {
            src = lay().logits;
            sz = 4 * T * M;
        } else if (n == "probs") {
            src = lay().probs;
            sz = 4 * T * M;
        } else if (n == "topk_idx") {
            src = lay().topk_idx;
            sz = 4 * T * k;
        } else if (n == "topk_w") {
            src = lay().topk_w;
            sz = 4 * T * k;
        } else if (n == "counts") {
            src = lay().counts;
            sz = 4 * M;
        } else if (n == "pad_off") {
            src = lay().pad_off;
            sz = 4 * (M + 1);
        } else if (n == "row_token") {
            src = lay().row_token;
            sz = 4 * c->R_cap;
        } else if (n == "slot_row") {
            src = lay().slot_row;
            sz = 4 * T * k;
        } else if (n == "grad_h0") {  // gradient w.r.t. the embedding output (last step)
            rows_out(c->gh);
            return;
        } else if (n == "head_logits") {
            if (L.V == 256)  // the fused head-CE epilogue never writes fp32 logits
                throw std::logic_error("debug_read: head_logits are not materialised for V == 256");
            src = c->head_logits;
            sz = 4 * T * L.V;
        } else if (n == "y") {
            src = lay().y;
            sz = 4 * c->R_cap * d;
        } else if (n == "perm") {
            // token of each routed row, expert-major, without padding (model.hpp:314-318)
            std::vector<int32_t> rt(c->R_cap), po(M + 1);
            ck(cudaMemcpy(rt.data(), lay().row_token, 4 * c->R_cap, cudaMemcpyDeviceToHost), "D2H");
            ck(cudaMemcpy(po.data(), lay().pad_off, 4 * (M + 1), cudaMemcpyDeviceToHost), "D2H");
            std::vector<int32_t> out;
            for (int j = 0; j < M; ++j)
                for (int r = po[j]; r < po[j + 1]; ++r)
                    if (rt[r] >= 0) out.push_back(rt[r]);
            if (bytes < static_cast<int64_t>(4 * out.size())) throw std::invalid_argument("debug_read: buffer too small");
            std::memcpy(host, out.data(), 4 * out.size());
            return;
        } else {
            throw std::invalid_argument("debug_read: unknown buffer " + n);
        }
        if (bytes < sz) throw std::invalid_argument("debug_read: buffer too small");
        ck(cudaMemcpyAsync(host, src, sz, cudaMemcpyDeviceToHost, c->stream), "D2H");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

spes_status spes_profile(spes_ctx* c, int32_t enable) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        prof_collect(c);
        c->prof = enable != 0;
    });
}

spes_status spes_profile_reset(spes_ctx* c) {
    return guard([&] {
        prof_collect(c);
        std::fill(c->fam_ms.begin(), c->fam_ms.end(), 0.0);
        std::fill(c->fam_n.begin(), c->fam_n.end(), 0);
    });
}

int32_t spes_profile_count(spes_ctx* c) {
    prof_collect(c);
    return static_cast<int32_t>(c->fam_names.size());
}

spes_status spes_profile_get(spes_ctx* c, int32_t i, char* name64, double* total_ms,
                             int64_t* launches) {
    return guard([&] {
        prof_collect(c);
        if (i < 0 || i >= static_cast<int32_t>(c->fam_names.size()))
            throw std::out_of_range("profile: bad index");
        std::strncpy(name64, c->fam_names[i].c_str(), 63);
        name64[63] = 0;
        *total_ms = c->fam_ms[i];
        *launches = c->fam_n[i];
    });
}

void* spes_stream(spes_ctx* c) { return c->stream; }
int64_t spes_kernel_launches(spes_ctx* c) { return c->launches; }

// ---- kernel-level entry points ----
spes_status spes_kernel_router(const spes_model_cfg* cfg, const float* h, const float* gain,
                               const float* router, int64_t T, float* normed, float* logits,
                               float* probs, int32_t* topk_idx, float* topk_w, int32_t* counts,
                               int32_t* perm, int32_t cuda_device) {
    return guard([&] {
        ck(cudaSetDevice(cuda_device), "cudaSetDevice");
        const int64_t d = cfg->hidden;
        const int M = cfg->experts_total, k = cfg->experts_active;
        if (k < 1 || k > M || M > 64 || k > 8) throw std::invalid_argument("route: need 1 <= k <= M");
        if (d % 64) throw std::invalid_argument("router kernel: hidden must be a multiple of 64");
        DevMem D;
        float* dh = D.alloc<float>(T * d);
        float* dg = D.alloc<float>(d);
        float* dr = D.alloc<float>(d * M);
        float* dn = D.alloc<float>(T * d);
        float* dl = D.alloc<float>(T * M);
        float* dp = D.alloc<float>(T * M);
        int32_t* di = D.alloc<int32_t>(T * k);
        float* dw = D.alloc<float>(T * k);
        float* dlse = D.alloc<float>(T);
        float* dinv = D.alloc<float>(T);
        float* dden = D.alloc<float>(T);
        ck(cudaMemcpy(dh, h, 4 * T * d, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dg, gain, 4 * d, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dr, router, 4 * d * M, cudaMemcpyHostToDevice), "H2D");
        const int variant = spes_expf::host_variant_from(&expf);
        spes_k::router_forward(dh, nullptr, dg, dr, T, d, d, M, k, cfg->renormalize_after_topk,
                               cfg->rms_eps,
                               variant, dn, nullptr, dl, dp, di, dw, dlse, dinv, dden, 0);
        // routing plan for counts / permutation
        const int64_t R = rup(T * k + static_cast<int64_t>(M) * 128, 128);
        const int64_t nchunks = (T + 255) / 256;
        spes_k::RoutePlan rp{D.alloc<int32_t>(nchunks * M), D.alloc<int32_t>(M),
                             D.alloc<int32_t>(M + 1), D.alloc<float>(M), D.alloc<int32_t>(T * k),
                             D.alloc<int32_t>(R), D.alloc<float>(R), D.alloc<GemmGroup>(6 * M),
                             D.alloc<int32_t>(6)};
        spes_k::GroupBases gb{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 128, 128,
                              128, 128, 128, 128, 128};
        spes_k::route_plan(di, dw, T, M, k, R, rp, gb, 0);
        ck(cudaDeviceSynchronize(), "router kernel");
        if (normed) ck(cudaMemcpy(normed, dn, 4 * T * d, cudaMemcpyDeviceToHost), "D2H");
        if (logits) ck(cudaMemcpy(logits, dl, 4 * T * M, cudaMemcpyDeviceToHost), "D2H");
        if (probs) ck(cudaMemcpy(probs, dp, 4 * T * M, cudaMemcpyDeviceToHost), "D2H");
        if (topk_idx) ck(cudaMemcpy(topk_idx, di, 4 * T * k, cudaMemcpyDeviceToHost), "D2H");
        if (topk_w) ck(cudaMemcpy(topk_w, dw, 4 * T * k, cudaMemcpyDeviceToHost), "D2H");
        if (counts) ck(cudaMemcpy(counts, rp.counts, 4 * M, cudaMemcpyDeviceToHost), "D2H");
        if (perm) {
            std::vector<int32_t> rt(R), po(M + 1), sr(static_cast<size_t>(T * k));
            ck(cudaMemcpy(rt.data(), rp.row_token, 4 * R, cudaMemcpyDeviceToHost), "D2H");
            ck(cudaMemcpy(po.data(), rp.pad_off, 4 * (M + 1), cudaMemcpyDeviceToHost), "D2H");
            ck(cudaMemcpy(sr.data(), rp.slot_row, 4 * T * k, cudaMemcpyDeviceToHost), "D2H");
            // the plan's two views must agree: row_token[slot_row[t][s]] == t
            for (int64_t i = 0; i < T * k; ++i)
                if (sr[i] < 0 || sr[i] >= R || rt[sr[i]] != i / k)
                    throw std::runtime_error(
                        "route plan inconsistent: token " + std::to_string(i / k) + " slot " +
                        std::to_string(i % k) + " -> row " + std::to_string(sr[i]) +
                        " holding token " + std::to_string(sr[i] >= 0 && sr[i] < R ? rt[sr[i]] : -2));
            int64_t q = 0;
            for (int j = 0; j < M; ++j)
                for (int r = po[j]; r < po[j + 1]; ++r)
                    if (rt[r] >= 0) {
                        if (q >= T * k || (q > 0 && r > po[j] && rt[r - 1] >= rt[r] && rt[r - 1] >= 0))
                            throw std::runtime_error(
                                "route plan: row " + std::to_string(r) + " of expert " +
                                std::to_string(j) + " holds token " + std::to_string(rt[r]) +
                                " after " + std::to_string(r > 0 ? rt[r - 1] : -9) + " (entry " +
                                std::to_string(q) + " of " + std::to_string(T * k) + ")");
                        perm[q++] = rt[r];
                    }
            if (q != T * k)
                throw std::runtime_error("route plan: " + std::to_string(q) + " routed rows, expected " +
                                         std::to_string(T * k));
        }
    });
}

spes_status spes_kernel_adamw(float* theta, const float* grad, float* m, float* v, int64_t n,
                              const spes_adamw_cfg* o, int64_t step, int32_t cuda_device) {
    return guard([&] {
        ck(cudaSetDevice(cuda_device), "cudaSetDevice");
        if (n % 4) throw std::invalid_argument("adamw kernel: n must be a multiple of 4");
        DevMem D;
        float* dt = D.alloc<float>(n);
        float* dgr = D.alloc<float>(n);
        float* dm = D.alloc<float>(n);
        float* dv = D.alloc<float>(n);
        spes_k::AdamSeg seg{0, 0, n, 0, 0};
        auto* ds = D.alloc<spes_k::AdamSeg>(1);
        ck(cudaMemcpy(ds, &seg, sizeof(seg), cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dt, theta, 4 * n, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dgr, grad, 4 * n, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dm, m, 4 * n, cudaMemcpyHostToDevice), "H2D");
        ck(cudaMemcpy(dv, v, 4 * n, cudaMemcpyHostToDevice), "H2D");
        const float bc1 = 1.f - static_cast<float>(std::pow(o->beta1, static_cast<double>(step)));
        const float bc2 = 1.f - static_cast<float>(std::pow(o->beta2, static_cast<double>(step)));
        const float b1 = static_cast<float>(o->beta1), b2 = static_cast<float>(o->beta2);
        volatile float one = 1.f;
        const spes_k::AdamScalars a{static_cast<float>(o->lr), b1, b2, one - b1, one - b2,
                                    static_cast<float>(o->eps),
                                    static_cast<float>(o->weight_decay), bc1, bc2};
        auto* da = D.alloc<spes_k::AdamScalars>(1);
        ck(cudaMemcpy(da, &a, sizeof(a), cudaMemcpyHostToDevice), "H2D");
        spes_k::adamw(dt, dgr, dm, dv, spes_k::SegTable{ds, 1, n, 4}, 0, 1, da,
                      spes_k::Shadows{nullptr, nullptr, nullptr, 0, 0},
                      nullptr, 0);
        ck(cudaDeviceSynchronize(), "adamw kernel");
        ck(cudaMemcpy(theta, dt, 4 * n, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(m, dm, 4 * n, cudaMemcpyDeviceToHost), "D2H");
        ck(cudaMemcpy(v, dv, 4 * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

spes_status spes_kernel_owner_mean(const float* x, int32_t n_owners, int64_t n, float* out,
                                   int32_t cuda_device) {
    return guard([&] {
        ck(cudaSetDevice(cuda_device), "cudaSetDevice");
        DevMem D;
        float* dx = D.alloc<float>(n * n_owners);
        float* dout = D.alloc<float>(n);
        ck(cudaMemcpy(dx, x, 4 * n * n_owners, cudaMemcpyHostToDevice), "H2D");
        spes_k::owner_mean_strided(dx, n_owners, n, n, dout, 0);
        ck(cudaDeviceSynchronize(), "owner mean");
        ck(cudaMemcpy(out, dout, 4 * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

spes_status spes_kernel_expf(const float* x, float* y, int64_t n, int32_t cuda_device) {
    return guard([&] {
        ck(cudaSetDevice(cuda_device), "cudaSetDevice");
        DevMem D;
        float* dx = D.alloc<float>(n);
        float* dy = D.alloc<float>(n);
        ck(cudaMemcpy(dx, x, 4 * n, cudaMemcpyHostToDevice), "H2D");
        spes_k::expf_port_device(dx, dy, n, spes_expf::host_variant_from(&expf), 0);
        ck(cudaDeviceSynchronize(), "expf");
        ck(cudaMemcpy(y, dy, 4 * n, cudaMemcpyDeviceToHost), "D2H");
    });
}

void spes_host_expf_port(const float* x, float* y, int64_t n, int32_t variant) {
    const int v = variant == 0 ? spes_expf::host_variant_from(&expf) : variant - 1;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        y[i] = v ? spes_expf::expf_glibc<1>(x[i]) : spes_expf::expf_glibc<0>(x[i]);
}

int32_t spes_host_expf_variant(void) { return spes_expf::host_variant_from(&expf); }

}  // extern "C"

// spes_b200.hpp -- C++ host mirror of the reference's operator interface over the C ABI.
//
// RAII context + the reference's exception types. When the reference headers are on
// the include path (building inside /root/reference/proj), the
// drop-in overloads below take and return the reference's own types with the same
// signatures and semantics as
//   local_round  (proj/include/spes/trainer.hpp:143-145)
//   merge_model  (proj/include/spes/merging.hpp:138)
//   Server::aggregate (proj/src/protocol.cpp:197-251; collective here: every node calls)
#pragma once

#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "spes_b200.h"

namespace spes_b200 {

// Rethrow a status as the exception class the reference would have thrown.
inline void check(spes_status s) {
    if (s == SPES_OK) return;
    const std::string msg = spes_last_error();
    switch (s) {
        case SPES_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SPES_OUT_OF_RANGE: throw std::out_of_range(msg);
        case SPES_LOGIC_ERROR: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

class Context {
public:
    Context(const spes_model_cfg& cfg, int node, int n_nodes, int device,
            const void* nccl_id = nullptr)
        : cfg_(cfg), node_(node), n_nodes_(n_nodes) {
        check(spes_create(&cfg_, node, n_nodes, device, nccl_id, &ctx_));
    }
    ~Context() { spes_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    spes_ctx* get() const { return ctx_; }
    const spes_model_cfg& cfg() const { return cfg_; }
    int64_t param_count() const { return spes_param_count(&cfg_); }

    // node -> sorted experts, identical on every node (TrainMask of this node derived)
    void set_ownership(const std::vector<std::vector<int>>& owned) {
        std::vector<int32_t> offs{0}, ex;
        for (const auto& o : owned) {
            ex.insert(ex.end(), o.begin(), o.end());
            offs.push_back(static_cast<int32_t>(ex.size()));
        }
        if (ex.empty()) ex.push_back(0);
        check(spes_set_ownership(ctx_, offs.data(), ex.data()));
        owned_ = owned;
    }
    int node() const { return node_; }
    int n_nodes() const { return n_nodes_; }
    // empty until set_ownership
    const std::vector<std::vector<int>>& ownership() const { return owned_; }
    void load(const std::vector<float>& flat) {
        check(spes_load_params(ctx_, flat.data(), static_cast<int64_t>(flat.size())));
    }
    std::vector<float> read() const {
        std::vector<float> out(static_cast<size_t>(param_count()));
        check(spes_read_params(ctx_, out.data(), static_cast<int64_t>(out.size())));
        return out;
    }
    std::vector<spes_losses> local_round(const std::vector<int32_t>& tokens, int64_t B, int64_t S,
                                         int H, const std::vector<double>& lr,
                                         const spes_adamw_cfg& opt, bool carry_state = false) {
        std::vector<spes_losses> out(static_cast<size_t>(H));
        check(spes_local_round(ctx_, tokens.data(), B, S, H, lr.empty() ? nullptr : lr.data(), &opt,
                               carry_state ? 1 : 0, out.data()));
        return out;
    }
    spes_sync_stats sync() {
        spes_sync_stats st{};
        check(spes_sync(ctx_, &st));
        return st;
    }

private:
    spes_model_cfg cfg_;
    int node_ = 0, n_nodes_ = 1;
    std::vector<std::vector<int>> owned_;
    spes_ctx* ctx_ = nullptr;
};

}  // namespace spes_b200

#if defined(__has_include)
#if __has_include("spes/trainer.hpp") && __has_include("spes/merging.hpp")
#include "spes/merging.hpp"
#include "spes/trainer.hpp"

namespace spes_b200 {

inline spes_model_cfg to_c(const spes::ModelConfig& c) {
    spes_model_cfg o{};
    o.vocab = c.vocab;
    o.hidden = c.hidden;
    o.intermediate = c.intermediate;
    o.layers = c.layers;
    o.experts_total = c.experts_total;
    o.experts_active = c.experts_active;
    o.renormalize_after_topk = c.renormalize_after_topk;
    o.tied_head = c.tied_head;
    o.coeff_ce = c.loss.ce;
    o.coeff_lb = c.loss.lb;
    o.coeff_moe_z = c.loss.moe_z;
    o.coeff_z = c.loss.z;
    o.rms_eps = c.rms_eps;
    return o;
}

inline std::vector<float> flatten(const spes::ModelParams& p) {
    std::vector<float> out;
    for (const auto& b : spes::enumerate_blocks(p.config)) {
        const auto& t = spes::block_tensor(p, b);
        out.insert(out.end(), t.data.begin(), t.data.end());
    }
    return out;
}

inline void unflatten(const std::vector<float>& flat, spes::ModelParams& p) {
    size_t off = 0;
    for (const auto& b : spes::enumerate_blocks(p.config)) {
        auto& t = spes::block_tensor(p, b);
        std::memcpy(t.data.data(), flat.data() + off, t.data.size() * sizeof(float));
        off += t.data.size();
    }
}

// Drop-in for spes::local_round (trainer.hpp:143-222): the H steps run on the device (one
// spes_local_step per batch, each with its own (B, S)); inner optimizer AdamW (fresh state
// per call unless carry_state) or SGD (trainer.hpp:197-204). record_trace (trainer.hpp:
// 183-219) reads each step's gradients and parameters back and forms the same statistics
// on the host in the reference's order: update_norms = sqrt(sum over trainable blocks of
// double(g)^2), grad_sum = per trainable block float sum over steps, drift_sq = sum over
// all blocks of (double(theta) - double(theta_global))^2.
inline spes::LocalRoundResult local_round(Context& ctx, const spes::ModelParams& global,
                                          const spes::BatchProvider& next_batch,
                                          const spes::LocalRoundConfig& cfg,
                                          const spes::TrainMask& mask, bool carry_state = false) {
    if (cfg.steps < 1) throw std::invalid_argument("local_round: need H >= 1");
    // The TrainMask must be this node's row of the context's ownership map (the map is
    // global because the sparse sync needs every node's owner set). A single-node
    // context adopts the mask as its map.
    if (mask.node_id != ctx.node())
        throw std::invalid_argument("b200 local_round: mask.node_id differs from the context's node");
    if (ctx.n_nodes() == 1 && (ctx.ownership().empty() || ctx.ownership()[0] != mask.owned_experts))
        ctx.set_ownership({mask.owned_experts});
    else if (ctx.ownership().empty() ||
             ctx.ownership()[static_cast<size_t>(ctx.node())] != mask.owned_experts)
        throw std::invalid_argument("b200 local_round: mask differs from the context's ownership map");
    const bool sgd = cfg.inner == spes::InnerOpt::SGD;
    check(spes_set_inner_optimizer(ctx.get(), sgd ? 1 : 0));
    if (cfg.record_trace) check(spes_set_fused_optimizer(ctx.get(), 0));  // gradients readable
    const std::vector<float> theta0 = flatten(global);
    ctx.load(theta0);
    check(spes_round_begin(ctx.get(), carry_state ? 1 : 0));
    const auto blocks = spes::enumerate_blocks(global.config);
    std::vector<size_t> offs;  // flat offset of every block
    {
        size_t o = 0;
        for (const auto& b : blocks) {
            offs.push_back(o);
            o += static_cast<size_t>(spes::block_tensor(global, b).numel());
        }
    }
    spes::LocalRoundResult res;
    res.params = global;
    spes_adamw_cfg opt{cfg.opt.lr, cfg.opt.beta1, cfg.opt.beta2, cfg.opt.eps,
                       cfg.opt.weight_decay};
    std::vector<float> g(theta0.size());
    for (int h = 0; h < cfg.steps; ++h) {
        if (cfg.lr_at) opt.lr = cfg.lr_at(cfg.first_step + h);
        spes::Batch b = next_batch();
        if (static_cast<int64_t>(b.tokens.size()) != b.batch * (b.seq + 1))
            throw std::invalid_argument("batch: tokens must hold batch * (seq + 1) ids");
        spes_losses l{};
        const spes_status st = spes_local_step(ctx.get(), b.tokens.data(), b.batch, b.seq, &opt, &l);
        if (st == SPES_RUNTIME_ERROR)  // the reference reports the step (trainer.hpp:166-167)
            throw std::runtime_error("local_round: non-finite loss at step " + std::to_string(h));
        check(st);
        res.step_losses.push_back({l.total, l.ce, l.lb, l.moe_z, l.z});
        if (cfg.record_trace) {
            check(spes_read_grads(ctx.get(), g.data(), static_cast<int64_t>(g.size())));
            double n2 = 0.0;
            size_t q = 0;
            for (size_t i = 0; i < blocks.size(); ++i) {
                if (!mask.trainable(blocks[i])) continue;
                const size_t n = static_cast<size_t>(spes::block_tensor(global, blocks[i]).numel());
                const float* gb = g.data() + offs[i];
                for (size_t j = 0; j < n; ++j) n2 += static_cast<double>(gb[j]) * gb[j];
                if (q == res.grad_sum.size()) {
                    spes::Tensor t = spes::Tensor::zeros(spes::block_tensor(global, blocks[i]).shape);
                    std::memcpy(t.data.data(), gb, n * sizeof(float));
                    res.grad_sum.push_back({i, std::move(t)});
                } else {
                    auto& acc = res.grad_sum[q].grad.data;
                    for (size_t j = 0; j < n; ++j) acc[j] += gb[j];
                }
                ++q;
            }
            res.update_norms.push_back(std::sqrt(n2));
            const std::vector<float> now = ctx.read();
            double d2 = 0.0;
            for (size_t j = 0; j < now.size(); ++j) {
                const double dd = static_cast<double>(now[j]) - static_cast<double>(theta0[j]);
                d2 += dd * dd;
            }
            res.drift_sq.push_back(d2);
        }
    }
    unflatten(ctx.read(), res.params);
    int64_t opt_state = 0, grads = 0, step = 0;
    check(spes_counts(ctx.get(), &opt_state, &grads, &step));
    res.grad_scalar_count = grads;
    return res;
}

// Drop-in for spes::merge_model (merging.hpp:138-150) on the context's model.
inline std::vector<spes::MergeEvent> merge_model(Context& ctx, spes::ModelParams& params,
                                                 const spes::MergeSchedule& sched, int round) {
    spes_merge_sched s{sched.warmup_rounds, sched.interval, sched.alpha0, sched.peers,
                       static_cast<int32_t>(sched.source)};
    ctx.load(flatten(params));
    const int L = params.config.layers, M = params.config.experts_total;
    const int K = std::max(1, std::min(sched.peers, M - 1));
    std::vector<spes_merge_event> ev(static_cast<size_t>(L));
    std::vector<int32_t> peers(static_cast<size_t>(L) * M * K);
    int32_t n = 0;
    check(spes_merge(ctx.get(), &s, round, ev.data(), peers.data(), &n));
    std::vector<spes::MergeEvent> out;
    for (int l = 0; l < n; ++l) {
        spes::MergeEvent e;
        e.layer = ev[l].layer;
        e.alpha = ev[l].alpha;
        e.displacement_sq = ev[l].displacement_sq;
        for (int j = 0; j < M; ++j)
            e.peer_sets.emplace_back(peers.begin() + (static_cast<size_t>(l) * M + j) * K,
                                     peers.begin() + (static_cast<size_t>(l) * M + j + 1) * K);
        out.push_back(std::move(e));
    }
    if (n > 0) unflatten(ctx.read(), params);
    return out;
}

}  // namespace spes_b200
#endif
#endif

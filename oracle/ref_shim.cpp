// ref_shim.cpp -- C ABI over the UNMODIFIED reference (/root/reference/proj), built
// by oracle/Makefile into oracle/_ref/libspes_ref.so. TEST INFRASTRUCTURE ONLY:
// it pins the C restatement (spes_oracle.c) bit-for-bit and is the reference arm
// / cpu_baseline of bench.py. It calls the reference's own public API; nothing
// of the reference is copied here.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <span>
#include <vector>

#include "spes/corpus.hpp"
#include "spes/experiment.hpp"
#include "spes/merging.hpp"
#include "spes/model.hpp"
#include "spes/protocol.hpp"
#include "spes/trainer.hpp"
#include "spes/wire.hpp"

#include "../include/spes_b200.h"

using namespace spes;

namespace {

ModelConfig to_cfg(const spes_model_cfg* c) {
    ModelConfig m;
    m.vocab = c->vocab;
    m.hidden = c->hidden;
    m.intermediate = c->intermediate;
    m.layers = c->layers;
    m.experts_total = c->experts_total;
    m.experts_active = c->experts_active;
    m.renormalize_after_topk = c->renormalize_after_topk != 0;
    m.tied_head = c->tied_head != 0;
    m.loss.ce = c->coeff_ce;
    m.loss.lb = c->coeff_lb;
    m.loss.moe_z = c->coeff_moe_z;
    m.loss.z = c->coeff_z;
    m.rms_eps = c->rms_eps;
    return m;
}

ModelParams from_flat(const ModelConfig& c, const float* flat) {
    ModelParams p = init_model<float>(c, 0, 0.0);
    size_t off = 0;
    for (const auto& b : enumerate_blocks(c)) {
        Tensor& t = block_tensor(p, b);
        std::memcpy(t.data.data(), flat + off, t.data.size() * sizeof(float));
        off += t.data.size();
    }
    return p;
}

void to_flat(const ModelParams& p, float* flat) {
    size_t off = 0;
    for (const auto& b : enumerate_blocks(p.config)) {
        const Tensor& t = block_tensor(p, b);
        std::memcpy(flat + off, t.data.data(), t.data.size() * sizeof(float));
        off += t.data.size();
    }
}

TrainMask mask_from(const ModelConfig& c, const uint8_t* trainable_expert, int node) {
    TrainMask m;
    m.node_id = node;
    for (int j = 0; j < c.experts_total; ++j)
        if (trainable_expert[j]) m.owned_experts.push_back(j);
    return m;
}

Batch batch_from(const int32_t* tokens, int64_t B, int64_t S) {
    Batch b;
    b.batch = B;
    b.seq = S;
    b.tokens.assign(tokens, tokens + B * (S + 1));
    return b;
}

}  // namespace

extern "C" {

void ref_set_parallel(int on) { kernels::set_parallel(on != 0); }

int64_t ref_param_count(const spes_model_cfg* c) {
    auto pc = param_counts(to_cfg(c));
    return pc.shared + pc.experts_total;
}

// init_model<float>(cfg, seed, std) (model.hpp:153-173)
void ref_init_model(const spes_model_cfg* c, uint64_t seed, double init_std, float* out) {
    to_flat(init_model<float>(to_cfg(c), seed, init_std), out);
}

// build_loss + backward (model.hpp:252-374); routing of every layer (model.hpp:185-216)
int ref_forward_backward(const spes_model_cfg* c, const float* params, const int32_t* tokens,
                         int64_t B, int64_t S, const uint8_t* trainable_expert, float* grads,
                         double* losses, float* probs, int32_t* topk_idx, float* topk_w) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams p = from_flat(cfg, params);
        TrainMask mask = mask_from(cfg, trainable_expert, 0);
        auto lg = build_loss(p, batch_from(tokens, B, S),
                             [&mask](const BlockDesc& b) { return mask.trainable(b); });
        losses[0] = lg.g.value(lg.total).data[0];
        losses[1] = lg.g.value(lg.ce).data[0];
        losses[2] = lg.g.value(lg.lb).data[0];
        losses[3] = lg.g.value(lg.moe_z).data[0];
        losses[4] = lg.g.value(lg.z).data[0];
        lg.g.backward(lg.total);
        auto blocks = enumerate_blocks(cfg);
        size_t off = 0;
        for (size_t i = 0; i < blocks.size(); ++i) {
            Tensor g = lg.g.grad(lg.block_leaves[i]);
            std::memcpy(grads + off, g.data.data(), g.data.size() * sizeof(float));
            off += g.data.size();
        }
        const int64_t T = B * S;
        const int M = cfg.experts_total, k = cfg.experts_active;
        for (size_t l = 0; l < lg.routing.size(); ++l) {
            const auto& rd = lg.routing[l];
            if (probs) std::memcpy(probs + l * T * M, rd.probs.data.data(), T * M * sizeof(float));
            for (int64_t t = 0; t < T; ++t)
                for (int s = 0; s < k; ++s) {
                    if (topk_idx) topk_idx[(l * T + t) * k + s] = rd.selected[t][s];
                    if (topk_w) topk_w[(l * T + t) * k + s] = rd.weights[t][s];
                }
        }
        return 0;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (...) {
        return 1;
    }
}

// local_round (trainer.hpp:143-222) with a fresh MaskedAdamW and per-step lr; seconds (if
// not null) receives the wall time of the reference's local_round call alone (the flat <->
// ModelParams conversions of this shim excluded).
static int local_round_impl(const spes_model_cfg* c, float* params, const int32_t* tokens,
                            int64_t B, int64_t S, int32_t H, const double* lr,
                            const spes_adamw_cfg* opt, const uint8_t* trainable_expert,
                            double* losses, double* seconds) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams p = from_flat(cfg, params);
        TrainMask mask = mask_from(cfg, trainable_expert, 0);
        int draw = 0;
        BatchProvider next = [&]() {
            return batch_from(tokens + static_cast<int64_t>(draw++) * B * (S + 1), B, S);
        };
        LocalRoundConfig rc;
        rc.steps = H;
        rc.opt.lr = opt->lr;
        rc.opt.beta1 = opt->beta1;
        rc.opt.beta2 = opt->beta2;
        rc.opt.eps = opt->eps;
        rc.opt.weight_decay = opt->weight_decay;
        if (lr) rc.lr_at = [lr](int64_t s) { return lr[s]; };
        rc.first_step = 0;
        const auto t0 = std::chrono::steady_clock::now();
        auto res = local_round(p, next, rc, mask);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (size_t h = 0; h < res.step_losses.size(); ++h) {
            losses[5 * h + 0] = res.step_losses[h].total;
            losses[5 * h + 1] = res.step_losses[h].ce;
            losses[5 * h + 2] = res.step_losses[h].lb;
            losses[5 * h + 3] = res.step_losses[h].moe_z;
            losses[5 * h + 4] = res.step_losses[h].z;
        }
        to_flat(res.params, params);
        return 0;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::runtime_error&) {
        return 3;
    } catch (...) {
        return 1;
    }
}

int ref_local_round(const spes_model_cfg* c, float* params, const int32_t* tokens, int64_t B,
                    int64_t S, int32_t H, const double* lr, const spes_adamw_cfg* opt,
                    const uint8_t* trainable_expert, double* losses) {
    return local_round_impl(c, params, tokens, B, S, H, lr, opt, trainable_expert, losses, nullptr);
}

int ref_local_round_timed(const spes_model_cfg* c, float* params, const int32_t* tokens, int64_t B,
                          int64_t S, int32_t H, const double* lr, const spes_adamw_cfg* opt,
                          const uint8_t* trainable_expert, double* losses, double* seconds) {
    return local_round_impl(c, params, tokens, B, S, H, lr, opt, trainable_expert, losses, seconds);
}

// Reference-arm timing (bench.py): local_round (H=1, fresh MaskedAdamW) from the same global
// model at S1 and then S2 tokens (B=1; tokens1 / tokens2 hold S+1 ids), each timed around
// the reference's local_round call alone; the model is converted from the flat vector once.
int ref_local_round_pair_timed(const spes_model_cfg* c, const float* params,
                               const int32_t* tokens1, int64_t S1, const int32_t* tokens2,
                               int64_t S2, const spes_adamw_cfg* opt,
                               const uint8_t* trainable_expert, double* seconds2) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams p = from_flat(cfg, params);
        TrainMask mask = mask_from(cfg, trainable_expert, 0);
        LocalRoundConfig rc;
        rc.steps = 1;
        rc.opt.lr = opt->lr;
        rc.opt.beta1 = opt->beta1;
        rc.opt.beta2 = opt->beta2;
        rc.opt.eps = opt->eps;
        rc.opt.weight_decay = opt->weight_decay;
        for (int i = 0; i < 2; ++i) {
            const int32_t* tk = i == 0 ? tokens1 : tokens2;
            const int64_t S = i == 0 ? S1 : S2;
            BatchProvider next = [&]() { return batch_from(tk, 1, S); };
            const auto t0 = std::chrono::steady_clock::now();
            auto res = local_round(p, next, rc, mask);
            seconds2[i] =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (!std::isfinite(res.step_losses.at(0).total)) return 3;
        }
        return 0;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::runtime_error&) {
        return 3;
    } catch (...) {
        return 1;
    }
}

// Server::aggregate through the reference's public protocol API (protocol.cpp:56-251):
// HELLO from every node, then each node's LocalUpdate with sparse_update_blocks under
// param_partition ownership. Result: the server's global model after round 1.
int ref_aggregate_partition(const spes_model_cfg* c, int32_t N, const float* node_params,
                            const float* global_in, float* global_out) {
    try {
        SyncConfig sc;
        sc.model = to_cfg(c);
        sc.nodes = N;
        sc.rounds = 1;
        sc.config_hash = 0;
        sc.merge.warmup_rounds = 0;
        ModelParams init = from_flat(sc.model, global_in);
        Server s(sc, init);
        auto part = param_partition(sc.model, N);
        auto frame = [](MsgKind kind, uint32_t round, std::vector<uint8_t> payload) {
            WireMessage m;
            m.kind = kind;
            m.round = round;
            m.payload = std::move(payload);
            return encode_message(m);
        };
        for (int n = 0; n < N; ++n) {
            HelloPayload h;
            h.node_id = static_cast<uint32_t>(n);
            h.config_hash = 0;
            auto bytes = frame(MsgKind::Hello, 0, encode_hello(h));
            s.on_bytes(n, bytes);
        }
        const int64_t P = ref_param_count(c);
        for (int n = 0; n < N; ++n) {
            ModelParams local = from_flat(sc.model, node_params + static_cast<int64_t>(n) * P);
            TrainMask m;
            m.node_id = n;
            m.owned_experts = part[static_cast<size_t>(n)];
            auto bytes = frame(MsgKind::LocalUpdate, 1, encode_blocks(sparse_update_blocks(local, m)));
            s.on_bytes(n, bytes);
        }
        to_flat(s.global(), global_out);
        return 0;
    } catch (...) {
        return 1;
    }
}

void ref_similarity(const spes_model_cfg* c, const float* params, int32_t layer, int32_t source,
                    double* sim) {
    ModelConfig cfg = to_cfg(c);
    ModelParams p = from_flat(cfg, params);
    auto s = similarity_matrix(p.experts[static_cast<size_t>(layer)],
                               static_cast<SimilaritySource>(source));
    std::memcpy(sim, s.a.data(), s.a.size() * sizeof(double));
}

int32_t ref_select_peers(const double* sim, int32_t M, int32_t j, int32_t K, int32_t* peers) {
    SimilarityMatrix s;
    s.experts = M;
    s.a.assign(sim, sim + static_cast<int64_t>(M) * M);
    auto v = select_peers(s, j, K);
    for (size_t i = 0; i < v.size(); ++i) peers[i] = v[i];
    return static_cast<int32_t>(v.size());
}

int32_t ref_merge_model(const spes_model_cfg* c, float* params, const spes_merge_sched* sch,
                        int32_t round, spes_merge_event* events, int32_t* peers) {
    ModelConfig cfg = to_cfg(c);
    ModelParams p = from_flat(cfg, params);
    MergeSchedule s;
    s.warmup_rounds = sch->warmup_rounds;
    s.interval = sch->interval;
    s.alpha0 = sch->alpha0;
    s.peers = sch->peers;
    s.source = static_cast<SimilaritySource>(sch->source);
    auto evs = merge_model(p, s, round);
    for (size_t l = 0; l < evs.size(); ++l) {
        if (events) {
            events[l].layer = evs[l].layer;
            events[l].alpha = evs[l].alpha;
            events[l].displacement_sq = evs[l].displacement_sq;
            events[l].peers_k = evs[l].peer_sets.empty() ? 0 : (int32_t)evs[l].peer_sets[0].size();
        }
        if (peers) {
            int32_t K = evs[l].peer_sets.empty() ? 0 : (int32_t)evs[l].peer_sets[0].size();
            for (int j = 0; j < cfg.experts_total; ++j)
                for (int q = 0; q < K; ++q)
                    peers[(l * cfg.experts_total + j) * K + q] = evs[l].peer_sets[j][q];
        }
    }
    to_flat(p, params);
    return static_cast<int32_t>(evs.size());
}

// One MaskedAdamW step from a fresh state (trainer.hpp:56-94).
int ref_adamw_first_step(const spes_model_cfg* c, float* params, const float* grads,
                         const uint8_t* trainable_expert, const spes_adamw_cfg* opt) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams p = from_flat(cfg, params);
        TrainMask mask = mask_from(cfg, trainable_expert, 0);
        MaskedAdamW o(cfg, mask);
        AdamWConfig ac;
        ac.lr = opt->lr;
        ac.beta1 = opt->beta1;
        ac.beta2 = opt->beta2;
        ac.eps = opt->eps;
        ac.weight_decay = opt->weight_decay;
        std::vector<GradBlock> gb;
        auto blocks = enumerate_blocks(cfg);
        size_t off = 0;
        for (size_t i = 0; i < blocks.size(); ++i) {
            int64_t n = Tensor::numel_of(blocks[i].shape);
            if (mask.trainable(blocks[i]))
                gb.push_back({i, Tensor(blocks[i].shape,
                                        std::vector<float>(grads + off, grads + off + n))});
            off += n;
        }
        o.step(p, gb, ac);
        to_flat(p, params);
        return 0;
    } catch (const std::logic_error&) {
        return 3;
    } catch (...) {
        return 1;
    }
}

double ref_lr_at(double peak, double min_frac, int64_t warmup, int64_t total, int64_t step) {
    LrSchedule s;
    s.peak = peak;
    s.min_frac = min_frac;
    s.warmup_steps = warmup;
    s.total_steps = total;
    return s.at(step);
}

void ref_param_partition(const spes_model_cfg* c, int32_t N, int32_t* node_offsets,
                         int32_t* experts) {
    auto part = param_partition(to_cfg(c), N);
    int32_t q = 0;
    node_offsets[0] = 0;
    for (int n = 0; n < N; ++n) {
        for (int e : part[static_cast<size_t>(n)]) experts[q++] = e;
        node_offsets[n + 1] = q;
    }
}

}  // extern "C"

// ---- wire / checkpoint format (proj/src/wire.cpp) ----
namespace {
const char* proto_name(ProtoError e) {
    switch (e) {
        case ProtoError::BadMagic: return "BadMagic";
        case ProtoError::BadVersion: return "BadVersion";
        case ProtoError::UnknownKind: return "UnknownKind";
        case ProtoError::Truncated: return "Truncated";
        case ProtoError::LengthMismatch: return "LengthMismatch";
        case ProtoError::MalformedPayload: return "MalformedPayload";
        case ProtoError::ConfigMismatch: return "ConfigMismatch";
        case ProtoError::RoundMismatch: return "RoundMismatch";
        case ProtoError::DuplicatePush: return "DuplicatePush";
        case ProtoError::NotOwnedBlock: return "NotOwnedBlock";
        case ProtoError::UnexpectedMessage: return "UnexpectedMessage";
        case ProtoError::BarrierViolation: return "BarrierViolation";
        case ProtoError::Timeout: return "Timeout";
    }
    return "?";
}
void put_err(char* err, int cap, const std::string& m) {
    if (err && cap > 0) std::snprintf(err, static_cast<size_t>(cap), "%s", m.c_str());
}
}  // namespace

extern "C" {
// encode_blocks(model_to_blocks(params)) -> out; returns the byte count (or needed size)
int64_t ref_encode_model(const spes_model_cfg* c, const float* params, uint8_t* out, int64_t cap) {
    ModelConfig cfg = to_cfg(c);
    auto bytes = encode_blocks(model_to_blocks(from_flat(cfg, params)));
    if (out && cap >= static_cast<int64_t>(bytes.size())) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<int64_t>(bytes.size());
}
// blocks_into_model(decode_blocks(payload)); 0 ok, 1 ProtocolError ("[Code] msg"), 2 other
int ref_decode_model(const spes_model_cfg* c, const uint8_t* payload, int64_t len, float* params,
                     char* err, int errcap) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams p = init_model<float>(cfg, 0, 0.0);
        blocks_into_model(p, decode_blocks(std::span<const uint8_t>(payload, static_cast<size_t>(len))));
        to_flat(p, params);
        return 0;
    } catch (const ProtocolError& e) {
        put_err(err, errcap, std::string("[") + proto_name(e.code()) + "] " + e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what());
        return 2;
    }
}
int ref_write_checkpoint(const spes_model_cfg* c, const float* params, const char* path,
                         uint64_t round) {
    try {
        write_checkpoint(path, from_flat(to_cfg(c), params), round);
        return 0;
    } catch (...) {
        return 2;
    }
}
int ref_read_checkpoint(const spes_model_cfg* c, const char* path, float* params, uint64_t* round,
                        char* err, int errcap) {
    try {
        ModelConfig cfg = to_cfg(c);
        auto [blocks, r] = read_checkpoint(path);
        ModelParams p = init_model<float>(cfg, 0, 0.0);
        blocks_into_model(p, blocks);
        to_flat(p, params);
        *round = r;
        return 0;
    } catch (const ProtocolError& e) {
        put_err(err, errcap, std::string("[") + proto_name(e.code()) + "] " + e.what());
        return 1;
    } catch (const std::exception& e) {
        put_err(err, errcap, e.what());
        return 2;
    }
}
}  // extern "C"

// ---- OuterOptimizer (trainer.hpp:228-271): persistent handle (Nesterov state) ----
extern "C" {
void* ref_outer_create(int32_t kind, double lr, double momentum) {
    return new OuterOptimizer(kind == 0 ? OuterKind::SGD : OuterKind::Nesterov, lr, momentum);
}
void ref_outer_destroy(void* h) { delete static_cast<OuterOptimizer*>(h); }
// theta (in/out, flat), locals N x P flat
int ref_outer_step(void* h, const spes_model_cfg* c, float* theta, const float* locals, int32_t N) {
    try {
        ModelConfig cfg = to_cfg(c);
        ModelParams t = from_flat(cfg, theta);
        const int64_t P = ref_param_count(c);
        std::vector<ModelParams> ls;
        for (int32_t i = 0; i < N; ++i) ls.push_back(from_flat(cfg, locals + i * P));
        std::vector<const ModelParams*> ptrs;
        for (auto& l : ls) ptrs.push_back(&l);
        static_cast<OuterOptimizer*>(h)->step(t, ptrs);
        to_flat(t, theta);
        return 0;
    } catch (...) {
        return 2;
    }
}
}  // extern "C"

// ---- upcycle_from_dense (model.hpp:415-460) ----
extern "C" int ref_upcycle(const spes_model_cfg* dense_cfg, const float* dense, int32_t m,
                           double noise_frac, double noise_std, uint64_t seed, float* out) {
    try {
        ModelConfig cfg = to_cfg(dense_cfg);
        ModelParams up = upcycle_from_dense(from_flat(cfg, dense), m, noise_frac, noise_std, seed);
        to_flat(up, out);
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 2;
    }
}

// ---- corpus.cpp: gen_corpus / shard_corpus / make_batch_provider ----
extern "C" {
int ref_gen_corpus(int64_t vocab, int64_t seq, int32_t sources, int64_t sequences, uint64_t seed,
                   double skew, int32_t* tokens, int32_t* source_id) {
    try {
        SyntheticCorpus c = gen_corpus(vocab, seq, sources, sequences, seed, skew);
        std::memcpy(tokens, c.tokens.data(), sizeof(int32_t) * c.tokens.size());
        for (size_t i = 0; i < c.source_id.size(); ++i) source_id[i] = c.source_id[i];
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}
// shards flattened: order + node offsets (N + 1)
int ref_shard_corpus(int64_t vocab, int64_t seq, int32_t sources, int64_t sequences,
                     uint64_t cseed, int32_t nodes, int32_t by_source, uint64_t seed,
                     int64_t* order, int64_t* offsets) {
    SyntheticCorpus c = gen_corpus(vocab, seq, sources, sequences, cseed, 0.0);
    auto sh = shard_corpus(c, nodes, by_source ? ShardPolicy::BySource : ShardPolicy::Random, seed);
    int64_t k = 0;
    offsets[0] = 0;
    for (size_t i = 0; i < sh.size(); ++i) {
        for (int64_t r : sh[i]) order[k++] = r;
        offsets[i + 1] = k;
    }
    return 0;
}
// H batches of the provider over a shard -> tokens H x B x (S+1)
int ref_batches(int64_t vocab, int64_t seq, int32_t sources, int64_t sequences, uint64_t cseed,
                const int64_t* shard, int64_t n, int64_t batch, uint64_t seed, int32_t H,
                int32_t* out) {
    SyntheticCorpus c = gen_corpus(vocab, seq, sources, sequences, cseed, 0.0);
    BatchProvider p = make_batch_provider(c, std::vector<int64_t>(shard, shard + n), batch, seed);
    for (int32_t h = 0; h < H; ++h) {
        Batch b = p();
        std::memcpy(out + static_cast<int64_t>(h) * batch * (seq + 1), b.tokens.data(),
                    sizeof(int32_t) * b.tokens.size());
    }
    return 0;
}
}  // extern "C"

// ---- CommLedger of an in-process protocol run (protocol.hpp:29-52, protocol.cpp:56-175,
// run_inproc :368-405), SURVEY §8(f) f3 -------------------------------------------------
extern "C" int ref_run_inproc_ledger(const spes_model_cfg* c, int32_t N, int32_t rounds,
                                     int32_t H, int64_t B, int64_t S, int32_t diloco,
                                     uint64_t seed, int32_t* nodes_out, int32_t* rounds_out,
                                     uint64_t* up_out, uint64_t* down_out, int32_t cap,
                                     int32_t* n_out, uint64_t* totals) {
    try {
        SyncConfig sc;
        sc.model = to_cfg(c);
        sc.nodes = N;
        sc.rounds = rounds;
        sc.diloco = diloco != 0;
        sc.config_hash = 7;
        sc.merge.warmup_rounds = 0;
        std::vector<float> flat(static_cast<size_t>(ref_param_count(c)));
        ref_init_model(c, seed, 0.02, flat.data());
        ModelParams init = from_flat(sc.model, flat.data());
        Worker::Options wo;
        wo.round.steps = H;
        std::vector<int32_t> toks(static_cast<size_t>(B * (S + 1)));
        for (size_t i = 0; i < toks.size(); ++i)
            toks[i] = static_cast<int32_t>((i * 2654435761ull + seed) % static_cast<uint64_t>(c->vocab));
        auto provider = [&](int) -> BatchProvider {
            return [&]() { return batch_from(toks.data(), B, S); };
        };
        RunResult r = run_inproc(sc, init, wo, provider);
        int32_t n = 0;
        for (const auto& [key, e] : r.ledger.per_node_round) {
            if (n < cap) {
                nodes_out[n] = key.first;
                rounds_out[n] = key.second;
                up_out[n] = e.up;
                down_out[n] = e.down;
            }
            ++n;
        }
        *n_out = n;
        totals[0] = r.ledger.total_up;
        totals[1] = r.ledger.total_down;
        totals[2] = r.ledger.pushes;
        totals[3] = r.ledger.broadcasts;
        return 0;
    } catch (...) {
        return 1;
    }
}

// ---- metrics.csv of run_experiment (experiment.cpp:270-420), SURVEY §8(f) f3 ----
struct RefRoundRow {
    int32_t round;
    double mean_total, mean_ce, mean_lb, mean_moe_z, mean_z, merge_displacement_sq;
    uint64_t bytes_up, bytes_down;
};

extern "C" int ref_run_experiment(const spes_model_cfg* c, int32_t nodes, int32_t H,
                                  int32_t rounds, int64_t batch, int64_t seq_len,
                                  const char* out_root, const char* name, RefRoundRow* rows,
                                  int32_t cap, int32_t* n_out, int64_t* tokens_per_round) {
    try {
        ExperimentConfig ec;
        ec.name = name;
        ec.model = to_cfg(c);
        ec.paradigm = Paradigm::Spes;
        ec.nodes = nodes;
        ec.local_steps = H;
        ec.rounds = rounds;
        ec.batch = batch;
        ec.seq_len = seq_len;
        ec.corpus_sequences = 64;
        ec.lr.total_steps = static_cast<int64_t>(H) * rounds;
        ExperimentResult r = run_experiment(ec, out_root);
        int32_t n = 0;
        for (const RoundMetrics& m : r.rounds) {
            if (n < cap)
                rows[n] = {m.round, m.mean_total, m.mean_ce, m.mean_lb, m.mean_moe_z, m.mean_z,
                           m.merge_displacement_sq, m.bytes_up, m.bytes_down};
            ++n;
        }
        *n_out = n;
        *tokens_per_round = static_cast<int64_t>(nodes) * H * batch * seq_len;
        return 0;
    } catch (...) {
        return 1;
    }
}

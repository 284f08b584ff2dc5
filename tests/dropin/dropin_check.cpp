// Drop-in check (test infrastructure): the reference's own header-only entry points,
//   spes::local_round (proj/include/spes/trainer.hpp:143-222)
//   spes::merge_model (proj/include/spes/merging.hpp:138-150)
// run on the CPU next to their B200 drop-ins from include/spes_b200.hpp on the SAME
// model, batches, mask and schedule. The binary is compiled in the build container
// (where the reference headers exist) and runs on the GPU box; tests/test_dropin.py
// drives it.
//
// Checks:
//   local_round: per-step total loss within LOSS_RTOL (bf16 tensor-core GEMMs), frozen
//                experts bit-identical to the input, grad_scalar_count identical,
//                trainable displacement within DELTA_RTOL after H AdamW steps;
//   merge_model: peer sets and every parameter bit-identical (fp64 merge, identical input).
//   SGD inner steps with record_trace: losses, update norms, drift and per-block gradient
//                sums within bf16 tolerance of the reference's;
//   batches of different (B, S) in one round: per-step losses within LOSS_RTOL;
//   errors:      H < 1 -> std::invalid_argument; token out of range -> std::out_of_range.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "spes/merging.hpp"
#include "spes/model.hpp"
#include "spes/trainer.hpp"
#include "spes_b200.hpp"

namespace {

constexpr double LOSS_RTOL = 5e-3;
// bf16 GEMM gradients vs fp32: the H-step parameter displacement of the trainable
// blocks, ||d_b200 - d_ref|| / ||d_ref|| with d = theta_H - theta_0
constexpr double DELTA_RTOL = 5e-2;

int failures = 0;
void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

spes::BatchProvider batches(const spes::ModelConfig& c, int64_t B, int64_t S, uint64_t seed) {
    auto rng = std::make_shared<std::mt19937_64>(seed);
    return [c, B, S, rng]() {
        spes::Batch b;
        b.batch = B;
        b.seq = S;
        std::uniform_int_distribution<int32_t> u(0, static_cast<int32_t>(c.vocab - 1));
        b.tokens.resize(static_cast<size_t>(B * (S + 1)));
        for (auto& t : b.tokens) t = u(*rng);
        return b;
    };
}

}  // namespace

int main(int argc, char** argv) {
    const int device = argc > 1 ? std::atoi(argv[1]) : 0;
    spes::ModelConfig cfg;
    cfg.vocab = 256;
    cfg.hidden = 128;
    cfg.intermediate = 256;
    cfg.layers = 2;
    cfg.experts_total = 8;
    cfg.experts_active = 2;
    const int64_t B = 4, S = 64;
    const int H = 4;

    const spes::ModelParams global = spes::init_model<float>(cfg, 1, 0.02);
    spes::TrainMask mask;
    mask.node_id = 0;
    mask.owned_experts = {0, 1, 2, 3};
    spes::LocalRoundConfig rc;
    rc.steps = H;

    // ---- local_round: reference (CPU) vs B200 drop-in ----
    const spes::LocalRoundResult ref = spes::local_round(global, batches(cfg, B, S, 7), rc, mask);
    spes_b200::Context ctx(spes_b200::to_c(cfg), 0, 1, device);
    const spes::LocalRoundResult gpu =
        spes_b200::local_round(ctx, global, batches(cfg, B, S, 7), rc, mask);

    bool loss_ok = ref.step_losses.size() == gpu.step_losses.size();
    for (size_t h = 0; loss_ok && h < ref.step_losses.size(); ++h) {
        const double a = gpu.step_losses[h].total, b = ref.step_losses[h].total;
        std::printf("  step %zu loss ref %.7f b200 %.7f\n", h, b, a);
        loss_ok = std::fabs(a - b) <= LOSS_RTOL * std::fabs(b);
    }
    expect(loss_ok, "local_round per-step total loss within 5e-3 rel");
    expect(gpu.grad_scalar_count == ref.grad_scalar_count, "local_round grad_scalar_count");

    bool frozen_same = true;
    double dd2 = 0.0, dr2 = 0.0;
    for (const auto& b : spes::enumerate_blocks(cfg)) {
        const auto& g = spes::block_tensor(gpu.params, b).data;
        const auto& r = spes::block_tensor(ref.params, b).data;
        const auto& x = spes::block_tensor(global, b).data;
        for (size_t i = 0; i < g.size(); ++i) {
            if (!mask.trainable(b)) {
                frozen_same &= std::memcmp(&g[i], &x[i], sizeof(float)) == 0;
            } else {
                const double dg = static_cast<double>(g[i]) - x[i];
                const double dr = static_cast<double>(r[i]) - x[i];
                dd2 += (dg - dr) * (dg - dr);
                dr2 += dr * dr;
            }
        }
    }
    const double rel = dr2 > 0 ? std::sqrt(dd2 / dr2) : 1.0;
    std::printf("  trainable displacement rel err = %.3e\n", rel);
    expect(frozen_same, "local_round frozen experts bit-identical to the input");
    expect(rel < DELTA_RTOL, "local_round trainable displacement within 5e-2 rel of the reference");

    // ---- SGD inner steps with record_trace (trainer.hpp:116-122, 183-219) ----
    {
        spes::LocalRoundConfig sc = rc;
        sc.inner = spes::InnerOpt::SGD;
        sc.opt.lr = 0.05;
        sc.record_trace = true;
        const auto r2 = spes::local_round(global, batches(cfg, B, S, 9), sc, mask);
        const auto g2 = spes_b200::local_round(ctx, global, batches(cfg, B, S, 9), sc, mask);
        bool ok = r2.step_losses.size() == g2.step_losses.size() &&
                  r2.update_norms.size() == g2.update_norms.size() &&
                  r2.drift_sq.size() == g2.drift_sq.size() &&
                  r2.grad_sum.size() == g2.grad_sum.size();
        double worst = 0.0;
        auto rel = [&](double a, double b) {
            const double e = std::fabs(a - b) / std::max(std::fabs(b), 1e-30);
            worst = std::max(worst, e);
            return e;
        };
        for (size_t h = 0; ok && h < r2.step_losses.size(); ++h) {
            ok &= rel(g2.step_losses[h].total, r2.step_losses[h].total) <= LOSS_RTOL;
            ok &= rel(g2.update_norms[h], r2.update_norms[h]) <= 2e-2;
            ok &= rel(g2.drift_sq[h], r2.drift_sq[h]) <= DELTA_RTOL;
        }
        for (size_t i = 0; ok && i < r2.grad_sum.size(); ++i) {
            const auto& a = g2.grad_sum[i];
            const auto& b = r2.grad_sum[i];
            ok &= a.block_index == b.block_index && a.grad.shape == b.grad.shape;
            double e2 = 0.0, n2 = 0.0;
            for (size_t j = 0; ok && j < b.grad.data.size(); ++j) {
                const double d = static_cast<double>(a.grad.data[j]) - b.grad.data[j];
                e2 += d * d;
                n2 += static_cast<double>(b.grad.data[j]) * b.grad.data[j];
            }
            if (n2 > 0) worst = std::max(worst, std::sqrt(e2 / n2));
            ok &= n2 == 0 ? e2 == 0 : std::sqrt(e2 / n2) <= 2e-2;
        }
        std::printf("  sgd + record_trace: worst relative deviation %.3e\n", worst);
        expect(ok, "local_round SGD + record_trace (losses, update norms, drift, grad sums)");
    }

    // ---- batches of different shapes within one round (trainer.hpp:163: each its own) ----
    {
        auto mixed = [&](uint64_t seed) {
            auto base = std::make_shared<int>(0);
            auto rng = std::make_shared<std::mt19937_64>(seed);
            return spes::BatchProvider([cfg, base, rng]() {
                static const int64_t shapes[3][2] = {{4, 64}, {8, 32}, {2, 100}};
                const auto* sh = shapes[(*base)++ % 3];
                spes::Batch b;
                b.batch = sh[0];
                b.seq = sh[1];
                std::uniform_int_distribution<int32_t> u(0, static_cast<int32_t>(cfg.vocab - 1));
                b.tokens.resize(static_cast<size_t>(b.batch * (b.seq + 1)));
                for (auto& t : b.tokens) t = u(*rng);
                return b;
            });
        };
        spes::LocalRoundConfig mc = rc;
        mc.steps = 5;
        const auto r3 = spes::local_round(global, mixed(11), mc, mask);
        const auto g3 = spes_b200::local_round(ctx, global, mixed(11), mc, mask);
        bool ok = r3.step_losses.size() == g3.step_losses.size();
        for (size_t h = 0; ok && h < r3.step_losses.size(); ++h) {
            std::printf("  mixed-shape step %zu loss ref %.7f b200 %.7f\n", h,
                        r3.step_losses[h].total, g3.step_losses[h].total);
            ok = std::fabs(g3.step_losses[h].total - r3.step_losses[h].total) <=
                 LOSS_RTOL * std::fabs(r3.step_losses[h].total);
        }
        expect(ok, "local_round over batches of different (B, S) within one round");
    }

    // ---- merge_model: bit-exact on identical input ----
    spes::MergeSchedule ms;
    ms.warmup_rounds = 10;
    ms.interval = 1;
    ms.alpha0 = 0.1;
    ms.peers = 3;
    spes::ModelParams pr = ref.params, pg = ref.params;
    const auto ev_ref = spes::merge_model(pr, ms, 2);
    const auto ev_gpu = spes_b200::merge_model(ctx, pg, ms, 2);
    bool peers_same = ev_ref.size() == ev_gpu.size();
    for (size_t l = 0; peers_same && l < ev_ref.size(); ++l)
        peers_same = ev_ref[l].peer_sets == ev_gpu[l].peer_sets &&
                     ev_ref[l].alpha == ev_gpu[l].alpha &&
                     std::fabs(ev_ref[l].displacement_sq - ev_gpu[l].displacement_sq) <=
                         1e-9 * std::fabs(ev_ref[l].displacement_sq);
    expect(peers_same, "merge_model events (peer sets, alpha, displacement)");
    bool merged_same = true;
    for (const auto& b : spes::enumerate_blocks(cfg)) {
        const auto& g = spes::block_tensor(pg, b).data;
        const auto& r = spes::block_tensor(pr, b).data;
        merged_same &= std::memcmp(g.data(), r.data(), g.size() * sizeof(float)) == 0;
    }
    expect(merged_same, "merge_model parameters bit-identical");
    expect(spes_b200::merge_model(ctx, pg, ms, 11).empty(), "merge_model outside warm-up is a no-op");

    // ---- error conventions (trainer.hpp:146, model.hpp:280-281) ----
    spes::LocalRoundConfig bad = rc;
    bad.steps = 0;
    try {
        spes_b200::local_round(ctx, global, batches(cfg, B, S, 1), bad, mask);
        expect(false, "H < 1 throws invalid_argument");
    } catch (const std::invalid_argument&) {
        expect(true, "H < 1 throws invalid_argument");
    }
    try {
        auto oob = [&]() {
            spes::Batch b = batches(cfg, B, S, 3)();
            b.tokens[5] = static_cast<int32_t>(cfg.vocab);
            return b;
        };
        spes_b200::local_round(ctx, global, oob, rc, mask);
        expect(false, "token id out of vocabulary throws out_of_range");
    } catch (const std::out_of_range&) {
        expect(true, "token id out of vocabulary throws out_of_range");
    }
    // ---- the reference's default ModelConfig (model.hpp:21-31; off the 128-wide tiles) ----
    {
        spes::ModelConfig dc;  // vocab 64, hidden 32, intermediate 64, 2 layers, 4 experts top-2
        const spes::ModelParams g0 = spes::init_model<float>(dc, 3, 0.02);
        spes::TrainMask m0;
        m0.node_id = 0;
        m0.owned_experts = {1, 2};
        spes::LocalRoundConfig c0;
        c0.steps = 3;
        const auto r4 = spes::local_round(g0, batches(dc, 2, 16, 21), c0, m0);
        spes_b200::Context dctx(spes_b200::to_c(dc), 0, 1, device);
        const auto g4 = spes_b200::local_round(dctx, g0, batches(dc, 2, 16, 21), c0, m0);
        bool ok = r4.step_losses.size() == g4.step_losses.size() &&
                  r4.grad_scalar_count == g4.grad_scalar_count;
        for (size_t h = 0; ok && h < r4.step_losses.size(); ++h) {
            std::printf("  default-config step %zu loss ref %.7f b200 %.7f\n", h,
                        r4.step_losses[h].total, g4.step_losses[h].total);
            ok = std::fabs(g4.step_losses[h].total - r4.step_losses[h].total) <=
                 LOSS_RTOL * std::fabs(r4.step_losses[h].total);
        }
        for (const auto& b : spes::enumerate_blocks(dc))
            if (!m0.trainable(b)) {
                const auto& a = spes::block_tensor(g4.params, b).data;
                const auto& x = spes::block_tensor(g0, b).data;
                ok &= std::memcmp(a.data(), x.data(), a.size() * sizeof(float)) == 0;
            }
        expect(ok, "local_round on the reference's default ModelConfig (padded on the device)");
    }
    std::printf(failures ? "DROPIN FAILED\n" : "DROPIN OK\n");
    return failures ? 1 : 0;
}

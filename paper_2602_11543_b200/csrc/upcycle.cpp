// Upcycling of a dense model into an M-expert SPES model, following
// upcycle_from_dense (proj/include/spes/model.hpp:415-460): embedding / norm / head copied,
// each router widened by replicating its single column, every expert a copy of the dense
// FFN with a random subset (noise_frac of the elements, partial Fisher-Yates with
// std::uniform_int_distribution) perturbed by std::normal_distribution(0, noise_std)
// draws, renormalize_after_topk switched on. The draws use the same std::mt19937_64 and
// libstdc++ distributions in the same order, so the result is bit-identical.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

namespace spes_upcycle {

// flat enumerate_blocks layout helpers
struct Dims {
    int64_t V, d, f;
    int L, M;
    int64_t psi() const { return 2 * V * d + L * (d + d * M); }
    int64_t off_norm(int l) const { return 2 * V * d + l * (d + d * M); }
    int64_t off_router(int l) const { return off_norm(l) + d; }
    int64_t off_expert(int l, int j) const { return psi() + (static_cast<int64_t>(l) * M + j) * 3 * d * f; }
    int64_t total() const { return off_expert(L, 0); }
};

void upcycle(int64_t V, int64_t d, int64_t f, int L, const float* dense, int m, double noise_frac,
             double noise_std, uint64_t seed, float* out) {
    if (m < 2) throw std::invalid_argument("upcycle: need M >= 2");
    const Dims src{V, d, f, L, 1}, dst{V, d, f, L, m};
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> noise(0.0, noise_std);
    // embedding and head
    std::memcpy(out, dense, sizeof(float) * 2 * V * d);
    for (int l = 0; l < L; ++l) {
        std::memcpy(out + dst.off_norm(l), dense + src.off_norm(l), sizeof(float) * d);
        const float* r = dense + src.off_router(l);  // d x 1
        float* w = out + dst.off_router(l);          // d x m
        for (int64_t row = 0; row < d; ++row)
            for (int j = 0; j < m; ++j) w[row * m + j] = r[row];
    }
    auto perturb = [&](const float* t, size_t n, float* o) {
        std::memcpy(o, t, sizeof(float) * n);
        const size_t subset = static_cast<size_t>(std::llround(noise_frac * static_cast<double>(n)));
        std::vector<size_t> order(n);
        std::iota(order.begin(), order.end(), size_t{0});
        for (size_t i = 0; i < subset; ++i) {
            std::uniform_int_distribution<size_t> pick(i, n - 1);
            std::swap(order[i], order[pick(rng)]);
            const double nz = noise(rng);
            if (noise_std > 0.0) o[order[i]] += static_cast<float>(nz);
        }
    };
    const size_t df = static_cast<size_t>(d * f);
    for (int l = 0; l < L; ++l) {
        const float* e = dense + src.off_expert(l, 0);
        for (int j = 0; j < m; ++j) {
            float* o = out + dst.off_expert(l, j);
            perturb(e, df, o);               // wg
            perturb(e + df, df, o + df);     // wu
            perturb(e + 2 * df, df, o + 2 * df);  // wd
        }
    }
}

}  // namespace spes_upcycle

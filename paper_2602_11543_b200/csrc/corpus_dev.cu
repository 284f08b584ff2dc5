// Device-side synthetic corpus: gen_corpus's token sampling
// (proj/src/corpus.cpp:49-79, sample_from :35-44) regenerated on the GPU, bit-identical.
//
// The host builds the Markov sources (corpus.cpp prepare_device_corpus) and hands over
// the std::mt19937_64 state that follows them. From there each token consumes exactly one
// 64-bit engine output (uniform_real_distribution<double>(0, 1) = generate_canonical<double,
// 53> over a 64-bit engine: double(x) / 2^64, kept below 1), so:
//   mt_draws_k      one CTA runs the engine: each refill (_M_gen_rand) is three dependency
//                   phases over the 312-word state in shared memory, then the 312 tempered
//                   outputs go to HBM as the uniform doubles;
//   corpus_chain_k  one thread per sequence walks its Markov chain: sample_from's "first i
//                   with r < acc_i" is a binary search over the source row's prefix sums
//                   (acc is non-decreasing, and the host computed it in the same order).
// Sequence r uses draws [r (S+1), (r+1)(S+1)): its first token from the initial row, then
// one transition per position (corpus.cpp:70-77).
#include "kernels.h"

namespace spes_k {

namespace {
constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_A = 0xB5026F5AA96619E9ull;
constexpr uint64_t MT_UPPER = 0xFFFFFFFF80000000ull;  // upper 33 bits (r = 31)
constexpr uint64_t MT_LOWER = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_step(uint64_t xk, uint64_t xk1, uint64_t xkm) {
    const uint64_t y = (xk & MT_UPPER) | (xk1 & MT_LOWER);
    return xkm ^ (y >> 1) ^ ((y & 1ull) ? MT_A : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

__device__ __forceinline__ double canonical53(uint64_t x) {
    const double r = __ull2double_rn(x) * 0x1p-64;
    return r >= 1.0 ? 0x1.fffffffffffffp-1 : r;  // nextafter(1, 0)
}
}  // namespace

__global__ void __launch_bounds__(MT_N) mt_draws_k(const uint64_t* __restrict__ state, int pos,
                                                   int64_t n, double* __restrict__ out) {
    __shared__ uint64_t s[MT_N];
    const int i = threadIdx.x;
    s[i] = state[i];
    __syncthreads();
    int64_t done = 0;
    int p = pos;
    while (done < n) {
        if (p >= MT_N) {  // refill: x[k] for k < n-m, then k < n-1 (reads new x[k-(n-m)]), then n-1
            uint64_t v = 0;
            if (i < MT_N - MT_M) v = mt_step(s[i], s[i + 1], s[i + MT_M]);
            __syncthreads();
            if (i < MT_N - MT_M) s[i] = v;
            __syncthreads();
            if (i >= MT_N - MT_M && i < MT_N - 1) v = mt_step(s[i], s[i + 1], s[i - (MT_N - MT_M)]);
            __syncthreads();
            if (i >= MT_N - MT_M && i < MT_N - 1) s[i] = v;
            __syncthreads();
            if (i == MT_N - 1) s[i] = mt_step(s[i], s[0], s[MT_M - 1]);
            __syncthreads();
            p = 0;
        }
        const int64_t o = done + (i - p);
        if (i >= p && o < n) out[o] = canonical53(mt_temper(s[i]));
        done += MT_N - p;
        p = MT_N;
    }
}

__global__ void corpus_chain_k(const double* __restrict__ cum, const double* __restrict__ u,
                               int64_t sequences, int64_t seq, int V, int C,
                               int32_t* __restrict__ tokens) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= sequences) return;
    const double* tab = cum + static_cast<int64_t>(r % C) * (V + 1) * V;
    const int64_t base = r * (seq + 1);
    auto sample = [&](const double* row, double x) {
        int lo = 0, hi = V;  // first index with x < row[i]; none -> V - 1
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (x < __ldg(row + mid))
                hi = mid;
            else
                lo = mid + 1;
        }
        return lo < V ? lo : V - 1;
    };
    int tok = sample(tab, u[base]);
    tokens[base] = tok;
    for (int64_t p = 0; p < seq; ++p) {
        tok = sample(tab + static_cast<int64_t>(1 + tok) * V, u[base + 1 + p]);
        tokens[base + 1 + p] = tok;
    }
}

void corpus_draws(const uint64_t* state, int pos, int64_t n, double* out, cudaStream_t s) {
    mt_draws_k<<<1, MT_N, 0, s>>>(state, pos, n, out);
}

void corpus_chains(const double* cum, const double* u, int64_t sequences, int64_t seq, int V,
                   int C, int32_t* tokens, cudaStream_t s) {
    const int tpb = 64;
    corpus_chain_k<<<static_cast<unsigned>((sequences + tpb - 1) / tpb), tpb, 0, s>>>(
        cum, u, sequences, seq, V, C, tokens);
}

}  // namespace spes_k

// Router forward, bit-exact with the reference given identical h:
//   rmsnorm_forward (kernels.hpp:117-128): sequential sum of squares, y = (x*inv)*g
//   matmul (kernels.hpp:27-38): logit_e = sum_p normed_p * R[p][e], p ascending, no FMA
//   softmax_rows (kernels.hpp:156-172) with the glibc-compatible expf; logsumexp (:174-185)
//   route_from_logits (model.hpp:185-216): stable top-k, ascending indices, weights
//
// Block = NT tokens x (MAXM/4) expert quads = 256 threads. Token rows stream through
// shared memory in 64-column chunks twice: pass 1 accumulates the sequential sum of
// squares (one thread per token), pass 2 forms normed = (x*inv)*g and advances every
// logit chain over the chunk. Each thread owns one token x four experts, so one
// broadcast load of normed and one 16-byte load of router weights feed four
// independent exact-order chains.
#include "common.cuh"
#include "glibc_expf.h"
#include "kernels.h"

namespace spes_k {

using namespace spes_dev;

constexpr int RF_QC = 64;  // columns per chunk

template <int MAXM>
__global__ void __launch_bounds__(256) router_fwd_k(
    const float* __restrict__ h, const float* __restrict__ gain, const float* __restrict__ R,
    int T, int d, int M, int k, int renorm, float eps, int variant, float* __restrict__ normed,
    float* __restrict__ logits, float* __restrict__ probs, int32_t* __restrict__ topk_idx,
    float* __restrict__ topk_w, float* __restrict__ lse_out, float* __restrict__ inv_out,
    float* __restrict__ denom_out) {
    constexpr int EG = MAXM / 4;      // expert quads
    constexpr int NT = 256 / EG;      // tokens per block
    __shared__ float sx[NT][RF_QC + 1];
    __shared__ __align__(16) float sR[RF_QC][MAXM];
    __shared__ float sv[NT][MAXM + 1];
    __shared__ float sinv[NT], smx[NT];
    const int t0 = blockIdx.x * NT;
    const int nt = min(NT, T - t0);
    const int tq = threadIdx.x / EG, eg = threadIdx.x % EG;

    auto load_chunk = [&](int q0) {
        for (int i = threadIdx.x; i < NT * (RF_QC / 4); i += blockDim.x) {
            const int tt = i / (RF_QC / 4), c = (i % (RF_QC / 4)) * 4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (tt < nt) v = __ldg(reinterpret_cast<const float4*>(h + static_cast<int64_t>(t0 + tt) * d + q0 + c));
            sx[tt][c] = v.x;
            sx[tt][c + 1] = v.y;
            sx[tt][c + 2] = v.z;
            sx[tt][c + 3] = v.w;
        }
    };

    // pass 1: sum of squares, sequential per token
    float ms = 0.f;
    for (int q0 = 0; q0 < d; q0 += RF_QC) {
        __syncthreads();
        load_chunk(q0);
        __syncthreads();
        if (threadIdx.x < nt) {
            const float* xr = sx[threadIdx.x];
#pragma unroll 16
            for (int c = 0; c < RF_QC; ++c) ms = fadd(ms, fmul(xr[c], xr[c]));
        }
    }
    if (threadIdx.x < nt) {
        const float inv = fdiv(1.f, fsqrt(fadd(fdiv(ms, static_cast<float>(d)), eps)));
        sinv[threadIdx.x] = inv;
        inv_out[t0 + threadIdx.x] = inv;
    }

    // pass 2: normed chunk + logits
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const bool active = tq < nt;
    for (int q0 = 0; q0 < d; q0 += RF_QC) {
        __syncthreads();
        load_chunk(q0);
        for (int i = threadIdx.x; i < RF_QC * MAXM; i += blockDim.x) {
            const int c = i / MAXM, e = i % MAXM;
            sR[c][e] = e < M ? __ldg(R + static_cast<int64_t>(q0 + c) * M + e) : 0.f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nt * RF_QC; i += blockDim.x) {
            const int tt = i / RF_QC, c = i % RF_QC;
            const float nv = fmul(fmul(sx[tt][c], sinv[tt]), __ldg(gain + q0 + c));
            sx[tt][c] = nv;
            normed[static_cast<int64_t>(t0 + tt) * d + q0 + c] = nv;
        }
        __syncthreads();
        if (active) {
            const float* xr = sx[tq];
#pragma unroll 8
            for (int c = 0; c < RF_QC; ++c) {
                const float nv = xr[c];
                const float4 r = *reinterpret_cast<const float4*>(&sR[c][4 * eg]);
                acc[0] = fadd(acc[0], fmul(nv, r.x));
                acc[1] = fadd(acc[1], fmul(nv, r.y));
                acc[2] = fadd(acc[2], fmul(nv, r.z));
                acc[3] = fadd(acc[3], fmul(nv, r.w));
            }
        }
    }
    if (active) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = 4 * eg + u;
            if (e < M) {
                sv[tq][e] = acc[u];
                logits[static_cast<int64_t>(t0 + tq) * M + e] = acc[u];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < nt) {  // std::max scan (kernels.hpp:160)
        const float* lr = sv[threadIdx.x];
        float mx = lr[0];
        for (int j = 1; j < M; ++j) mx = (mx < lr[j]) ? lr[j] : mx;
        smx[threadIdx.x] = mx;
    }
    __syncthreads();
    if (active) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = 4 * eg + u;
            if (e < M) {
                const float z = fsub(acc[u], smx[tq]);
                sv[tq][e] = variant ? spes_expf::expf_glibc<1>(z) : spes_expf::expf_glibc<0>(z);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < nt) {  // sequential sum, 1/sum, lse
        const float* ex = sv[threadIdx.x];
        float sum = 0.f;
        for (int j = 0; j < M; ++j) sum = fadd(sum, ex[j]);
        sinv[threadIdx.x] = fdiv(1.f, sum);
        lse_out[t0 + threadIdx.x] = smx[threadIdx.x] + logf(sum);
    }
    __syncthreads();
    if (active) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = 4 * eg + u;
            if (e < M) {
                const float p = fmul(sv[tq][e], sinv[tq]);
                sv[tq][e] = p;
                probs[static_cast<int64_t>(t0 + tq) * M + e] = p;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < nt) {
        // iterative argmax (strict '>' scanning ascending => lowest index on ties) ==
        // the first k of a stable descending sort; then ascending order
        const int t = t0 + threadIdx.x;
        const float* p = sv[threadIdx.x];
        uint64_t chosen = 0;
        for (int s = 0; s < k; ++s) {
            int best = -1;
            float bv = 0.f;
            for (int j = 0; j < M; ++j) {
                if ((chosen >> j) & 1ull) continue;
                if (best < 0 || p[j] > bv) {
                    best = j;
                    bv = p[j];
                }
            }
            chosen |= 1ull << best;
        }
        float dn = 0.f;
        for (int j = 0; j < M; ++j)
            if ((chosen >> j) & 1ull) dn = fadd(dn, p[j]);
        int slot = 0;
        for (int j = 0; j < M; ++j) {
            if ((chosen >> j) & 1ull) {
                topk_idx[static_cast<int64_t>(t) * k + slot] = j;
                topk_w[static_cast<int64_t>(t) * k + slot] = renorm ? fdiv(p[j], dn) : p[j];
                ++slot;
            }
        }
        if (denom_out) denom_out[t] = dn;
    }
}

void router_forward(const float* h, const float* gain, const float* router, int64_t T, int64_t d,
                    int M, int k, int renorm, float eps, int variant, float* normed,
                    float* logits, float* probs, int32_t* topk_idx, float* topk_w, float* lse,
                    float* inv_rms, float* denom, cudaStream_t s) {
    const int maxm = M <= 8 ? 8 : (M <= 16 ? 16 : (M <= 32 ? 32 : 64));
    const int NT = 256 / (maxm / 4);
    const unsigned grid = static_cast<unsigned>((T + NT - 1) / NT);
#define SPES_RF(MM)                                                                              \
    router_fwd_k<MM><<<grid, 256, 0, s>>>(h, gain, router, (int)T, (int)d, M, k, renorm, eps,    \
                                          variant, normed, logits, probs, topk_idx, topk_w, lse, \
                                          inv_rms, denom)
    if (maxm == 8)
        SPES_RF(8);
    else if (maxm == 16)
        SPES_RF(16);
    else if (maxm == 32)
        SPES_RF(32);
    else
        SPES_RF(64);
#undef SPES_RF
    count_launch();
}

}  // namespace spes_k

// Router forward, bit-exact with the reference given identical h:
//   rmsnorm_forward (kernels.hpp:117-128): sequential sum of squares, y = (x*inv)*g
//   matmul (kernels.hpp:27-38): logit_e = sum_p normed_p * R[p][e], p ascending, no FMA
//   softmax_rows (kernels.hpp:156-172) with the glibc-compatible expf; logsumexp (:174-185)
//   route_from_logits (model.hpp:185-216): stable top-k, ascending indices, weights
//
// Block = NT tokens x MAXM experts (256 threads). The token rows are staged in
// shared memory once; the one inherently sequential chain per token (sum of squares)
// runs on one thread per token, every logit chain (sequential over d) on its own
// thread, so a block keeps NT*M independent chains in flight.
#include "common.cuh"
#include "glibc_expf.h"
#include "kernels.h"

namespace spes_k {

using namespace spes_dev;

constexpr int RF_RQ = 64;  // router rows per smem chunk

template <int MAXM>
__global__ void __launch_bounds__(256) router_fwd_k(
    const float* __restrict__ h, const float* __restrict__ gain, const float* __restrict__ R,
    int T, int d, int NT, int M, int k, int renorm, float eps, int variant,
    float* __restrict__ normed, float* __restrict__ logits, float* __restrict__ probs,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, float* __restrict__ lse_out,
    float* __restrict__ inv_out, float* __restrict__ denom_out) {
    extern __shared__ float sm[];
    const int ld = d + 1;                   // row stride: odd -> conflict-free per-token walks
    float* sx = sm;                         // [NT][ld]   rows, then normed rows
    float* sR = sx + NT * ld;               // [RF_RQ][MAXM]
    float* sv = sR + RF_RQ * MAXM;          // [NT][MAXM] logits / exps / probs
    float* sinv = sv + NT * MAXM;           // [NT]
    float* smx = sinv + NT;                 // [NT]
    const int t0 = blockIdx.x * NT;
    const int nt = min(NT, T - t0);

    for (int i = threadIdx.x; i < nt * (d / 4); i += blockDim.x) {
        const int tt = i / (d / 4), q = (i % (d / 4)) * 4;
        const float4 v = __ldg(reinterpret_cast<const float4*>(h + static_cast<int64_t>(t0 + tt) * d + q));
        float* dst = sx + tt * ld + q;
        dst[0] = v.x;
        dst[1] = v.y;
        dst[2] = v.z;
        dst[3] = v.w;
    }
    __syncthreads();
    if (threadIdx.x < nt) {
        const float* xr = sx + threadIdx.x * ld;
        float ms = 0.f;
        for (int q = 0; q < d; ++q) ms = fadd(ms, fmul(xr[q], xr[q]));
        const float inv = fdiv(1.f, fsqrt(fadd(fdiv(ms, static_cast<float>(d)), eps)));
        sinv[threadIdx.x] = inv;
        inv_out[t0 + threadIdx.x] = inv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nt * d; i += blockDim.x) {
        const int tt = i / d, q = i % d;
        const float nv = fmul(fmul(sx[tt * ld + q], sinv[tt]), __ldg(gain + q));
        sx[tt * ld + q] = nv;
        normed[static_cast<int64_t>(t0 + tt) * d + q] = nv;
    }
    // logits: thread (tt, e), sequential over q
    const int tt = threadIdx.x / MAXM, e = threadIdx.x % MAXM;
    const bool active = tt < nt && e < M;
    float acc = 0.f;
    for (int q0 = 0; q0 < d; q0 += RF_RQ) {
        __syncthreads();
        for (int i = threadIdx.x; i < RF_RQ * M; i += blockDim.x) {
            const int qq = i / M, ee = i % M;
            sR[qq * MAXM + ee] = __ldg(R + static_cast<int64_t>(q0 + qq) * M + ee);
        }
        __syncthreads();
        if (active) {
            const float* xr = sx + tt * ld + q0;
#pragma unroll 16
            for (int qq = 0; qq < RF_RQ; ++qq) acc = fadd(acc, fmul(xr[qq], sR[qq * MAXM + e]));
        }
    }
    if (active) {
        sv[tt * MAXM + e] = acc;
        logits[static_cast<int64_t>(t0 + tt) * M + e] = acc;
    }
    __syncthreads();
    if (threadIdx.x < nt) {  // std::max scan (kernels.hpp:160)
        const float* lr = sv + threadIdx.x * MAXM;
        float mx = lr[0];
        for (int j = 1; j < M; ++j) mx = (mx < lr[j]) ? lr[j] : mx;
        smx[threadIdx.x] = mx;
    }
    __syncthreads();
    if (active) {
        const float z = fsub(acc, smx[tt]);
        sv[tt * MAXM + e] = variant ? spes_expf::expf_glibc<1>(z) : spes_expf::expf_glibc<0>(z);
    }
    __syncthreads();
    if (threadIdx.x < nt) {  // sequential sum, 1/sum, lse
        const float* ex = sv + threadIdx.x * MAXM;
        float sum = 0.f;
        for (int j = 0; j < M; ++j) sum = fadd(sum, ex[j]);
        sinv[threadIdx.x] = fdiv(1.f, sum);
        lse_out[t0 + threadIdx.x] = smx[threadIdx.x] + logf(sum);
    }
    __syncthreads();
    if (active) {
        const float p = fmul(sv[tt * MAXM + e], sinv[tt]);
        sv[tt * MAXM + e] = p;
        probs[static_cast<int64_t>(t0 + tt) * M + e] = p;
    }
    __syncthreads();
    if (threadIdx.x < nt) {
        // iterative argmax (strict '>' scanning ascending => lowest index on ties) ==
        // the first k of a stable descending sort; then ascending order
        const int t = t0 + threadIdx.x;
        const float* p = sv + threadIdx.x * MAXM;
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
    int NT = 256 / maxm;
    while (NT > 1 && static_cast<int64_t>(NT) * (d + 1) * 4 > 96 * 1024) NT /= 2;
    const size_t smem = sizeof(float) * (static_cast<size_t>(NT) * (d + 1) + RF_RQ * maxm +
                                         static_cast<size_t>(NT) * maxm + 2 * NT);
    const unsigned grid = static_cast<unsigned>((T + NT - 1) / NT);
#define SPES_RF(MM)                                                                          \
    do {                                                                                     \
        cudaFuncSetAttribute(router_fwd_k<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                     \
        router_fwd_k<MM><<<grid, 256, smem, s>>>(h, gain, router, (int)T, (int)d, NT, M, k,  \
                                                 renorm, eps, variant, normed, logits, probs, \
                                                 topk_idx, topk_w, lse, inv_rms, denom);     \
    } while (0)
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

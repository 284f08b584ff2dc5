// Router backward + rmsnorm backward of one layer (the non-GEMM half of the layer's
// backward pass), following the reverse tape:
//   probs.grad  = (0 + g_lb*coeff_j) [lb, model.hpp:358] + gate-weight grads (experts desc.)
//   logits.grad = (0 + gl*p_j) [moe_z logsumexp] + p_j*(gprobs_j - dot) [softmax bwd]
//   normed.grad = dX of selected experts (desc.) + glog . R^T [matmul_nt_acc]
//   h.grad     += rmsnorm backward (kernels.hpp:130-152)
// Two kernels here, each streaming its operands once:
//   router_scalar_bwd_k : thread per token, the M-wide scalar chain  -> glog [T x M]
//   normed_grad_k       : 32-token x 128-column tiles; per element the dX sum (descending
//                         experts) then the router product over e ascending (fused
//                         multiply-adds: a gradient, tolerance-level); per-tile partial of
//                         sum_q (gy*g)*x for the rmsnorm dot
// The rmsnorm backward itself (h.grad += (gy*g)*inv - coef*x) runs inside
// norm_router_partial_k (kernels.cu), which streams h and gnormed for the gain and router
// gradients anyway. Every element keeps the reference's accumulation order (the router
// product with FMA); the rmsnorm dot (a sum over d) is a fixed-order tree.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace spes_k {

using namespace spes_dev;

template <int MAXM>
__global__ void __launch_bounds__(128) router_scalar_bwd_k(
    const float* __restrict__ probs, const float* __restrict__ lse_r,
    const float* __restrict__ denom, const int32_t* __restrict__ topk_idx,
    const int32_t* __restrict__ slot_row, const float* __restrict__ gw_row,
    const float* __restrict__ lb_coeff, int T, int M, int k, int renorm, float g_lbsum, float g_s,
    float* __restrict__ glog, bf16* __restrict__ glog_bf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    float p[MAXM], gp[MAXM];
    const float* prow = probs + static_cast<int64_t>(t) * M;
#pragma unroll
    for (int e = 0; e < MAXM; ++e) {
        if (e < M) {
            p[e] = prow[e];
            gp[e] = fadd(0.f, fmul(g_lbsum, __ldg(lb_coeff + e)));
        }
    }
    const float dn = renorm ? denom[t] : 1.f;
    float gden = 0.f;
    int32_t sel[8];
    for (int s = k - 1; s >= 0; --s) {  // experts in descending order
        const int j = topk_idx[static_cast<int64_t>(t) * k + s];
        sel[s] = j;
        const float gw = gw_row[slot_row[static_cast<int64_t>(t) * k + s]];
#pragma unroll
        for (int e = 0; e < MAXM; ++e) {
            if (e == j) {
                if (renorm) {
                    gden = fsub(gden, fdiv(fmul(gw, p[e]), fmul(dn, dn)));
                    gp[e] = fadd(gp[e], fadd(0.f, fdiv(gw, dn)));
                } else {
                    gp[e] = fadd(gp[e], fadd(0.f, gw));
                }
            }
        }
    }
    if (renorm)
        for (int s = k - 1; s >= 0; --s) {
#pragma unroll
            for (int e = 0; e < MAXM; ++e)
                if (e == sel[s]) gp[e] = fadd(gp[e], gden);
        }
    const float lv = lse_r[t];
    const float gl = fadd(fadd(0.f, fmul(g_s, lv)), fmul(g_s, lv));
    float dot = 0.f;
#pragma unroll
    for (int e = 0; e < MAXM; ++e)
        if (e < M) dot = fadd(dot, fmul(gp[e], p[e]));
    float* grow = glog + static_cast<int64_t>(t) * M;
    float gv[MAXM];
#pragma unroll
    for (int e = 0; e < MAXM; ++e) {
        gv[e] = e < M ? fadd(fadd(0.f, fmul(gl, p[e])), fmul(p[e], fsub(gp[e], dot))) : 0.f;
        if (e < M) grow[e] = gv[e];
    }
    if (glog_bf) {  // the router-gradient GEMM operand: [T_pad x 128], columns >= M stay zero
        __nv_bfloat162* brow = reinterpret_cast<__nv_bfloat162*>(glog_bf + static_cast<int64_t>(t) * 128);
#pragma unroll
        for (int e = 0; e < MAXM; e += 2)
            if (e < M) brow[e / 2] = __floats2bfloat162_rn(gv[e], e + 1 < M ? gv[e + 1] : 0.f);
    }
}

constexpr int NG_TT = 32;   // tokens per tile
constexpr int NG_QT = 128;  // columns per tile

// grid (T/32, d/128), 256 threads: thread (ty, tx) -> tokens 4ty..4ty+3, columns 4tx..4tx+3
template <int MAXM, bool ALLK>
__global__ void __launch_bounds__(256, ALLK ? 4 : 1) normed_grad_k(
    const float* __restrict__ h, const int32_t* __restrict__ hrow, const float* __restrict__ gain,
    const float* __restrict__ R,
    const float* __restrict__ glog, const int32_t* __restrict__ slot_row,
    const float* __restrict__ dxp, int T, int d, int M, int k, float* __restrict__ gnormed,
    float* __restrict__ dot_part, int prefetch) {
    // router tile, transposed: [e][q]; pitch NG_QT + 4 makes the staging stores 2-way
    // instead of 16-way bank conflicts (float4 reads stay aligned and conflict-free)
    __shared__ __align__(16) float sRT[MAXM][NG_QT + 4];
    __shared__ float sG[NG_TT][MAXM];
    __shared__ int32_t sRow[NG_TT][8];
    const int t0 = blockIdx.x * NG_TT, q0 = blockIdx.y * NG_QT;
    // the tile's router rows [q0, q0 + 128) x M and glog rows [t0, t0 + 32) x M are contiguous;
    // power-of-two M and k (every shipped config) index them by shifts, not integer division
    if ((M & (M - 1)) == 0 && (k & (k - 1)) == 0) {
        const int lm = __ffs(M) - 1, lk = __ffs(k) - 1;
        const float* Rt = R + static_cast<int64_t>(q0) * M;
        for (int i = threadIdx.x; i < NG_QT * M; i += blockDim.x) sRT[i & (M - 1)][i >> lm] = __ldg(Rt + i);
        const float* Gt = glog + static_cast<int64_t>(t0) * M;
        for (int i = threadIdx.x; i < NG_TT * M; i += blockDim.x)
            sG[i >> lm][i & (M - 1)] = (t0 + (i >> lm) < T) ? Gt[i] : 0.f;
        const int32_t* St = slot_row + static_cast<int64_t>(t0) * k;
        for (int i = threadIdx.x; i < NG_TT * k; i += blockDim.x)
            sRow[i >> lk][i & (k - 1)] = (t0 + (i >> lk) < T) ? St[i] : 0;
    } else {
        for (int i = threadIdx.x; i < NG_QT * M; i += blockDim.x) {
            const int qq = i / M, e = i % M;
            sRT[e][qq] = __ldg(R + static_cast<int64_t>(q0 + qq) * M + e);
        }
        for (int i = threadIdx.x; i < NG_TT * M; i += blockDim.x) {
            const int tt = i / M, e = i % M;
            sG[tt][e] = (t0 + tt < T) ? glog[static_cast<int64_t>(t0 + tt) * M + e] : 0.f;
        }
        for (int i = threadIdx.x; i < NG_TT * k; i += blockDim.x) {
            const int tt = i / k, s = i % k;
            sRow[tt][s] = (t0 + tt < T) ? slot_row[static_cast<int64_t>(t0 + tt) * k + s] : 0;
        }
    }
    __syncthreads();
    const int ty = threadIdx.x >> 5, tx = threadIdx.x & 31;
    // the expert dX rows this thread sums after the router product: their DRAM reads start
    // now (L2 prefetch), under the product's chains, instead of after them
    if (prefetch) {
        const float* dxc = dxp + q0 + 4 * tx;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int tt = ty * 4 + i;
            if (t0 + tt >= T) break;
            for (int s = 0; s < k; ++s)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(dxc + static_cast<int64_t>(sRow[tt][s]) * d));
        }
    }
    // router product for 4 tokens x 4 columns: one broadcast glog load per token and
    // one router load per column feed 16 independent sequential-e chains
    float sr[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sr[i][j] = 0.f;
    // this thread's columns: q0 + 4tx .. q0 + 4tx + 3 (float4 everywhere)
#pragma unroll 4
    for (int e = 0; e < M; ++e) {
        float g[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) g[i] = sG[ty * 4 + i][e];
        const float4 r4 = *reinterpret_cast<const float4*>(&sRT[e][4 * tx]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // fused multiply-adds (a gradient: tolerance-level)
            sr[i][0] = fmaf(g[i], r4.x, sr[i][0]);
            sr[i][1] = fmaf(g[i], r4.y, sr[i][1]);
            sr[i][2] = fmaf(g[i], r4.z, sr[i][2]);
            sr[i][3] = fmaf(g[i], r4.w, sr[i][3]);
        }
    }
    const float4 gq = __ldg(reinterpret_cast<const float4*>(gain + q0 + 4 * tx));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int tt = ty * 4 + i;
        const int t = t0 + tt;
        if (t >= T) break;
        // expert dX rows in descending expert order (select_rows backward, j descending)
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        const float* dxc = dxp + q0 + 4 * tx;
        if constexpr (ALLK) {  // all k row pieces in flight at once (k <= 8), summed descending
            float4 v[8];
#pragma unroll
            for (int s = 0; s < 8; ++s)
                if (s < k)
                    v[s] = __ldg(reinterpret_cast<const float4*>(dxc + static_cast<int64_t>(sRow[tt][s]) * d));
#pragma unroll
            for (int s = 7; s >= 0; --s) {
                if (s < k) {
                    a[0] = fadd(a[0], v[s].x);
                    a[1] = fadd(a[1], v[s].y);
                    a[2] = fadd(a[2], v[s].z);
                    a[3] = fadd(a[3], v[s].w);
                }
            }
        } else {
#pragma unroll 2
            for (int s = k - 1; s >= 0; --s) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(dxc + static_cast<int64_t>(sRow[tt][s]) * d));
                a[0] = fadd(a[0], v.x);
                a[1] = fadd(a[1], v.y);
                a[2] = fadd(a[2], v.z);
                a[3] = fadd(a[3], v.w);
            }
        }
        const int64_t xr_t = hrow ? static_cast<int64_t>(hrow[t]) : t;
        const float4 xv = __ldg(reinterpret_cast<const float4*>(h + xr_t * d + q0 + 4 * tx));
        float4 o;
        o.x = fadd(a[0], sr[i][0]);
        o.y = fadd(a[1], sr[i][1]);
        o.z = fadd(a[2], sr[i][2]);
        o.w = fadd(a[3], sr[i][3]);
        *reinterpret_cast<float4*>(gnormed + static_cast<int64_t>(t) * d + q0 + 4 * tx) = o;
        float part = (o.x * gq.x) * xv.x + (o.y * gq.y) * xv.y + (o.z * gq.z) * xv.z +
                     (o.w * gq.w) * xv.w;
        part = warp_sum(part);
        if (tx == 0) dot_part[static_cast<int64_t>(t) * (d / NG_QT) + blockIdx.y] = part;
    }
}

void router_scalar_backward(const float* probs, const float* lse_r, const float* denom,
                            const int32_t* topk_idx, const int32_t* slot_row, const float* gw_row,
                            const float* lb_coeff, int64_t T, int M, int k, int renorm,
                            float g_lbsum, float g_s, float* glog, bf16* glog_bf,
                            cudaStream_t s) {
    const unsigned g1 = static_cast<unsigned>((T + 127) / 128);
    auto f = M <= 8    ? router_scalar_bwd_k<8>
             : M <= 16 ? router_scalar_bwd_k<16>
             : M <= 32 ? router_scalar_bwd_k<32>
                       : router_scalar_bwd_k<64>;
    f<<<g1, 128, 0, s>>>(probs, lse_r, denom, topk_idx, slot_row, gw_row, lb_coeff, (int)T, M, k,
                         renorm, g_lbsum, g_s, glog, glog_bf);
    count_launch();
}

void normed_grad(const float* h, const int32_t* hrow, const float* gain, const float* router,
                 const int32_t* slot_row, const float* dxp, int64_t T, int64_t d, int M, int k,
                 const float* glog, float* gnormed, float* dot_part, cudaStream_t s) {
    const dim3 g2(static_cast<unsigned>((T + NG_TT - 1) / NG_TT), static_cast<unsigned>(d / NG_QT));
    // all k expert pieces in flight (64 registers, 4 blocks per SM) for k > 4: cfg5 router
    // backward 218 -> 210 ms per round; at k = 2 (cfg2) the 2-deep loop is faster (4.4 vs
    // 4.7 ms). SPES_NG_ALLK=0/1 overrides.
    const char* allk_env = std::getenv("SPES_NG_ALLK");  // read per launch (graph-captured)
    const bool allk = allk_env ? std::atoi(allk_env) != 0 : k > 4;
    auto f = M <= 8    ? (allk ? normed_grad_k<8, true> : normed_grad_k<8, false>)
             : M <= 16 ? (allk ? normed_grad_k<16, true> : normed_grad_k<16, false>)
             : M <= 32 ? (allk ? normed_grad_k<32, true> : normed_grad_k<32, false>)
                       : (allk ? normed_grad_k<64, true> : normed_grad_k<64, false>);
    static const int pf = [] {
        const char* e = std::getenv("SPES_NG_PREFETCH");
        return e ? std::atoi(e) : 1;
    }();
    f<<<g2, 256, 0, s>>>(h, hrow, gain, router, glog, slot_row, dxp, (int)T, (int)d, M, k, gnormed,
                         dot_part, pf);
    count_launch();
}

}  // namespace spes_k

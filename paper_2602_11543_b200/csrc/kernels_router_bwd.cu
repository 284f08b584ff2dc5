// Router backward + rmsnorm backward of one layer (the non-GEMM half of the layer's
// backward pass), following the reverse tape:
//   probs.grad  = (0 + g_lb*coeff_j) [lb, model.hpp:358] + gate-weight grads (experts desc.)
//   logits.grad = (0 + gl*p_j) [moe_z logsumexp] + p_j*(gprobs_j - dot) [softmax bwd]
//   normed.grad = dX of selected experts (desc.) + glog . R^T [matmul_nt_acc]
//   h.grad     += rmsnorm backward (kernels.hpp:130-152)
// Block = 8 warps x TPW tokens. Lanes < TPW of each warp do the per-token scalar
// part (M values) in the reference's order; the d-wide part runs across the warp
// with the router weights staged through shared memory one 128-row chunk at a
// time (each chunk serves all the block's tokens), keeping every element's own
// accumulation order.
#include "common.cuh"
#include "kernels.h"

namespace spes_k {

using namespace spes_dev;

constexpr int RB_TPW = 4;   // tokens per warp
constexpr int RB_QCH = 128; // router rows per smem chunk

template <int MAXM>
__global__ void __launch_bounds__(256) router_bwd_k(
    const float* __restrict__ h, const float* __restrict__ gain, const float* __restrict__ R,
    const float* __restrict__ probs, const float* __restrict__ lse_r,
    const float* __restrict__ inv_rms, const float* __restrict__ denom,
    const int32_t* __restrict__ topk_idx, const int32_t* __restrict__ slot_row,
    const float* __restrict__ gw_row, const float* __restrict__ dxp,
    const float* __restrict__ lb_coeff, int T, int d, int M, int k, int renorm, float g_lbsum,
    float g_s, float* __restrict__ glog, float* __restrict__ gnormed, float* __restrict__ gh) {
    __shared__ float sR[RB_QCH * (MAXM + 1)];
    __shared__ float sg[8][RB_TPW][MAXM];
    __shared__ int32_t srow[8][RB_TPW][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tbase = (blockIdx.x * 8 + warp) * RB_TPW;

    // ---- per-token scalar part: lane i handles token tbase + i ----
    if (lane < RB_TPW) {
        const int t = tbase + lane;
        if (t < T) {
            float p[MAXM], gp[MAXM];
            const float* prow = probs + static_cast<int64_t>(t) * M;
#pragma unroll
            for (int e = 0; e < MAXM; ++e) {
                if (e < M) {
                    p[e] = prow[e];
                    gp[e] = fadd(0.f, fmul(g_lbsum, __ldg(lb_coeff + e)));
                }
            }
            int32_t sel[8];
            for (int s = 0; s < k; ++s) {
                sel[s] = topk_idx[static_cast<int64_t>(t) * k + s];
                srow[warp][lane][s] = slot_row[static_cast<int64_t>(t) * k + s];
            }
            const float dn = renorm ? denom[t] : 1.f;
            float gden = 0.f;
            for (int s = k - 1; s >= 0; --s) {  // experts in descending order
                const float gw = gw_row[srow[warp][lane][s]];
                const int j = sel[s];
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
#pragma unroll
            for (int e = 0; e < MAXM; ++e) {
                if (e < M) {
                    const float g = fadd(fadd(0.f, fmul(gl, p[e])), fmul(p[e], fsub(gp[e], dot)));
                    grow[e] = g;
                    sg[warp][lane][e] = g;
                }
            }
        }
    }

    // ---- d-wide part ----
    float dot2[RB_TPW];
#pragma unroll
    for (int i = 0; i < RB_TPW; ++i) dot2[i] = 0.f;
    for (int q0 = 0; q0 < d; q0 += RB_QCH) {
        __syncthreads();  // also publishes sg / srow on the first chunk
        for (int i = threadIdx.x; i < RB_QCH * M; i += blockDim.x) {
            const int qq = i / M, e = i % M;
            sR[qq * (MAXM + 1) + e] = __ldg(R + static_cast<int64_t>(q0 + qq) * M + e);
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < RB_TPW; ++i) {
            const int t = tbase + i;
            if (t >= T) break;
            const float* xr = h + static_cast<int64_t>(t) * d;
            float* gy = gnormed + static_cast<int64_t>(t) * d;
#pragma unroll
            for (int u = 0; u < RB_QCH / 32; ++u) {
                const int qq = lane + 32 * u;
                const int q = q0 + qq;
                float a = 0.f;
                for (int s = k - 1; s >= 0; --s)
                    a = fadd(a, __ldg(dxp + static_cast<int64_t>(srow[warp][i][s]) * d + q));
                float sr = 0.f;
                const float* rr = sR + qq * (MAXM + 1);
#pragma unroll
                for (int e = 0; e < MAXM; ++e)
                    if (e < M) sr = fadd(sr, fmul(sg[warp][i][e], rr[e]));
                a = fadd(a, sr);
                gy[q] = a;
                dot2[i] += (a * __ldg(gain + q)) * __ldg(xr + q);
            }
        }
    }
    // ---- rmsnorm backward into h.grad ----
#pragma unroll
    for (int i = 0; i < RB_TPW; ++i) {
        const int t = tbase + i;
        const float tot = warp_sum(dot2[i]);
        if (t >= T) continue;
        const float inv = inv_rms[t];
        const float coef = fdiv(fmul(fmul(fmul(tot, inv), inv), inv), static_cast<float>(d));
        const float* xr = h + static_cast<int64_t>(t) * d;
        const float* gy = gnormed + static_cast<int64_t>(t) * d;
        float* ghr = gh + static_cast<int64_t>(t) * d;
        for (int q0 = lane * 4; q0 < d; q0 += 128) {
            const float4 a = *reinterpret_cast<const float4*>(gy + q0);
            const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + q0));
            const float4 gv = __ldg(reinterpret_cast<const float4*>(gain + q0));
            float4 o = *reinterpret_cast<const float4*>(ghr + q0);
            o.x = fadd(o.x, fsub(fmul(fmul(a.x, gv.x), inv), fmul(coef, xv.x)));
            o.y = fadd(o.y, fsub(fmul(fmul(a.y, gv.y), inv), fmul(coef, xv.y)));
            o.z = fadd(o.z, fsub(fmul(fmul(a.z, gv.z), inv), fmul(coef, xv.z)));
            o.w = fadd(o.w, fsub(fmul(fmul(a.w, gv.w), inv), fmul(coef, xv.w)));
            *reinterpret_cast<float4*>(ghr + q0) = o;
        }
    }
}

void router_backward(const float* h, const float* gain, const float* router, const float* probs,
                     const float* lse_r, const float* inv_rms, const float* denom,
                     const int32_t* topk_idx, const int32_t* slot_row, const float* gw_row,
                     const float* dxp, const float* lb_coeff, int64_t T, int64_t d, int M, int k,
                     int renorm, float g_lbsum, float g_s, float* glog, float* gnormed,
                     float* gh, cudaStream_t s) {
    const unsigned grid = static_cast<unsigned>((T + 8 * RB_TPW - 1) / (8 * RB_TPW));
#define SPES_RB(MM)                                                                              \
    router_bwd_k<MM><<<grid, 256, 0, s>>>(h, gain, router, probs, lse_r, inv_rms, denom, topk_idx, \
                                          slot_row, gw_row, dxp, lb_coeff, (int)T, (int)d, M, k,   \
                                          renorm, g_lbsum, g_s, glog, gnormed, gh)
    if (M <= 8)
        SPES_RB(8);
    else if (M <= 16)
        SPES_RB(16);
    else if (M <= 32)
        SPES_RB(32);
    else
        SPES_RB(64);
#undef SPES_RB
    count_launch();
}

}  // namespace spes_k

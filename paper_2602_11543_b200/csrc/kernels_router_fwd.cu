// Router forward, bit-exact with the reference given identical h:
//   rmsnorm_forward (kernels.hpp:117-128): sequential sum of squares, y = (x*inv)*g
//   matmul (kernels.hpp:27-38): logit_e = sum_p normed_p * R[p][e], p ascending, no FMA
//   softmax_rows (kernels.hpp:156-172) with the glibc-compatible expf; logsumexp (:174-185)
//   route_from_logits (model.hpp:185-216): stable top-k, ascending indices, weights
//
// Layout: a token's (padded) experts are split over LPT lanes, 8 experts per lane
// (lane = token * LPT + part). A warp stages its TPW = 32/LPT token rows
// through a per-warp cp.async ring (64-column chunks, padded pitch => conflict-free
// LDS.128), the block stages the matching router rows and gain chunk, so every lane runs
// its token's sequential sum-of-squares chain and then 8 independent exact-order logit
// chains fed by broadcast LDS.128 of router rows. Softmax / top-k run on the token's
// first lane over the logits gathered in smem. normed is emitted as bf16 (the expert
// GEMM operand, permuted by route_plan) and, for the kernel-level API only, as fp32.
#include "common.cuh"
#include "glibc_expf.h"
#include "kernels.h"

namespace spes_k {

using namespace spes_dev;

constexpr int RF_WARPS = 4;  // warps per block (march through p together)
constexpr int RF_RCH = 64;   // router rows per smem chunk
constexpr int RF_XS = 3;     // ring depth (chunks of RF_RCH columns of x and rows of R)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

__device__ __forceinline__ uint2 pack_bf16x4(float a, float b, float c, float d) {
    __nv_bfloat162 x = __floats2bfloat162_rn(a, b);
    __nv_bfloat162 y = __floats2bfloat162_rn(c, d);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&x);
    u.y = *reinterpret_cast<uint32_t*>(&y);
    return u;
}

// TT = tokens per lane: 1 for M <= 16; 4 for M = 32 / 64, where each router value read
// from shared memory then feeds 4 tokens' chains (the M = 64 kernel was bound by
// shared-memory wavefronts at TT = 1)
template <int MAXM>
struct RfSmem {
    static constexpr int EPL = MAXM < 8 ? MAXM : 8;  // experts per lane
    static constexpr int LPT = MAXM / EPL;           // lanes per token group
    static constexpr int TT = MAXM >= 32 ? 4 : 1;    // tokens per lane (per group)
    static constexpr int TPW = TT * (32 / LPT);      // tokens per warp
    static constexpr int RCH = MAXM >= 32 ? 32 : RF_RCH;  // columns (router rows) per chunk
    static constexpr int PITCH = RCH + 4;  // padded row pitch (floats): conflict-free LDS.128
    static constexpr int R_FLOATS = RF_XS * RCH * MAXM;   // router row ring
    static constexpr int G_FLOATS = RF_XS * RCH;          // gain ring
    static constexpr int X_FLOATS = RF_WARPS * RF_XS * TPW * PITCH;  // per-warp token-row rings
    static constexpr int BYTES = 4 * (R_FLOATS + G_FLOATS + X_FLOATS);
};

template <int MAXM>
__global__ void __launch_bounds__(32 * RF_WARPS) router_fwd_k(
    const float* __restrict__ h, const int32_t* __restrict__ hrow, const float* __restrict__ gain,
    const float* __restrict__ R,
    int T, int d, int dn_rms, int M, int k, int renorm, float eps, int variant,
    float* __restrict__ normed,
    bf16* __restrict__ normed_bf, float* __restrict__ logits, float* __restrict__ probs,
    int32_t* __restrict__ topk_idx, float* __restrict__ topk_w, float* __restrict__ lse_out,
    float* __restrict__ inv_out, float* __restrict__ denom_out) {
    using SM = RfSmem<MAXM>;
    constexpr int EPL = SM::EPL, LPT = SM::LPT, TPW = SM::TPW, TT = SM::TT;
    constexpr int RCH = SM::RCH;
    constexpr int QC = RCH / 4;  // float4 per row chunk
    constexpr int PITCH = SM::PITCH;
    extern __shared__ __align__(16) float rf_smem[];
    float(*sR)[RCH][MAXM] = reinterpret_cast<float(*)[RCH][MAXM]>(rf_smem);  // [RF_XS]
    float(*sG)[RCH] = reinterpret_cast<float(*)[RCH]>(rf_smem + SM::R_FLOATS);
    float(*sxw)[TPW][PITCH] = reinterpret_cast<float(*)[TPW][PITCH]>(
        rf_smem + SM::R_FLOATS + SM::G_FLOATS);  // [warp * RF_XS + slot]
    __shared__ float sv_all[RF_WARPS][TPW][MAXM + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float(*sv)[MAXM + 1] = sv_all[warp];
    const int grp = lane / LPT, part = lane % LPT, e0 = part * EPL;
    const int tw0 = (blockIdx.x * RF_WARPS + warp) * TPW;  // first token of this warp
    const int r0 = grp * TT;                                // this lane's first row in the warp
    const int nrc = d / RCH;  // row chunks (= router / gain chunks)

    // chunk c of the warp's TPW rows (RCH floats each) -> ring slot c % RF_XS;
    // 16 lanes per row => 256-byte contiguous cp.async runs; rows past T are clamped.
    auto issue_x = [&](int c) {
        float(*dst)[PITCH] = sxw[warp * RF_XS + c % RF_XS];
#pragma unroll 4
        for (int i = lane; i < TPW * QC; i += 32) {
            const int row = i / QC, q = i % QC;
            const int tc = min(tw0 + row, T - 1);
            const int64_t tr = hrow ? static_cast<int64_t>(__ldg(hrow + tc)) : tc;
            cp_async16(&dst[row][4 * q], h + tr * d + c * RCH + 4 * q);
        }
    };
    // router rows [c*RCH, +RCH) -> sR[c % RF_XS] and gain -> sG (block-cooperative);
    // experts M..MAXM-1 are zero columns
    auto issue_rg = [&](int c) {
        float* dst = &sR[c % RF_XS][0][0];
        const float* src = R + static_cast<int64_t>(c) * RCH * M;
        if ((M & 3) == 0 && M == MAXM) {
            for (int i = threadIdx.x; i < RCH * MAXM / 4; i += blockDim.x)
                cp_async16(dst + 4 * i, src + 4 * i);
        } else {
            for (int i = threadIdx.x; i < RCH * MAXM; i += blockDim.x) {
                const int rr = i / MAXM, e = i % MAXM;
                dst[i] = e < M ? __ldg(src + static_cast<int64_t>(rr) * M + e) : 0.f;
            }
        }
        if (threadIdx.x < QC)
            cp_async16(&sG[c % RF_XS][4 * threadIdx.x], gain + c * RCH + 4 * threadIdx.x);
    };
    auto wait_oldest = [&]() {  // group of the oldest in-flight chunk complete
        asm volatile("cp.async.wait_group %0;" ::"n"(RF_XS - 2) : "memory");
    };

    // ---- pass 1: rmsnorm_forward sum of squares, sequential over p (kernels.hpp:117-128);
    // the LPT lanes of a group run the same TT chains
    float ms[TT];
#pragma unroll
    for (int j = 0; j < TT; ++j) ms[j] = 0.f;
#pragma unroll
    for (int c = 0; c < RF_XS - 1; ++c) {
        if (c < nrc) issue_x(c);
        cp_async_commit();
    }
    for (int c = 0; c < nrc; ++c) {
        wait_oldest();
        __syncwarp();  // every lane's copies of chunk c visible; slot (c-1) % XS free
        if (c + RF_XS - 1 < nrc) issue_x(c + RF_XS - 1);
        cp_async_commit();
#pragma unroll
        for (int j = 0; j < TT; ++j) {
            const float* xrow = sxw[warp * RF_XS + c % RF_XS][r0 + j];
#pragma unroll
            for (int i = 0; i < QC; ++i) {
                const float4 x = *reinterpret_cast<const float4*>(xrow + 4 * i);
                const float2 lo = fmul2(make_float2(x.x, x.y), make_float2(x.x, x.y));
                const float2 hi = fmul2(make_float2(x.z, x.w), make_float2(x.z, x.w));
                ms[j] = fadd(ms[j], lo.x);
                ms[j] = fadd(ms[j], lo.y);
                ms[j] = fadd(ms[j], hi.x);
                ms[j] = fadd(ms[j], hi.y);
            }
        }
    }
    float inv[TT];
#pragma unroll
    for (int j = 0; j < TT; ++j)  // mean over the model's hidden width (rows may be zero-padded)
        inv[j] = fdiv(1.f, fsqrt(fadd(fdiv(ms[j], static_cast<float>(dn_rms)), eps)));
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // all warps done with pass 1 before the rings are reused

    // ---- pass 2: normed = (x * inv) * g; logit_e = sum_p normed_p * R[p][e], p ascending,
    // no FMA; this lane owns experts [e0, e0 + EPL) of its TT tokens. Each cp.async group
    // carries {x chunk c of this warp, this thread's share of R / gain chunk c}; the block
    // barrier after the wait makes chunk c visible to all and frees slot (c-1) % XS.
    float acc[TT][EPL];
#pragma unroll
    for (int j = 0; j < TT; ++j)
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[j][e] = 0.f;
#pragma unroll
    for (int c = 0; c < RF_XS - 1; ++c) {
        if (c < nrc) {
            issue_x(c);
            issue_rg(c);
        }
        cp_async_commit();
    }
    for (int c = 0; c < nrc; ++c) {
        wait_oldest();
        __syncthreads();
        if (c + RF_XS - 1 < nrc) {
            issue_x(c + RF_XS - 1);
            issue_rg(c + RF_XS - 1);
        }
        cp_async_commit();
        const float(*rr)[MAXM] = sR[c % RF_XS];
        const float* gg = sG[c % RF_XS];
#pragma unroll 2
        for (int i = 0; i < QC; i += 2) {  // 8 p per iteration => one 16-byte bf16 store
            float nv[TT][8];
#pragma unroll
            for (int j = 0; j < TT; ++j) {
                const float* xrow = sxw[warp * RF_XS + c % RF_XS][r0 + j];
#pragma unroll
                for (int u = 0; u < 2; ++u) {  // (x * inv) * g, two lanes per FMUL2
                    const float4 x = *reinterpret_cast<const float4*>(xrow + 4 * (i + u));
                    const float4 g = *reinterpret_cast<const float4*>(gg + 4 * (i + u));
                    const float2 iv = make_float2(inv[j], inv[j]);
                    const float2 lo = fmul2(fmul2(make_float2(x.x, x.y), iv), make_float2(g.x, g.y));
                    const float2 hi = fmul2(fmul2(make_float2(x.z, x.w), iv), make_float2(g.z, g.w));
                    nv[j][4 * u + 0] = lo.x;
                    nv[j][4 * u + 1] = lo.y;
                    nv[j][4 * u + 2] = hi.x;
                    nv[j][4 * u + 3] = hi.y;
                }
            }
#pragma unroll
            for (int jp = 0; jp < 8; ++jp) {
                const float* rrow = rr[4 * i + jp] + e0;
#pragma unroll
                for (int e4 = 0; e4 < EPL; e4 += 4) {
                    const float4 r = *reinterpret_cast<const float4*>(rrow + e4);
#pragma unroll
                    for (int j = 0; j < TT; ++j) {
                        const float2 nn = make_float2(nv[j][jp], nv[j][jp]);
                        const float2 p01 = fmul2(nn, make_float2(r.x, r.y));
                        const float2 p23 = fmul2(nn, make_float2(r.z, r.w));
                        acc[j][e4 + 0] = fadd(acc[j][e4 + 0], p01.x);
                        acc[j][e4 + 1] = fadd(acc[j][e4 + 1], p01.y);
                        acc[j][e4 + 2] = fadd(acc[j][e4 + 2], p23.x);
                        acc[j][e4 + 3] = fadd(acc[j][e4 + 3], p23.y);
                    }
                }
            }
            // normed stores: each (token, 8-column group) written once, spread over the group
#pragma unroll
            for (int j = 0; j < TT; ++j) {
                const int t = tw0 + r0 + j;
                if (t < T && ((i >> 1) % LPT) == part) {
                    const int p0 = c * RCH + 4 * i;
                    if (normed_bf) {
                        uint4 pk;
                        const uint2 lo = pack_bf16x4(nv[j][0], nv[j][1], nv[j][2], nv[j][3]);
                        const uint2 hi = pack_bf16x4(nv[j][4], nv[j][5], nv[j][6], nv[j][7]);
                        pk.x = lo.x; pk.y = lo.y; pk.z = hi.x; pk.w = hi.y;
                        *reinterpret_cast<uint4*>(normed_bf + static_cast<int64_t>(t) * d + p0) = pk;
                    }
                    if (normed) {
                        float* nf = normed + static_cast<int64_t>(t) * d + p0;
                        *reinterpret_cast<float4*>(nf) = make_float4(nv[j][0], nv[j][1], nv[j][2], nv[j][3]);
                        *reinterpret_cast<float4*>(nf + 4) = make_float4(nv[j][4], nv[j][5], nv[j][6], nv[j][7]);
                    }
                }
            }
        }
    }

    // ---- softmax_rows (kernels.hpp:156-172) and route_from_logits (model.hpp:185-216):
    // logits gathered per token in smem; the scans of token r0 + j run on the group's lane
    // part == j
#pragma unroll
    for (int j = 0; j < TT; ++j)
#pragma unroll
        for (int e = 0; e < EPL; ++e) sv[r0 + j][e0 + e] = acc[j][e];
    __syncwarp();
    if (part >= TT) return;
    const int j = part;
    const int t = tw0 + r0 + j;
    if (t >= T) return;
    float* lrow = logits + static_cast<int64_t>(t) * M;
    float* prow = probs + static_cast<int64_t>(t) * M;
    float* pv = sv[r0 + j];
    float mx = pv[0];
    for (int e = 0; e < M; ++e) {
        lrow[e] = pv[e];
        if (e > 0) mx = (mx < pv[e]) ? pv[e] : mx;  // std::max scan (kernels.hpp:160)
    }
    float sum = 0.f;
    for (int e = 0; e < M; ++e) {
        const float z = fsub(pv[e], mx);
        const float ex = variant ? spes_expf::expf_glibc<1>(z) : spes_expf::expf_glibc<0>(z);
        pv[e] = ex;
        sum = fadd(sum, ex);
    }
    const float rs = fdiv(1.f, sum);
    lse_out[t] = mx + logf(sum);
    float invj = inv[0];
#pragma unroll
    for (int jj = 1; jj < TT; ++jj)
        if (jj == j) invj = inv[jj];
    inv_out[t] = invj;
    for (int e = 0; e < M; ++e) {
        pv[e] = fmul(pv[e], rs);  // probabilities
        prow[e] = pv[e];
    }
    // iterative argmax (strict '>' scanning ascending => lowest index on ties) == the
    // first k of a stable descending sort; then ascending order
    uint64_t chosen = 0;
    for (int s2 = 0; s2 < k; ++s2) {
        int best = -1;
        float bv = 0.f;
        for (int jj = 0; jj < M; ++jj) {
            if (!((chosen >> jj) & 1ull) && (best < 0 || pv[jj] > bv)) {
                best = jj;
                bv = pv[jj];
            }
        }
        chosen |= 1ull << best;
    }
    float dn = 0.f;
    for (int jj = 0; jj < M; ++jj)
        if ((chosen >> jj) & 1ull) dn = fadd(dn, pv[jj]);
    int slot = 0;
    for (int jj = 0; jj < M; ++jj) {
        if ((chosen >> jj) & 1ull) {
            topk_idx[static_cast<int64_t>(t) * k + slot] = jj;
            topk_w[static_cast<int64_t>(t) * k + slot] = renorm ? fdiv(pv[jj], dn) : pv[jj];
            ++slot;
        }
    }
    if (denom_out) denom_out[t] = dn;
}

template <int MM>
static void launch_rf(unsigned grid, cudaStream_t s, const float* h, const int32_t* hrow,
                      const float* gain,
                      const float* router, int64_t T, int64_t d, int64_t dn, int M, int k,
                      int renorm,
                      float eps, int variant, float* normed, bf16* normed_bf, float* logits,
                      float* probs, int32_t* topk_idx, float* topk_w, float* lse, float* inv_rms,
                      float* denom) {
    static std::atomic<uint64_t> configured{0};
    if (first_use_on_device(configured))
        cudaFuncSetAttribute(router_fwd_k<MM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             RfSmem<MM>::BYTES);
    router_fwd_k<MM><<<grid, 32 * RF_WARPS, RfSmem<MM>::BYTES, s>>>(
        h, hrow, gain, router, (int)T, (int)d, (int)dn, M, k, renorm, eps, variant, normed, normed_bf,
        logits,
        probs, topk_idx, topk_w, lse, inv_rms, denom);
}

void router_forward(const float* h, const int32_t* hrow, const float* gain, const float* router,
                    int64_t T, int64_t d, int64_t dn,
                    int M, int k, int renorm, float eps, int variant, float* normed,
                    bf16* normed_bf, float* logits, float* probs, int32_t* topk_idx,
                    float* topk_w, float* lse, float* inv_rms, float* denom, cudaStream_t s) {
    const int maxm = M <= 8 ? 8 : (M <= 16 ? 16 : (M <= 32 ? 32 : 64));
    const int per_block = RF_WARPS * (maxm == 8    ? RfSmem<8>::TPW
                                      : maxm == 16 ? RfSmem<16>::TPW
                                      : maxm == 32 ? RfSmem<32>::TPW
                                                   : RfSmem<64>::TPW);
    const unsigned grid = static_cast<unsigned>((T + per_block - 1) / per_block);
    auto* f = maxm == 8 ? launch_rf<8> : maxm == 16 ? launch_rf<16> : maxm == 32 ? launch_rf<32>
                                                                                  : launch_rf<64>;
    f(grid, s, h, hrow, gain, router, T, d, dn, M, k, renorm, eps, variant, normed, normed_bf, logits,
      probs,
      topk_idx, topk_w, lse, inv_rms, denom);
    count_launch();
}

}  // namespace spes_k

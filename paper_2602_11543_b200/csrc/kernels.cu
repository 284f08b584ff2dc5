// SPES device kernels other than the tensor-core GEMMs (see gemm.cu).
//
// Exactness policy: kernels on the routing path, the AdamW
// update, the owner-set mean and the merge apply reproduce the reference's fp32
// / fp64 operation order exactly (explicitly rounded ops, sequential reductions,
// glibc-compatible expf), so they are bit-exact given identical inputs. Loss
// scalars and the column reductions feeding parameter gradients use fixed-order
// parallel trees: deterministic run to run, within tolerance of the reference.
#include <cuda_bf16.h>
#include <stdio.h>

#include <algorithm>

#include <stdexcept>
#include <type_traits>

#include "common.cuh"
#include "glibc_expf.h"
#include "kernels.h"
#include "sm100_primitives.cuh"

namespace spes_k {

thread_local int64_t* g_launch_counter = nullptr;

using namespace spes_dev;

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ============================ embedding gather ============================
// h0[t] = emb[inputs[t]] (model.hpp:286, graph.hpp:208-219)
__global__ void embed_gather_k(const float* __restrict__ emb, const int32_t* __restrict__ tokens,
                               int64_t S, int64_t d, int64_t V, float* __restrict__ h,
                               int32_t* __restrict__ inputs, int32_t* __restrict__ targets,
                               int32_t* err) {
    const int64_t t = blockIdx.x;
    const int64_t b = t / S, s = t % S;
    int32_t tin = tokens[b * (S + 1) + s], tout = tokens[b * (S + 1) + s + 1];
    const bool bad = tin < 0 || tin >= V || tout < 0 || tout >= V;
    if (threadIdx.x == 0) {
        inputs[t] = bad ? 0 : tin;
        targets[t] = bad ? 0 : tout;
        if (bad) atomicOr(err, 1);
    }
    if (bad) tin = 0;
    if (!h) return;  // layer-0 input read in place as emb[inputs[t]] by its consumers
    const float4* src = reinterpret_cast<const float4*>(emb + static_cast<int64_t>(tin) * d);
    float4* dst = reinterpret_cast<float4*>(h + t * d);
    for (int64_t q = threadIdx.x; q < d / 4; q += blockDim.x) dst[q] = __ldg(src + q);
}

// inputs / targets only (layer 0 reads emb[inputs] in place): a thread per token
__global__ void split_tokens_k(const int32_t* __restrict__ tokens, int64_t T, int64_t S, int64_t V,
                               int32_t* __restrict__ inputs, int32_t* __restrict__ targets,
                               int32_t* err) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const int64_t b = t / S, s = t % S;
    const int32_t tin = tokens[b * (S + 1) + s], tout = tokens[b * (S + 1) + s + 1];
    const bool bad = tin < 0 || tin >= V || tout < 0 || tout >= V;
    inputs[t] = bad ? 0 : tin;
    targets[t] = bad ? 0 : tout;
    if (bad) atomicOr(err, 1);
}

void embed_gather(const float* emb, const int32_t* tokens, int64_t B, int64_t S, int64_t d,
                  int64_t V, float* h, int32_t* inputs, int32_t* targets, int32_t* err,
                  cudaStream_t s) {
    if (!h) {
        split_tokens_k<<<static_cast<unsigned>(cdiv(B * S, 256)), 256, 0, s>>>(
            tokens, B * S, S, V, inputs, targets, err);
    } else {
        embed_gather_k<<<static_cast<unsigned>(B * S), 128, 0, s>>>(emb, tokens, S, d, V, h,
                                                                    inputs, targets, err);
    }
    count_launch();
}

// ============================ routing plan ============================
constexpr int ROUTE_CH = 256;  // tokens per chunk

__global__ void route_count_k(const int32_t* __restrict__ idx, int T, int M, int k,
                              int32_t* __restrict__ chunk_counts) {
    __shared__ int32_t hist[64];
    for (int j = threadIdx.x; j < M; j += blockDim.x) hist[j] = 0;
    __syncthreads();
    const int t = blockIdx.x * ROUTE_CH + threadIdx.x;
    if (t < T)
        for (int s = 0; s < k; ++s) atomicAdd(&hist[idx[static_cast<int64_t>(t) * k + s]], 1);
    __syncthreads();
    for (int j = threadIdx.x; j < M; j += blockDim.x)
        chunk_counts[static_cast<int64_t>(blockIdx.x) * M + j] = hist[j];
}

// Single block: per-expert scan over chunks, padded offsets, lb coefficients
// (model.hpp:344-353, computed in double exactly as the reference), and the six
// GEMM group tables of the layer.
__global__ void route_scan_k(int32_t* __restrict__ chunk_counts, int nchunks, int T, int M,
                             int k, int32_t* __restrict__ counts, int32_t* __restrict__ pad_off,
                             float* __restrict__ lb_coeff, GemmGroup* __restrict__ groups,
                             int32_t* __restrict__ tiles, GroupBases gb) {
    __shared__ int32_t s_cnt[64];
    __shared__ int32_t s_off[65];
    const int j = threadIdx.x;
    // stage the per-chunk counts (loads in parallel, not one dependent chain per expert)
    extern __shared__ int32_t s_cc[];  // [nchunks][M]
    for (int i = threadIdx.x; i < nchunks * M; i += blockDim.x) s_cc[i] = chunk_counts[i];
    __syncthreads();
    if (j < M) {
        int32_t run = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int32_t v = s_cc[c * M + j];
            s_cc[c * M + j] = run;  // becomes chunk base
            run += v;
        }
        s_cnt[j] = run;
        counts[j] = run;
        const double assignments = static_cast<double>(T) * k;
        const double f_j = static_cast<double>(run) / assignments;
        lb_coeff[j] = static_cast<float>(static_cast<double>(M) * f_j / static_cast<double>(T));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t acc = 0;
        for (int e = 0; e < M; ++e) {
            s_off[e] = acc;
            acc += (s_cnt[e] + gb.tile_rows - 1) / gb.tile_rows * gb.tile_rows;
        }
        s_off[M] = acc;
        for (int e = 0; e <= M; ++e) pad_off[e] = s_off[e];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nchunks * M; i += blockDim.x) chunk_counts[i] = s_cc[i];
    // groups: thread e builds expert e's six groups; tile_start is a prefix over experts
    __shared__ int32_t s_nt[6][64];
    __shared__ GemmGroup s_g[6][64];
    const int64_t d = gb.d, f = gb.f;
    if (j < 6 * M) {  // thread (g, e) builds expert e's group of GEMM g
        const int g = j / M, e = j % M;
        const int32_t mt = (s_off[e + 1] - s_off[e]) / gb.tile_rows;
        const int64_t goff = gb.grad_off_layer ? gb.grad_off_layer[e] : -1;
        {
            GemmGroup G{};
            G.bk0 = 0;
            G.out_row0 = s_off[e];
            G.a_row0 = s_off[e];
            G.k0 = 0;
            G.m_tiles = mt;
            switch (g) {
                case 0:  // fwd gate||up: Xp[R x d] . W1_e[d x 2f] (B MN-major, rows e*d..)
                    G.b_row0 = 0;
                    G.bk0 = static_cast<int32_t>(e * d);
                    G.n_tiles = static_cast<int32_t>(2 * f / 256);
                    G.k_len = static_cast<int32_t>(d);
                    G.out0 = gb.gu;
                    G.ldo = 2 * f;
                    break;
                case 1:  // fwd down: Hact[R x f] . Wd_e[f x d] (B MN-major, rows e*f..)
                    G.b_row0 = 0;
                    G.bk0 = static_cast<int32_t>(e * f);
                    G.n_tiles = static_cast<int32_t>(d / gb.bn_fwd2);
                    G.k_len = static_cast<int32_t>(f);
                    G.out0 = gb.y;
                    G.ldo = d;
                    break;
                case 2:  // bwd dH: dYw[R x d] . Wd_e[f x d]^T
                    G.b_row0 = static_cast<int32_t>(e * f);
                    G.n_tiles = static_cast<int32_t>(f / gb.bn_dh);
                    G.k_len = static_cast<int32_t>(d);
                    G.out0 = gb.dgu;
                    G.ldo = 2 * f;
                    break;
                case 3:  // bwd dX: dGU[R x 2f] . W1_e[d x 2f]^T
                    G.b_row0 = static_cast<int32_t>(e * d);
                    G.n_tiles = static_cast<int32_t>(d / gb.bn_dx);
                    G.k_len = static_cast<int32_t>(2 * f);
                    G.out0 = gb.dxp;
                    G.ldo = d;
                    break;
                case 4:  // bwd dW1 (owned): XpT[d x R] . dGUT[2f x R]^T over this expert's rows
                    G.a_row0 = 0;
                    G.b_row0 = 0;
                    G.k0 = s_off[e];
                    G.bk0 = s_off[e];
                    G.k_len = s_off[e + 1] - s_off[e];
                    G.m_tiles = goff >= 0 ? static_cast<int32_t>(d / gb.tile_rows) : 0;
                    G.n_tiles = static_cast<int32_t>(2 * f / 256);
                    G.out_row0 = 0;
                    G.out0 = goff >= 0 ? gb.grad_expert_base + goff : nullptr;
                    G.out1 = goff >= 0 ? gb.grad_expert_base + goff + d * f : nullptr;
                    G.ldo = f;
                    if (gb.fused_adam && goff >= 0) {  // params / Adam state of wg (wu = +df)
                        G.out0 = gb.param_expert_base + e * 3 * d * f;
                        G.out1 = nullptr;
                        G.out_row0 = goff;
                        G.aux = gb.slot0 + e;
                    }
                    break;
                default:  // bwd dW2 (owned): HactT[f x R] . dYwT[d x R]^T
                    G.a_row0 = 0;
                    G.b_row0 = 0;
                    G.k0 = s_off[e];
                    G.bk0 = s_off[e];
                    G.k_len = s_off[e + 1] - s_off[e];
                    G.m_tiles = goff >= 0 ? static_cast<int32_t>(f / gb.tile_rows) : 0;
                    G.n_tiles = static_cast<int32_t>(d / gb.bn_dw2);
                    G.out_row0 = 0;
                    G.out0 = goff >= 0 ? gb.grad_expert_base + goff + 2 * d * f : nullptr;
                    G.ldo = d;
                    if (gb.fused_adam && goff >= 0) {  // params / Adam state of wd
                        G.out0 = gb.param_expert_base + e * 3 * d * f + 2 * d * f;
                        G.out_row0 = goff + 2 * d * f;
                        G.aux = gb.slot0 + e;
                    }
                    break;
            }
            s_g[g][e] = G;
            s_nt[g][e] = G.m_tiles * G.n_tiles;
        }
    }
    __syncthreads();
    if (j < 6) {
        int32_t acc = 0;
        for (int e = 0; e < M; ++e) {
            const int32_t n = s_nt[j][e];
            s_nt[j][e] = acc;
            acc += n;
        }
        tiles[j] = acc;
    }
    __syncthreads();
    if (j < 6 * M) {
        const int g = j / M, e = j % M;
        GemmGroup G = s_g[g][e];
        G.tile_start = s_nt[g][e];
        groups[g * M + e] = G;
    }
}

// Stable scatter: rows of expert j in ascending token order (model.hpp:314-318).
// Warps of a chunk run one after another; inside a warp, ballots give ranks.
__global__ void route_scatter_k(const int32_t* __restrict__ idx, const float* __restrict__ w,
                                int T, int M, int k, const int32_t* __restrict__ chunk_base,
                                const int32_t* __restrict__ pad_off, int32_t* __restrict__ slot_row,
                                int32_t* __restrict__ row_token, float* __restrict__ row_w) {
    __shared__ int32_t wbase[ROUTE_CH / 32][64];  // per-warp counts, then per-warp bases
    const int t = blockIdx.x * ROUTE_CH + threadIdx.x;
    const bool valid = t < T;
    int32_t sel[8], rank[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        sel[s] = (valid && s < k) ? idx[static_cast<int64_t>(t) * k + s] : -1;
        rank[s] = 0;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    // in-warp ranks: all warps in parallel, one ballot per expert
    for (int j = 0; j < M; ++j) {
        bool has = false;
#pragma unroll
        for (int s = 0; s < 8; ++s) has |= (sel[s] == j);
        const uint32_t mask = __ballot_sync(0xffffffffu, has);
        const int32_t r = __popc(mask & lt);
#pragma unroll
        for (int s = 0; s < 8; ++s)
            if (sel[s] == j) rank[s] = r;
        if (lane == 0) wbase[warp][j] = __popc(mask);
    }
    __syncthreads();
    // exclusive scan over warps in token order, seeded with this chunk's base
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
        int32_t acc = pad_off[j] + chunk_base[static_cast<int64_t>(blockIdx.x) * M + j];
        for (int w8 = 0; w8 < ROUTE_CH / 32; ++w8) {
            const int32_t c = wbase[w8][j];
            wbase[w8][j] = acc;
            acc += c;
        }
    }
    __syncthreads();
    if (!valid) return;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        if (s < k) {
            const int32_t row = wbase[warp][sel[s]] + rank[s];
            slot_row[static_cast<int64_t>(t) * k + s] = row;
            row_token[row] = t;
            row_w[row] = w[static_cast<int64_t>(t) * k + s];
        }
    }
}

void route_plan(const int32_t* topk_idx, const float* topk_w, int64_t T, int M, int k,
                int64_t R_cap, const RoutePlan& p, const GroupBases& gb, cudaStream_t s) {
    const int nchunks = static_cast<int>(cdiv(T, ROUTE_CH));
    route_count_k<<<nchunks, ROUTE_CH, 0, s>>>(topk_idx, (int)T, M, k, p.chunk_counts);
    const size_t scan_smem = static_cast<size_t>(nchunks) * M * sizeof(int32_t);
    if (scan_smem > 16 * 1024)
        cudaFuncSetAttribute(route_scan_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(scan_smem));
    const int scan_threads = std::max(64, (6 * M + 31) / 32 * 32);  // one per (GEMM, expert)
    route_scan_k<<<1, scan_threads, scan_smem, s>>>(
        p.chunk_counts, nchunks, (int)T, M, k, p.counts, p.pad_off,
                                  p.lb_coeff, p.groups, p.tiles, gb);
    cudaMemsetAsync(p.row_token, 0xFF, sizeof(int32_t) * R_cap, s);
    cudaMemsetAsync(p.row_w, 0, sizeof(float) * R_cap, s);
    route_scatter_k<<<nchunks, ROUTE_CH, 0, s>>>(topk_idx, topk_w, (int)T, M, k, p.chunk_counts,
                                                 p.pad_off, p.slot_row, p.row_token, p.row_w);
    count_launch(3);
}

// ============================ dispatch (permute) ============================
// Xp[slot_row[t][s]] = normed_bf[t] for every token t and selected slot s (model.hpp:314-318,
// 327: select_rows by the expert-major, token-ascending plan), as a scatter of whole rows
// staged by TMA bulk copies: one bulk load of the token's 2d-byte row into shared memory,
// then k bulk stores of it to its routed rows. A warp drives one token at a time from its
// elected lane with two row buffers (the next token's load is in flight while the current
// one is stored). Padding rows of every expert (row_token < 0) are written as zeros by the
// whole warp afterwards. Deterministic: every Xp row has exactly one writer.
constexpr int PERM_WARPS = 4;
__global__ void __launch_bounds__(32 * PERM_WARPS) permute_tma_k(
    const bf16* __restrict__ src, uint32_t row_bytes, const int32_t* __restrict__ slot_row,
    const int32_t* __restrict__ row_token, const int32_t* __restrict__ nrows_dev, int T, int k,
    bf16* __restrict__ xp) {
    extern __shared__ __align__(128) uint8_t psm[];
    __shared__ __align__(8) uint64_t bars[PERM_WARPS][2];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* buf0 = psm + static_cast<size_t>(w) * 2 * row_bytes;
    const int gw = blockIdx.x * PERM_WARPS + w, nw = gridDim.x * PERM_WARPS;
    if (lane == 0) {
        mbar_init(&bars[w][0], 1);
        mbar_init(&bars[w][1], 1);
        fence_barrier_init();
    }
    __syncwarp();
    if (lane == 0 && gw < T) {
        uint32_t phase[2] = {0, 0};
        mbar_arrive_expect_tx(&bars[w][0], row_bytes);
        bulk_load(buf0, reinterpret_cast<const uint8_t*>(src) + static_cast<size_t>(gw) * row_bytes,
                  row_bytes, &bars[w][0]);
        int it = 0;
        for (int t = gw; t < T; t += nw, ++it) {
            const int b = it & 1;
            const int tn = t + nw;
            if (tn < T) {  // next token into the other buffer once its stores have read it
                bulk_wait_read<0>();
                mbar_arrive_expect_tx(&bars[w][b ^ 1], row_bytes);
                bulk_load(buf0 + (b ^ 1) * row_bytes,
                          reinterpret_cast<const uint8_t*>(src) + static_cast<size_t>(tn) * row_bytes,
                          row_bytes, &bars[w][b ^ 1]);
            }
            mbar_wait(&bars[w][b], phase[b]);
            phase[b] ^= 1;
            for (int s = 0; s < k; ++s) {
                const int64_t r = slot_row[static_cast<int64_t>(t) * k + s];
                bulk_store(reinterpret_cast<uint8_t*>(xp) + r * row_bytes, buf0 + b * row_bytes,
                           row_bytes);
            }
            bulk_commit();
        }
        bulk_wait<0>();
    }
    // padding rows (the tail of every expert's tile-aligned range) as zeros
    const int64_t nrows = *nrows_dev;
    const int n16 = static_cast<int>(row_bytes / 16);
    for (int64_t r = gw; r < nrows; r += nw) {
        if (row_token[r] >= 0) continue;
        uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(xp) + r * row_bytes);
        for (int i = lane; i < n16; i += 32) d4[i] = make_uint4(0, 0, 0, 0);
    }
}

void permute_rows_tma(const bf16* src, int64_t cols, const int32_t* slot_row,
                      const int32_t* row_token, const int32_t* nrows_dev, int64_t T, int k,
                      bf16* dst, cudaStream_t s) {
    const uint32_t row_bytes = static_cast<uint32_t>(cols * sizeof(bf16));
    const int smem = PERM_WARPS * 2 * static_cast<int>(row_bytes);
    static std::atomic<uint64_t> attr{0};
    if (first_use_on_device(attr))
        cudaFuncSetAttribute(permute_tma_k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PERM_WARPS * 2 * 8192 * 2);
    const int per_sm = std::max(1, std::min(8, (200 * 1024) / std::max(smem, 1)));
    const int blocks = static_cast<int>(std::min<int64_t>(148 * per_sm, cdiv(T, PERM_WARPS)));
    permute_tma_k<<<std::max(blocks, 1), 32 * PERM_WARPS, smem, s>>>(
        src, row_bytes, slot_row, row_token, nrows_dev, static_cast<int>(T), k, dst);
    count_launch();
}

// ============================ combine (forward) ============================
// h_next[t] = h[t] + sum over selected experts in ascending order of (0 + w*y)
// (model.hpp:330-338: rowwise_mul, scatter_rows into zeros, add chain, residual add)
// Block per token; each thread owns CF_U float4 columns (all their loads in flight first).
constexpr int CF_U = 2;
template <int KMAX>
__global__ void combine_fwd_k(const float* __restrict__ h, const int32_t* __restrict__ hrow,
                              const float* __restrict__ y,
                              const int32_t* __restrict__ slot_row, const float* __restrict__ w,
                              int64_t d, int k, float* __restrict__ h_next,
                              bf16* __restrict__ h_next_bf) {
    const int64_t t = blockIdx.x;
    const float* hr = h + (hrow ? static_cast<int64_t>(hrow[t]) : t) * d;
    int32_t rows[KMAX];
    float ws[KMAX];
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
        rows[s] = s < k ? slot_row[t * k + s] : 0;
        ws[s] = s < k ? w[t * k + s] : 0.f;
    }
    const int64_t step = static_cast<int64_t>(blockDim.x) * 4;
    for (int64_t q0 = threadIdx.x * 4; q0 < d; q0 += step * CF_U) {
        float4 yv[CF_U][KMAX], hv[CF_U];
#pragma unroll
        for (int u = 0; u < CF_U; ++u) {
            const int64_t q = q0 + u * step;
            if (q < d) {
#pragma unroll
                for (int s = 0; s < KMAX; ++s)
                    if (s < k) yv[u][s] = __ldg(reinterpret_cast<const float4*>(y + rows[s] * d + q));
                hv[u] = __ldg(reinterpret_cast<const float4*>(hr + q));
            }
        }
#pragma unroll
        for (int u = 0; u < CF_U; ++u) {
            const int64_t q = q0 + u * step;
            if (q >= d) continue;
            float4 acc;
            acc.x = fadd(0.f, fmul(yv[u][0].x, ws[0]));
            acc.y = fadd(0.f, fmul(yv[u][0].y, ws[0]));
            acc.z = fadd(0.f, fmul(yv[u][0].z, ws[0]));
            acc.w = fadd(0.f, fmul(yv[u][0].w, ws[0]));
#pragma unroll
            for (int s = 1; s < KMAX; ++s) {
                if (s >= k) break;
                acc.x = fadd(acc.x, fadd(0.f, fmul(yv[u][s].x, ws[s])));
                acc.y = fadd(acc.y, fadd(0.f, fmul(yv[u][s].y, ws[s])));
                acc.z = fadd(acc.z, fadd(0.f, fmul(yv[u][s].z, ws[s])));
                acc.w = fadd(acc.w, fadd(0.f, fmul(yv[u][s].w, ws[s])));
            }
            const float4 o = make_float4(fadd(hv[u].x, acc.x), fadd(hv[u].y, acc.y),
                                         fadd(hv[u].z, acc.z), fadd(hv[u].w, acc.w));
            if (h_next) *reinterpret_cast<float4*>(h_next + t * d + q) = o;
            if (h_next_bf) {  // last layer: the head GEMM's bf16 operand, no separate pass
                __nv_bfloat162 a = __floats2bfloat162_rn(o.x, o.y), b = __floats2bfloat162_rn(o.z, o.w);
                uint2 pk;
                pk.x = *reinterpret_cast<uint32_t*>(&a);
                pk.y = *reinterpret_cast<uint32_t*>(&b);
                *reinterpret_cast<uint2*>(h_next_bf + t * d + q) = pk;
            }
        }
    }
}

void combine_forward(const float* h, const int32_t* hrow, const float* y, const int32_t* slot_row,
                     const int32_t* topk_idx, const float* topk_w, int64_t T, int64_t d, int k,
                     float* h_next, bf16* h_next_bf, cudaStream_t s) {
    (void)topk_idx;
    const int threads = d >= 4 * 128 * CF_U ? 128 : static_cast<int>(cdiv(d / 4, CF_U));
    if (k <= 2)
        combine_fwd_k<2><<<static_cast<unsigned>(T), threads, 0, s>>>(h, hrow, y, slot_row, topk_w, d, k,
                                                                      h_next, h_next_bf);
    else
        combine_fwd_k<8><<<static_cast<unsigned>(T), threads, 0, s>>>(h, hrow, y, slot_row, topk_w, d, k,
                                                                      h_next, h_next_bf);
    count_launch();
}

// ============================ head: CE + z ============================
// Warp per token. lse, picked (graph.hpp:410-423); d logits following the
// reverse tape: gather_cols then logsumexp backward (graph.hpp:192-204, 274-281).
// Warp per token; the row is read once into registers (HC_MAXJ values per lane) and each
// exponential is evaluated once (V <= 32 * HC_MAXJ; larger V takes the streaming path).
constexpr int HC_MAXJ = 16;
__global__ void head_ce_k(const float* __restrict__ logits, const int32_t* __restrict__ targets,
                          int64_t T, int64_t T_pad, int64_t V, int64_t Vt, float g_s2,
                          float g_ssum, bf16* __restrict__ dlogits, float* __restrict__ diff,
                          float* __restrict__ lse_out) {
    const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= T_pad) return;
    bf16* drow = dlogits + t * V;  // the head backward GEMMs' bf16 operand, written directly
    if (t >= T) {
        for (int64_t j = lane; j < V; j += 32) drow[j] = __float2bfloat16_rn(0.f);
        return;
    }
    const float* row = logits + t * V;
    // CUDA's full-precision expf: the logits come from a bf16 tensor-core GEMM, so the loss
    // is a tolerance quantity and the glibc-exact exp (router path) buys nothing here
    auto ex = [](float z) { return expf(z); };
    const int32_t tgt = targets[t];
    if (V <= 32 * HC_MAXJ) {
        float x[HC_MAXJ];
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < HC_MAXJ; ++u) {
            const int64_t j = lane + 32 * u;
            x[u] = j < Vt ? row[j] : -INFINITY;
            mx = fmaxf(mx, x[u]);
        }
        mx = warp_max(mx);
        float sum = 0.f;
#pragma unroll
        for (int u = 0; u < HC_MAXJ; ++u) {
            const int64_t j = lane + 32 * u;
            x[u] = j < Vt ? ex(fsub(x[u], mx)) : 0.f;
            sum += x[u];
        }
        sum = warp_sum(sum);
        const float lse = mx + logf(sum);
        if (lane == 0) {
            diff[t] = lse + row[tgt] * -1.f;
            lse_out[t] = lse;
        }
        // lse.grad = (0 + g_s2*lse) + g_s2*lse + g_ssum (z-loss mul, then ce add)
        const float glse = fadd(fadd(fadd(0.f, fmul(g_s2, lse)), fmul(g_s2, lse)), g_ssum);
        const float isum = 1.f / sum;
#pragma unroll
        for (int u = 0; u < HC_MAXJ; ++u) {
            const int64_t j = lane + 32 * u;
            if (j < Vt) {
                const float base = (j == tgt) ? -1.f * g_ssum : 0.f;
                drow[j] = __float2bfloat16_rn(fadd(base, fmul(glse, x[u] * isum)));
            } else if (j < V) {
                drow[j] = __float2bfloat16_rn(0.f);
            }
        }
        return;
    }
    float mx = -INFINITY;
    for (int64_t j = lane; j < Vt; j += 32) mx = fmaxf(mx, row[j]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int64_t j = lane; j < Vt; j += 32) sum += ex(fsub(row[j], mx));
    sum = warp_sum(sum);
    const float lse = mx + logf(sum);
    const float picked = row[tgt];
    if (lane == 0) {
        diff[t] = lse + picked * -1.f;
        lse_out[t] = lse;
    }
    const float glse = fadd(fadd(fadd(0.f, fmul(g_s2, lse)), fmul(g_s2, lse)), g_ssum);
    const float isum = 1.f / sum;
    for (int64_t j = lane; j < V; j += 32) {
        if (j >= Vt) {
            drow[j] = __float2bfloat16_rn(0.f);
            continue;
        }
        const float p = ex(fsub(row[j], mx)) * isum;
        const float base = (j == tgt) ? -1.f * g_ssum : 0.f;
        drow[j] = __float2bfloat16_rn(fadd(base, fmul(glse, p)));
    }
}

void head_ce(const float* logits, const int32_t* targets, int64_t T, int64_t T_pad, int64_t V,
             int64_t Vt, float g_s2, float g_ssum, bf16* dlogits, float* diff, float* lse,
             cudaStream_t s) {
    const int64_t threads = T_pad * 32;
    head_ce_k<<<static_cast<unsigned>(cdiv(threads, 256)), 256, 0, s>>>(
        logits, targets, T, T_pad, V, Vt, g_s2, g_ssum, dlogits, diff, lse);
    count_launch();
}

// ============================ loss scalars ============================
__device__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
    return r;  // valid in thread 0
}

// Per-block partial sums (thread per token, fixed-order tree), then one block
// combines the partials in block order: deterministic, tolerance-level vs the
// reference's sequential fp32 sums. Slots: 0 ce terms, 1 lse_head^2, then per
// layer (lse_router^2, sum_j p_j*coeff_j).
__global__ void __launch_bounds__(256) losses_partial_k(
    const float* __restrict__ diff, const float* __restrict__ lse_head,
    const float* __restrict__ lse_r, const float* __restrict__ probs,
    const float* __restrict__ lb_coeff, int64_t T, int64_t Tstride, int L, int M,
    double* __restrict__ part) {
    __shared__ double sh[32];
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool v = t < T;
    const int ns = 2 + 2 * L;
    double a = v ? static_cast<double>(diff[t]) : 0.0;
    double b = v ? static_cast<double>(lse_head[t]) * lse_head[t] : 0.0;
    a = block_sum_d(a, sh);
    if (threadIdx.x == 0) part[static_cast<int64_t>(blockIdx.x) * ns + 0] = a;
    b = block_sum_d(b, sh);
    if (threadIdx.x == 0) part[static_cast<int64_t>(blockIdx.x) * ns + 1] = b;
    for (int l = 0; l < L; ++l) {
        double c = 0, e = 0;
        if (v) {
            const float lv = lse_r[static_cast<int64_t>(l) * Tstride + t];
            c = static_cast<double>(lv) * lv;
            const float* pr = probs + (static_cast<int64_t>(l) * Tstride + t) * M;
            for (int j = 0; j < M; ++j) e += static_cast<double>(pr[j]) * lb_coeff[l * M + j];
        }
        c = block_sum_d(c, sh);
        if (threadIdx.x == 0) part[static_cast<int64_t>(blockIdx.x) * ns + 2 + 2 * l] = c;
        e = block_sum_d(e, sh);
        if (threadIdx.x == 0) part[static_cast<int64_t>(blockIdx.x) * ns + 3 + 2 * l] = e;
    }
}

__global__ void losses_finish_k(const double* __restrict__ part, int nb, int L, float inv_T,
                                float inv_L, float c_ce, float c_lb, float c_mz, float c_z,
                                int32_t* status, double* __restrict__ out) {
    __shared__ double acc[2 + 2 * 64];
    const int ns = 2 + 2 * L;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        double s = 0.0;
        int b = 0;
        for (; b + 16 <= nb; b += 16) {  // 16 loads in flight, summed in order
            double v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = part[static_cast<int64_t>(b + u) * ns + i];
#pragma unroll
            for (int u = 0; u < 16; ++u) s += v[u];
        }
        for (; b < nb; ++b) s += part[static_cast<int64_t>(b) * ns + i];
        acc[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mz = 0, lb = 0;
        for (int l = 0; l < L; ++l) {
            mz += static_cast<float>(acc[2 + 2 * l]) * inv_T;
            lb += static_cast<float>(acc[3 + 2 * l]);
        }
        const float ce = static_cast<float>(acc[0]) * inv_T;
        const float z = static_cast<float>(acc[1]) * inv_T;
        const float moe_z = static_cast<float>(mz) * inv_L;
        const float lbv = static_cast<float>(lb) * inv_L;
        const float total = (ce * c_ce + lbv * c_lb) + (moe_z * c_mz + z * c_z);
        out[0] = total;
        out[1] = ce;
        out[2] = lbv;
        out[3] = moe_z;
        out[4] = z;
        // status word (see loss_ok): the token check of this or an unreported earlier step
        // (status bit 0, set by the token split) and this step's loss
        int32_t st = *status;
        if (!isfinite(total)) st |= 2;
        if (st) atomicOr(status, st);
        out[5] = static_cast<double>(st);
    }
}

void losses_reduce(const float* diff, const float* lse_head, const float* lse_r,
                   const float* probs, const float* lb_coeff, int64_t T, int64_t Tstride, int L,
                   int M, float inv_T, float inv_L, float c_ce, float c_lb, float c_mz, float c_z,
                   int32_t* status, double* part, double* out, cudaStream_t s) {
    const int nb = static_cast<int>(cdiv(T, 256));
    losses_partial_k<<<nb, 256, 0, s>>>(diff, lse_head, lse_r, probs, lb_coeff, T, Tstride, L, M,
                                        part);
    losses_finish_k<<<1, 128, 0, s>>>(part, nb, L, inv_T, inv_L, c_ce, c_lb, c_mz, c_z,
                                      status, out);
    count_launch(2);
}

// ============================ combine (backward) ============================
// Warp per routed row r (token t_r, weight w_r): dYw[r] = bf16(gh[t_r] * w_r)
// (rowwise_mul backward, graph.hpp:299-305) and the gate-weight gradient
// <gh[t_r], Y[r]> (graph.hpp:307-316). Padding rows get zeros.
// A warp per routed row. With slot_row, warps take the (token, slot) pairs in token order,
// so the k rows of a token run side by side in one block and its upstream-gradient row is
// read from DRAM once (expert-major row order re-read it k times once T x d exceeds L2:
// cfg5 read 4.2 GB per layer for 2.4 GB of operands); blocks past the pairs zero the
// padding rows.
__global__ void __launch_bounds__(256) combine_bwd_k(
    const float* __restrict__ gh, const float* __restrict__ y, const int32_t* __restrict__ row_token,
    const float* __restrict__ row_w, const int32_t* __restrict__ R_total, int64_t d,
    bf16* __restrict__ dyw, float* __restrict__ gw, const int32_t* __restrict__ slot_row,
    int64_t npairs) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    int64_t r = i;
    if (slot_row) {
        if (i < npairs) {
            r = slot_row[i];
        } else {  // padding rows, a grid-stride over the rows
            const int64_t nrows = *R_total;
            const int64_t nw = static_cast<int64_t>(gridDim.x) * 8 - npairs;
            for (int64_t q = i - npairs; q < nrows; q += nw) {
                if (row_token[q] >= 0) continue;
                for (int64_t c = lane * 4; c < d; c += 128)
                    *reinterpret_cast<uint2*>(dyw + q * d + c) = make_uint2(0, 0);
                if (lane == 0) gw[q] = 0.f;
            }
            return;
        }
    } else if (r >= *R_total) {
        return;
    }
    const int32_t t = row_token[r];
    const float wv = t >= 0 ? row_w[r] : 0.f;
    float dot = 0.f;
    constexpr int CB_U = 4;  // column groups per pass, loads first
    for (int64_t q0 = lane * 4; q0 < d; q0 += 128 * CB_U) {
        float4 g[CB_U], yv[CB_U];
#pragma unroll
        for (int u = 0; u < CB_U; ++u) {
            const int64_t q = q0 + 128 * u;
            g[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            yv[u] = g[u];
            if (t >= 0 && q < d) {
                g[u] = __ldg(reinterpret_cast<const float4*>(gh + static_cast<int64_t>(t) * d + q));
                yv[u] = __ldg(reinterpret_cast<const float4*>(y + r * d + q));
            }
        }
#pragma unroll
        for (int u = 0; u < CB_U; ++u) {
            const int64_t q = q0 + 128 * u;
            if (q >= d) break;
            __nv_bfloat162 p0 = __floats2bfloat162_rn(g[u].x * wv, g[u].y * wv);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(g[u].z * wv, g[u].w * wv);
            uint2 pk;
            pk.x = *reinterpret_cast<uint32_t*>(&p0);
            pk.y = *reinterpret_cast<uint32_t*>(&p1);
            *reinterpret_cast<uint2*>(dyw + r * d + q) = pk;
            dot += ((g[u].x * yv[u].x + g[u].y * yv[u].y) + g[u].z * yv[u].z) + g[u].w * yv[u].w;
        }
    }
    dot = warp_sum(dot);
    if (lane == 0) gw[r] = dot;
}

void combine_backward(const float* gh, const float* y, const int32_t* row_token,
                      const float* row_w, const int32_t* R_total_dev, int64_t R_cap, int64_t d,
                      bf16* dyw, float* gw, cudaStream_t s, const int32_t* slot_row,
                      const float* topk_w, int64_t T, int k) {
    (void)topk_w;
    const int64_t npairs = slot_row ? T * k : 0;
    const int64_t blocks = slot_row ? cdiv(npairs, 8) + 148 : cdiv(R_cap, 8);
    combine_bwd_k<<<static_cast<unsigned>(blocks), 256, 0, s>>>(gh, y, row_token, row_w,
                                                                R_total_dev, d, dyw, gw, slot_row,
                                                                npairs);
    count_launch();
}

// ============================ norm-gain and router weight gradients ============================
// g_gain[q] = sum_t (gy*x)*inv ; g_router[q][e] = sum_t normed[t][q]*glog[t][e]
// Fixed-order partials over TC token chunks, then a fixed-order sum.
// grid (d/128, NRG_TC, ceil(M/16)), 256 threads: warp ph takes tokens t = ph (mod 8) of
// the chunk, lane tx the columns 4tx..4tx+3 of the 128-column slab (float4 streams);
// each thread keeps 4 columns x 16 experts of router-gradient partials in registers.
constexpr int NRG_TC = kNormRouterChunks;
constexpr int NG_QT_RMS = 128;  // columns per normed_grad tile = dot partials per token (d / 128)
// With `gh` non-null the z = 0 blocks also apply the rmsnorm backward to their columns
// (kernels.hpp:130-152; the dot from normed_grad's slab partials, summed in slab order):
// h.grad += (gy*g)*inv - coef*x, so h and gnormed
// are streamed once for both.
// Operand streaming: each thread prefetches its own tokens' x / gnormed / gh float4s through a
// per-thread cp.async ring (NRG_S stages: a token's three rows are one commit group), so the
// loads of the next NRG_S - 1 tokens are in flight while this one is processed; the 64-token
// batch's glog, dot partials and inv_rms are staged one batch ahead (4-byte cp.async, double
// buffered). Only the issuing thread reads a ring slot, so the ring needs no barrier; the
// batch staging needs one per batch. Arithmetic and its order are those of the plain loop.
constexpr int NRG_S = 4;
constexpr int NRG_NP_SMEM = 32;  // dot partials per token staged in smem (d <= 4096)
__device__ __forceinline__ void cp_async16_nr(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async4_nr(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_nr() { asm volatile("cp.async.commit_group;" ::: "memory"); }

template <int NRG_EG>
__global__ void __launch_bounds__(256) norm_router_partial_k(
    const float* __restrict__ h, const int32_t* __restrict__ hrow,
    const float* __restrict__ gain, const float* __restrict__ gnormed,
    const float* __restrict__ glog, const float* __restrict__ inv_rms, int T, int d, int dn, int M,
    float* __restrict__ partial, const float* __restrict__ dot_part, float* __restrict__ gh) {
    extern __shared__ __align__(16) float4 ring[];  // [NRG_S][3][256]
    // glog and dot-partial staging during the token loop; the final warp reduction reuses
    // the same bytes (static shared memory stays under 48 KB at 32 experts per block)
    constexpr int SGL = 2 * 64 * NRG_EG, SDOT = 2 * 64 * NRG_NP_SMEM, RED = 32 * 4 * (NRG_EG + 1);
    constexpr int RAW = (SGL + SDOT) > RED ? SGL + SDOT : RED;
    __shared__ __align__(16) float sraw[RAW];
    __shared__ float sinv[2][64];
    float(*sgl)[64][NRG_EG] = reinterpret_cast<float(*)[64][NRG_EG]>(sraw);
    float(*sdot)[64 * NRG_NP_SMEM] = reinterpret_cast<float(*)[64 * NRG_NP_SMEM]>(sraw + SGL);
    float(*red)[4][NRG_EG + 1] = reinterpret_cast<float(*)[4][NRG_EG + 1]>(sraw);
    const int ph = threadIdx.x >> 5, tx = threadIdx.x & 31;
    const int q = blockIdx.x * 128 + 4 * tx;
    const int chunk = blockIdx.y;
    const int e0 = blockIdx.z * NRG_EG;
    const int ne = min(NRG_EG, M - e0);
    const bool do_gain = blockIdx.z == 0;
    const bool do_rms = gh != nullptr && do_gain;
    const int np = d / NG_QT_RMS;
    const bool dot_smem = np <= NRG_NP_SMEM;
    const int per = (T + NRG_TC - 1) / NRG_TC;
    const int t0 = chunk * per, t1 = min(T, t0 + per);
    const int nbatch = t1 > t0 ? (t1 - t0 + 63) / 64 : 0;
    const int nseq = nbatch * 8;  // this thread's token slots: batch s/8, token ph + 8*(s%8)
    float gg[4] = {0.f, 0.f, 0.f, 0.f};
    float gr[4][NRG_EG];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < NRG_EG; ++e) gr[j][e] = 0.f;
    const float4 gq = __ldg(reinterpret_cast<const float4*>(gain + q));

    auto slot_token = [&](int s) { return t0 + 64 * (s >> 3) + ph + 8 * (s & 7); };
    // h row of slot s (the embedding row when layer 0 reads it in place)
    auto slot_row = [&](int s) {
        const int t = slot_token(s);
        return (hrow && s < nseq && t < t1) ? __ldg(hrow + t) : t;
    };
    auto issue = [&](int s, int xr) {
        if (s < nseq) {
            const int t = slot_token(s);
            if (t < t1) {
                float4* st = ring + (s % NRG_S) * 3 * 256;
                const int64_t o = static_cast<int64_t>(t) * d + q;
                const int64_t xo = static_cast<int64_t>(xr) * d + q;
                cp_async16_nr(st + threadIdx.x, h + xo);
                if (do_gain) cp_async16_nr(st + 256 + threadIdx.x, gnormed + o);
                if (do_rms) cp_async16_nr(st + 512 + threadIdx.x, gh + o);
            }
        }
        cp_async_commit_nr();
    };
    auto stage_batch = [&](int b) {  // glog / inv_rms / dot partials of batch b
        if (b >= nbatch) return;
        const int tb = t0 + 64 * b, buf = b & 1;
        for (int i = threadIdx.x; ne > 0 && i < 64 * NRG_EG; i += blockDim.x) {
            const int tt = i / NRG_EG, e = i % NRG_EG;
            if (tb + tt < t1 && e < ne)
                cp_async4_nr(&sgl[buf][tt][e], glog + static_cast<int64_t>(tb + tt) * M + e0 + e);
            else
                sgl[buf][tt][e] = 0.f;
        }
        if (threadIdx.x < 64 && tb + threadIdx.x < t1) cp_async4_nr(&sinv[buf][threadIdx.x], inv_rms + tb + threadIdx.x);
        if (do_rms && dot_smem)
            for (int i = threadIdx.x; i < 64 * np; i += blockDim.x)
                if (tb + i / np < t1)
                    cp_async4_nr(&sdot[buf][i], dot_part + static_cast<int64_t>(tb) * np + i);
    };

    stage_batch(0);
    cp_async_commit_nr();
#pragma unroll
    for (int s = 0; s < NRG_S - 1; ++s) issue(s, slot_row(s));
    int xr_next = slot_row(NRG_S - 1);  // row index loaded one slot ahead of its issue
    for (int b = 0; b < nbatch; ++b) {
        // batch b's staging went out with slot 8b - 8 + NRG_S - 1 (batch 0's is the first
        // group); all but the newest NRG_S - 1 groups complete covers it
        asm volatile("cp.async.wait_group %0;" ::"n"(NRG_S - 1) : "memory");
        __syncthreads();
        stage_batch(b + 1);  // buffer (b+1)&1 was last read in batch b - 1
        const int buf = b & 1;
        const int tb = t0 + 64 * b;
        // lane l < 8 forms the rmsnorm coefficient of this warp's token ph + 8l; the token
        // loop picks it up by shuffle
        float lane_coef = 0.f;
        if (do_rms && tx < 8 && tb + ph + 8 * tx < t1) {
            const int tt = ph + 8 * tx;
            float dot2 = 0.f;
            if (dot_smem)
                for (int i = 0; i < np; ++i) dot2 += sdot[buf][tt * np + i];
            else
                for (int i = 0; i < np; ++i) dot2 += dot_part[static_cast<int64_t>(tb + tt) * np + i];
            const float iv = sinv[buf][tt];
            lane_coef = fdiv(fmul(fmul(fmul(dot2, iv), iv), iv), static_cast<float>(dn));
        }
#pragma unroll 1
        for (int j = 0; j < 8; ++j) {
            const int s = 8 * b + j;
            issue(s + NRG_S - 1, xr_next);  // batch b+1's staging rides in the j == 0 group
            xr_next = slot_row(s + NRG_S);
            asm volatile("cp.async.wait_group %0;" ::"n"(NRG_S - 1) : "memory");
            const int tt = ph + 8 * j;
            if (tb + tt >= t1) continue;
            const float4* st = ring + (s % NRG_S) * 3 * 256;
            const float4 xv = st[threadIdx.x];
            const float iv = sinv[buf][tt];
            // normed exactly as the forward formed it: (x * inv) * g
            float4 nv;
            nv.x = fmul(fmul(xv.x, iv), gq.x);
            nv.y = fmul(fmul(xv.y, iv), gq.y);
            nv.z = fmul(fmul(xv.z, iv), gq.z);
            nv.w = fmul(fmul(xv.w, iv), gq.w);
            if (do_gain) {
                const float4 gv = st[256 + threadIdx.x];
                if (do_rms) {  // rmsnorm backward (kernels.hpp:130-152)
                    const float coef = __shfl_sync(0xffffffffu, lane_coef, j);
                    float4 ov = st[512 + threadIdx.x];
                    ov.x = fadd(ov.x, fsub(fmul(fmul(gv.x, gq.x), iv), fmul(coef, xv.x)));
                    ov.y = fadd(ov.y, fsub(fmul(fmul(gv.y, gq.y), iv), fmul(coef, xv.y)));
                    ov.z = fadd(ov.z, fsub(fmul(fmul(gv.z, gq.z), iv), fmul(coef, xv.z)));
                    ov.w = fadd(ov.w, fsub(fmul(fmul(gv.w, gq.w), iv), fmul(coef, xv.w)));
                    *reinterpret_cast<float4*>(gh + static_cast<int64_t>(tb + tt) * d + q) = ov;
                }
                gg[0] += (gv.x * xv.x) * iv;
                gg[1] += (gv.y * xv.y) * iv;
                gg[2] += (gv.z * xv.z) * iv;
                gg[3] += (gv.w * xv.w) * iv;
            }
            if (ne <= 0) continue;  // gain / rmsnorm only (router gradient on the tensor cores)
            const float n[4] = {nv.x, nv.y, nv.z, nv.w};
#pragma unroll
            for (int e4 = 0; e4 < NRG_EG; e4 += 4) {
                const float4 g4 = *reinterpret_cast<const float4*>(&sgl[buf][tt][e4]);
                const float g[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int u = 0; u < 4; ++u) gr[jj][e4 + u] += n[jj] * g[u];
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // the staging bytes become the reduction buffer
    // combine the 8 warps in warp order (fixed), then write this chunk's partial
    for (int w = 0; w < 8; ++w) {
        __syncthreads();
        if (ph == w) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                red[tx][j][0] = (w == 0 ? 0.f : red[tx][j][0]) + gg[j];
#pragma unroll
                for (int e = 0; e < NRG_EG; ++e)
                    red[tx][j][1 + e] = (w == 0 ? 0.f : red[tx][j][1 + e]) + gr[j][e];
            }
        }
    }
    __syncthreads();
    if (ph == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float* outp = partial + (static_cast<int64_t>(chunk) * d + q + j) * (M + 1);
            if (do_gain) outp[0] = red[tx][j][0];
            for (int e = 0; e < ne; ++e) outp[1 + e0 + e] = red[tx][j][1 + e];
        }
    }
}

__global__ void norm_router_finish_k(const float* __restrict__ partial, int d, int M,
                                     float* __restrict__ g_gain, float* __restrict__ g_router) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(d) * (M + 1)) return;
    const int q = static_cast<int>(i / (M + 1)), c = static_cast<int>(i % (M + 1));
    float v[NRG_TC];  // all chunk partials in flight, then summed in chunk order
#pragma unroll
    for (int ch = 0; ch < NRG_TC; ++ch) v[ch] = partial[(static_cast<int64_t>(ch) * d + q) * (M + 1) + c];
    float s = 0.f;
#pragma unroll
    for (int ch = 0; ch < NRG_TC; ++ch) s += v[ch];
    if (c == 0)
        g_gain[q] = s;
    else
        g_router[static_cast<int64_t>(q) * M + (c - 1)] = s;
}

// 32 experts per block (SPES_NRG_WIDE=1) measured slower at cfg5 (225 vs 177 ms per round:
// 184 registers, one block per SM), so 16 is the default
static const int g_nrg_wide = [] {
    const char* e = std::getenv("SPES_NRG_WIDE");
    return e ? std::atoi(e) : 0;
}();
void norm_router_grads(const float* h, const int32_t* hrow, const float* gain, const float* gnormed,
                       const float* glog, const float* inv_rms, int64_t T, int64_t d, int64_t dn,
                       int M, float* partial, float* g_gain, float* g_router, const float* dot_part,
                       float* gh, cudaStream_t s) {
    // 32 experts per block for M > 16: h streamed and normed rebuilt M/32 times, not M/16
    const int eg = (M > 16 && g_nrg_wide) ? 32 : 16;
    dim3 grid(static_cast<unsigned>(d / 128), NRG_TC,
              static_cast<unsigned>(M > 0 ? (M + eg - 1) / eg : 1));
    constexpr int ring_bytes = NRG_S * 3 * 256 * 16;
    static std::atomic<uint64_t> attr_set{0};
    if (first_use_on_device(attr_set)) {
        cudaFuncSetAttribute(norm_router_partial_k<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ring_bytes);
        cudaFuncSetAttribute(norm_router_partial_k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ring_bytes);
    }
    auto kern = eg == 32 ? norm_router_partial_k<32> : norm_router_partial_k<16>;
    kern<<<grid, 256, ring_bytes, s>>>(h, hrow, gain, gnormed, glog, inv_rms, (int)T, (int)d,
                                       (int)dn, M, partial, dot_part, gh);
    const int64_t n = d * (M + 1);
    norm_router_finish_k<<<static_cast<unsigned>(cdiv(n, 256)), 256, 0, s>>>(partial, (int)d, M,
                                                                            g_gain, g_router);
    count_launch(2);
}

// ============================ embedding gradient ============================
// g_emb[v] = sum over t ascending with inputs[t] == v of gh0[t] (graph.hpp:220-229):
// one block per (vocab id, 1024-column slab); the token list is compacted in
// order, the sum per column is sequential => bit-exact given identical gh0.
__global__ void __launch_bounds__(256) embed_grad_k(const int32_t* __restrict__ inputs,
                                                    const float* __restrict__ gh0, int64_t T,
                                                    int64_t d, float* __restrict__ g_emb) {
    __shared__ int32_t list[256];
    __shared__ int32_t wcount[8];
    const int v = blockIdx.x;
    const int64_t q = static_cast<int64_t>(blockIdx.y) * 1024 + threadIdx.x * 4;
    const bool active = q < d;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t base = 0; base < T; base += 256) {
        const int64_t t = base + threadIdx.x;
        const bool hit = t < T && inputs[t] == v;
        const uint32_t m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) wcount[warp] = __popc(m);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w = 0; w < 8; ++w) {
            if (w < warp) off += wcount[w];
            tot += wcount[w];
        }
        if (hit) list[off + __popc(m & lanemask_lt())] = static_cast<int32_t>(t);
        __syncthreads();
        if (active)
            for (int i = 0; i < tot; ++i) {
                const float4 g = __ldg(reinterpret_cast<const float4*>(gh0 + static_cast<int64_t>(list[i]) * d + q));
                acc.x = fadd(acc.x, g.x);
                acc.y = fadd(acc.y, g.y);
                acc.z = fadd(acc.z, g.z);
                acc.w = fadd(acc.w, g.w);
            }
        __syncthreads();
    }
    if (active) *reinterpret_cast<float4*>(g_emb + static_cast<int64_t>(v) * d + q) = acc;
}

// Fast path (V <= EG_MAXV): stable bucketing of the token positions by vocabulary id
// (histogram -> exclusive scan -> per-id ballot compaction in token order), then one
// thread per (id, 4 columns) sums its bucket's rows in ascending token order with the
// row loads batched in flight. Same per-column sequential order as embed_grad_k.
constexpr int EG_MAXV = 1024;

__global__ void vocab_hist_k(const int32_t* __restrict__ inputs, int64_t T,
                             int32_t* __restrict__ cnt) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < T) atomicAdd(&cnt[inputs[t]], 1);
}

__global__ void __launch_bounds__(EG_MAXV) vocab_scan_k(const int32_t* __restrict__ cnt, int V,
                                                        int32_t* __restrict__ off) {
    __shared__ int32_t sc[EG_MAXV];
    const int v = threadIdx.x;
    sc[v] = v < V ? cnt[v] : 0;
    __syncthreads();
    for (int o = 1; o < EG_MAXV; o <<= 1) {  // Hillis-Steele inclusive scan
        const int32_t x = v >= o ? sc[v - o] : 0;
        __syncthreads();
        sc[v] += x;
        __syncthreads();
    }
    if (v < V) off[v + 1] = sc[v];
    if (v == 0) off[0] = 0;
}

// block per vocabulary id; each pass covers 2048 tokens (8 contiguous per thread, so the
// per-thread order and the thread order are both ascending => stable)
__global__ void __launch_bounds__(256) vocab_bucket_k(const int32_t* __restrict__ inputs,
                                                      int64_t T, const int32_t* __restrict__ off,
                                                      int32_t* __restrict__ list) {
    __shared__ int32_t wsum[8];
    const int v = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int32_t base = off[v];
    for (int64_t b0 = 0; b0 < T; b0 += 2048) {
        const int64_t t0 = b0 + 8 * threadIdx.x;
        int32_t tok[8];
        if (t0 + 8 <= T) {
            const int4 x = __ldg(reinterpret_cast<const int4*>(inputs + t0));
            const int4 y = __ldg(reinterpret_cast<const int4*>(inputs + t0 + 4));
            tok[0] = x.x; tok[1] = x.y; tok[2] = x.z; tok[3] = x.w;
            tok[4] = y.x; tok[5] = y.y; tok[6] = y.z; tok[7] = y.w;
        } else {
#pragma unroll
            for (int u = 0; u < 8; ++u) tok[u] = t0 + u < T ? __ldg(inputs + t0 + u) : -1;
        }
        int h = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) h += tok[u] == v;
        int incl = h;  // inclusive warp scan of the hit counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int pre = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            pre += w < warp ? wsum[w] : 0;
            tot += wsum[w];
        }
        int pos = base + pre + incl - h;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (tok[u] == v) list[pos++] = static_cast<int32_t>(t0 + u);
        base += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(64) embed_grad_sum_k(const int32_t* __restrict__ off,
                                                       const int32_t* __restrict__ list,
                                                       const float* __restrict__ gh0, int64_t d,
                                                       float* __restrict__ g_emb) {
    // this id's token list staged in smem once (coalesced), then EU rows in flight per pass
    constexpr int LCAP = 1024, EU = 16;
    __shared__ int32_t sl[LCAP];
    const int v = blockIdx.x;
    const int64_t q = (static_cast<int64_t>(blockIdx.y) * 64 + threadIdx.x) * 4;
    const int32_t i0 = off[v], i1 = off[v + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int32_t c0 = i0; c0 < i1; c0 += LCAP) {
        const int32_t c1 = min(i1, c0 + LCAP);
        __syncthreads();
        for (int32_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) sl[i - c0] = list[i];
        __syncthreads();
        if (q >= d) continue;
        int32_t i = c0;
        for (; i + EU <= c1; i += EU) {
            float4 g[EU];
#pragma unroll
            for (int u = 0; u < EU; ++u)
                g[u] = __ldg(reinterpret_cast<const float4*>(gh0 + static_cast<int64_t>(sl[i - c0 + u]) * d + q));
#pragma unroll
            for (int u = 0; u < EU; ++u) {
                acc.x = fadd(acc.x, g[u].x);
                acc.y = fadd(acc.y, g[u].y);
                acc.z = fadd(acc.z, g[u].z);
                acc.w = fadd(acc.w, g[u].w);
            }
        }
        for (; i < c1; ++i) {
            const float4 g = __ldg(reinterpret_cast<const float4*>(gh0 + static_cast<int64_t>(sl[i - c0]) * d + q));
            acc.x = fadd(acc.x, g.x);
            acc.y = fadd(acc.y, g.y);
            acc.z = fadd(acc.z, g.z);
            acc.w = fadd(acc.w, g.w);
        }
    }
    if (q < d) *reinterpret_cast<float4*>(g_emb + static_cast<int64_t>(v) * d + q) = acc;
}

bool embed_grad_plan(const int32_t* inputs, int64_t T, int64_t V, int32_t* scratch,
                     cudaStream_t s) {
    if (!(V <= EG_MAXV && scratch)) return false;
    int32_t* cnt = scratch;               // [V]
    int32_t* off = scratch + V;           // [V + 1]
    int32_t* list = scratch + 2 * V + 1;  // [T]
    cudaMemsetAsync(cnt, 0, sizeof(int32_t) * V, s);
    vocab_hist_k<<<static_cast<unsigned>(cdiv(T, 256)), 256, 0, s>>>(inputs, T, cnt);
    vocab_scan_k<<<1, EG_MAXV, 0, s>>>(cnt, static_cast<int>(V), off);
    vocab_bucket_k<<<static_cast<unsigned>(V), 256, 0, s>>>(inputs, T, off, list);
    count_launch(3);
    return true;
}

void embed_grad_apply(const int32_t* inputs, const float* gh0, int64_t T, int64_t d, int64_t V,
                      float* g_emb, int32_t* scratch, cudaStream_t s) {
    if (V <= EG_MAXV && scratch) {  // planned by embed_grad_plan
        dim3 grid(static_cast<unsigned>(V), static_cast<unsigned>(cdiv(d, 256)));
        embed_grad_sum_k<<<grid, 64, 0, s>>>(scratch + V, scratch + 2 * V + 1, gh0, d, g_emb);
        count_launch();
        return;
    }
    dim3 grid(static_cast<unsigned>(V), static_cast<unsigned>(cdiv(d, 1024)));
    embed_grad_k<<<grid, 256, 0, s>>>(inputs, gh0, T, d, g_emb);
    count_launch();
}


// ============================ device corpus batches ============================
// batch row b = corpus row rows[b] (S+1 tokens), make_batch (corpus.cpp:81-87)
__global__ void corpus_gather_k(const int32_t* __restrict__ corpus, const int64_t* __restrict__ rows,
                                int64_t S1, int32_t* __restrict__ tokens) {
    const int64_t b = blockIdx.x;
    const int32_t* src = corpus + rows[b] * S1;
    int32_t* dst = tokens + b * S1;
    for (int64_t p = threadIdx.x; p < S1; p += blockDim.x) dst[p] = __ldg(src + p);
}

void corpus_gather(const int32_t* corpus, const int64_t* rows, int64_t B, int64_t S1,
                   int32_t* tokens, cudaStream_t s) {
    corpus_gather_k<<<static_cast<unsigned>(B), 256, 0, s>>>(corpus, rows, S1, tokens);
    count_launch();
}

// ============================ DiLoCo outer step (trainer.hpp:228-266) ============================
// This rank's slice of the global model: theta <- OuterOpt(theta, mean_i(local_i - theta)),
// per element in fp64 with the locals in node order (recv holds N x n, node-major); the
// Nesterov buffer of the slice persists in fp64. Bit-exact with OuterOptimizer::step.
__global__ void __launch_bounds__(256) outer_step_k(float* __restrict__ theta,
                                                    const float* __restrict__ recv, int N,
                                                    int64_t n, int64_t ld, int kind, double lr,
                                                    double momentum, double* __restrict__ buf,
                                                    float* __restrict__ out) {
    const double inv_n = 1.0 / static_cast<double>(N);
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double t = static_cast<double>(theta[j]);
        double delta = 0.0;
        for (int i = 0; i < N; ++i)
            delta = __dadd_rn(delta, __dmul_rn(__dsub_rn(static_cast<double>(recv[i * ld + j]), t), inv_n));
        float nt;
        if (kind == 0) {
            nt = static_cast<float>(__dadd_rn(t, __dmul_rn(lr, delta)));
        } else {
            const double g = -delta;
            const double b = __dadd_rn(__dmul_rn(momentum, buf[j]), g);
            buf[j] = b;
            nt = static_cast<float>(__dsub_rn(t, __dmul_rn(lr, __dadd_rn(g, __dmul_rn(momentum, b)))));
        }
        theta[j] = nt;
        out[j] = nt;
    }
}

void outer_step(float* theta, const float* recv, int N, int64_t n, int64_t ld, int kind, double lr,
                double momentum, double* buf, float* out, cudaStream_t s) {
    if (n <= 0) return;
    const int blocks = static_cast<int>(std::min<int64_t>(cdiv(n, 256), 148 * 8));
    outer_step_k<<<blocks, 256, 0, s>>>(theta, recv, N, n, ld, kind, lr, momentum, buf, out);
    count_launch();
}

// ============================ AdamW (+ bf16 operand copies) ============================
// MaskedAdamW::step element update (trainer.hpp:85-92; or the SGD inner step of
// trainer.hpp:197-204), exact fp32 op order, over the compact trainable segments (psi +
// owned experts). The updated values are also written as the bf16 GEMM operand copies
// (W1 interleaved gate|up, W2 = Wd, headB), so no separate shadow pass re-reads them.
//
// Segment lookup is by block: blockIdx.y picks the segment (a launch covers whole segments,
// or the same piece of consecutive expert segments), so no thread ever searches a table.
__device__ __forceinline__ int seg_of(const SegTable& t, int64_t i) {  // refresh pass only
    if (i >= t.psi_len) return t.npsi + static_cast<int>((i - t.psi_len) / t.per);
    int s = 0;
    while (s + 1 < t.npsi && t.segs[s + 1].comp_off <= i) ++s;
    return s;
}

// 4 consecutive parameters starting at offset o within segment sg -> bf16 copy
__device__ __forceinline__ void write_shadow4(const AdamSeg& sg, int64_t o, const float4& v,
                                              const Shadows& sh) {
    if (sg.kind == 0) return;
    bf16* dst;
    if (sg.kind == 2) {
        dst = sh.headB + o;
    } else {
        // per-expert offsets fit in 32 bits (d*f < 2^31): 32-bit index math
        const uint32_t df = static_cast<uint32_t>(sh.d * sh.f), f = static_cast<uint32_t>(sh.f);
        const uint32_t o32 = static_cast<uint32_t>(o);
        if (o32 < 2 * df) {  // wg / wu: [d x f] -> W1 [d x 2f] interleaved
            const bool up = o32 >= df;
            const uint32_t oo = up ? o32 - df : o32;
            const uint32_t q = (f & (f - 1)) == 0 ? oo >> (__ffs(f) - 1) : oo / f;  // uniform
            const uint32_t x = oo - q * f;
            dst = sh.w1 + static_cast<int64_t>(sg.slot) * 2 * df + static_cast<int64_t>(q) * 2 * f +
                  (up ? il_up(x) : il_gate(x));
        } else {  // wd: [f x d] -> W2 as is
            dst = sh.w2 + static_cast<int64_t>(sg.slot) * df + (o32 - 2 * df);
        }
    }
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&a);
    pk.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(dst) = pk;
}

// Each thread owns ADAM_U float4 groups of a tile (all loads in flight before any update);
// segment lengths are multiples of 4.
// Block (x, y): segment seg0 + y, its piece [off, off + len) (len < 0: to the segment's
// end), in chunks of tpb tiles of blockDim.x * U float4 groups: chunks x, x + gridDim.x, ...
// The standalone pass launches one chunk per block, so consecutive blocks stream each
// segment front to back (DRAM-page friendly); the background pass launches a few blocks
// per SM that walk their piece (so they never hold more registers than a resident GEMM
// CTA leaves free, and keep more bytes in flight per thread with U = 4).
template <int U>
__global__ void __launch_bounds__(256) adamw_k(float* __restrict__ params,
                                               const float* __restrict__ grads,
                                               float* __restrict__ m, float* __restrict__ v,
                                               const AdamSeg* __restrict__ segs, int seg0,
                                               int64_t off, int64_t len, int tpb,
                                               const AdamScalars* __restrict__ ap,
                                               Shadows sh, const double* __restrict__ loss_total) {
    if (!loss_ok(loss_total)) return;
    const AdamScalars a = *ap;
    const AdamSeg sg = segs[seg0 + blockIdx.y];
    const int64_t plen = len < 0 ? sg.len - off : len;
    const int64_t n4 = plen / 4;
    float* th_base = params + sg.param_off + off;  // piece element e: th_base[e], comp[e]
    const int64_t comp = sg.comp_off + off;
    const float* gb = grads + comp;
    float* mb = m + comp;
    float* vb = v + comp;
    const int nt = blockDim.x, tile4 = nt * U;
    const int64_t chunk4 = static_cast<int64_t>(tpb) * tile4;
    for (int64_t first = static_cast<int64_t>(blockIdx.x) * chunk4; first < n4;
         first += static_cast<int64_t>(gridDim.x) * chunk4) {
        const int64_t last = min(n4, first + chunk4);
        for (int64_t t0 = first; t0 < last; t0 += tile4) {
            float4 th[U], g[U], mm[U], vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = t0 + u * nt + threadIdx.x;  // coalesced per u
                if (q < last) {
                    th[u] = *reinterpret_cast<const float4*>(th_base + 4 * q);
                    g[u] = __ldcs(reinterpret_cast<const float4*>(gb + 4 * q));
                    if (!a.sgd) {
                        mm[u] = __ldcs(reinterpret_cast<const float4*>(mb + 4 * q));
                        vv[u] = __ldcs(reinterpret_cast<const float4*>(vb + 4 * q));
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t q = t0 + u * nt + threadIdx.x;
                if (q >= last) continue;
                if (a.sgd) {  // theta -= lr * g (trainer.hpp:197-204)
                    th[u].x = fsub(th[u].x, fmul(a.lr, g[u].x));
                    th[u].y = fsub(th[u].y, fmul(a.lr, g[u].y));
                    th[u].z = fsub(th[u].z, fmul(a.lr, g[u].z));
                    th[u].w = fsub(th[u].w, fmul(a.lr, g[u].w));
                } else {
                    th[u].x = adam_elem(th[u].x, g[u].x, mm[u].x, vv[u].x, a);
                    th[u].y = adam_elem(th[u].y, g[u].y, mm[u].y, vv[u].y, a);
                    th[u].z = adam_elem(th[u].z, g[u].z, mm[u].z, vv[u].z, a);
                    th[u].w = adam_elem(th[u].w, g[u].w, mm[u].w, vv[u].w, a);
                    __stcs(reinterpret_cast<float4*>(mb + 4 * q), mm[u]);
                    __stcs(reinterpret_cast<float4*>(vb + 4 * q), vv[u]);
                }
                *reinterpret_cast<float4*>(th_base + 4 * q) = th[u];
                write_shadow4(sg, off + 4 * q, th[u], sh);
            }
        }
    }
}

// Background (side-stream) launch shape: threads per block, tiles per chunk, blocks per SM
// over the whole launch (0: one chunk per block), float4 groups per thread (2 or 4).
// 64 threads (2 warps): fits in the registers a resident GEMM CTA leaves free, so the
// background launches really run beside the GEMMs (cfg5 N=1: 5845 -> 5779 ms per round
// against 256-thread blocks, which only run where no GEMM CTA is resident)
int g_adam_bg_threads = 64, g_adam_bg_tiles = 16, g_adam_bg_per_sm = 0, g_adam_bg_u = 2;
void adamw_background_shape(int threads, int tiles, int per_sm, int u) {
    g_adam_bg_threads = threads;
    g_adam_bg_tiles = tiles;
    g_adam_bg_per_sm = per_sm;
    g_adam_bg_u = u == 4 ? 4 : 2;
}

static void adamw_launch(float* params, const float* grads, float* m, float* v,
                         const AdamSeg* segs, int seg0, int nseg, int64_t off, int64_t len,
                         int64_t max_len, const AdamScalars* a, Shadows sh,
                         const double* loss_total, cudaStream_t s, bool background) {
    if (nseg <= 0 || max_len <= 0) return;
    // 256-thread blocks, one chunk of 8 tiles each; or the background shape above
    const int nt = background ? g_adam_bg_threads : 256;
    const int tpb = background ? g_adam_bg_tiles : 8;
    const int U = background ? g_adam_bg_u : 2;
    const int64_t chunks = cdiv(cdiv(max_len / 4, nt * U), tpb);
    int64_t bx = chunks;
    if (background && g_adam_bg_per_sm > 0)
        bx = std::max<int64_t>(1, std::min<int64_t>(chunks, 148 * g_adam_bg_per_sm / nseg));
    const dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(nseg));
    if (U == 4)
        adamw_k<4><<<grid, nt, 0, s>>>(params, grads, m, v, segs, seg0, off, len, tpb, a, sh,
                                       loss_total);
    else
        adamw_k<2><<<grid, nt, 0, s>>>(params, grads, m, v, segs, seg0, off, len, tpb, a, sh,
                                       loss_total);
    count_launch();
}

void adamw(float* params, const float* grads, float* m, float* v, const SegTable& tab,
           int seg0, int nseg, const AdamScalars* a, Shadows sh, const double* loss_total,
           cudaStream_t s) {
    const int64_t max_len = std::max<int64_t>(tab.per, tab.psi_len);  // bound on a segment
    adamw_launch(params, grads, m, v, tab.segs, seg0, nseg, 0, -1, max_len, a, sh, loss_total, s,
                 false);
}

void adamw_pieces(float* params, const float* grads, float* m, float* v, const SegTable& tab,
                  int seg0, int nseg, int64_t off, int64_t len, const AdamScalars* a, Shadows sh,
                  const double* loss_total, cudaStream_t s) {
    adamw_launch(params, grads, m, v, tab.segs, seg0, nseg, off, len, len, a, sh, loss_total, s,
                 true);
}

__global__ void __launch_bounds__(256) refresh_shadows_k(const float* __restrict__ params,
                                                         SegTable tab, int64_t total4, Shadows sh) {
    for (int64_t i4 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i4 < total4;
         i4 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = i4 * 4;
        const AdamSeg sg = tab.segs[seg_of(tab, i)];
        if (sg.kind == 0) continue;
        const int64_t o = i - sg.comp_off;
        write_shadow4(sg, o, __ldg(reinterpret_cast<const float4*>(params + sg.param_off + o)), sh);
    }
}

void refresh_shadows(const float* params, const SegTable& tab, int64_t total, Shadows sh,
                     cudaStream_t s) {
    const int64_t total4 = total / 4;
    const int blocks = static_cast<int>(std::min<int64_t>(cdiv(total4, 256), 148 * 8));
    refresh_shadows_k<<<blocks, 256, 0, s>>>(params, tab, total4, sh);
    count_launch();
}

// ============================ sync: owner-set mean ============================
// out[i] = float((sum over sources in order of double(x)) * (1.0/n))  (protocol.cpp:238-243)
__global__ void owner_mean_strided_k(const float* __restrict__ x, int n_src, int64_t stride,
                                     int64_t n, float* __restrict__ out) {
    const double inv = 1.0 / static_cast<double>(n_src);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < n_src; ++s) acc = __dadd_rn(acc, static_cast<double>(x[s * stride + i]));
        out[i] = __double2float_rn(__dmul_rn(acc, inv));
    }
}

void owner_mean_strided(const float* x, int n_src, int64_t stride, int64_t n, float* out,
                        cudaStream_t s) {
    const int blocks = static_cast<int>(std::min<int64_t>(cdiv(n, 256), 148 * 16));
    owner_mean_strided_k<<<blocks, 256, 0, s>>>(x, n_src, stride, n, out);
    count_launch();
}

struct SrcList {
    const float* p[16];
};
__global__ void owner_mean_list_k(SrcList L, int n_src, int64_t n, float* __restrict__ out) {
    const double inv = 1.0 / static_cast<double>(n_src);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < n_src; ++s) acc = __dadd_rn(acc, static_cast<double>(L.p[s][i]));
        out[i] = __double2float_rn(__dmul_rn(acc, inv));
    }
}

// float4 columns, every source's load in flight before the fp64 sums (the sources may be
// peer GPUs' memory read over NVLink); same per-element operations as owner_mean_list_k
__global__ void owner_mean_list4_k(SrcList L, int n_src, int64_t n4, float* __restrict__ out,
                                   Shadows sh, int slot) {
    const double inv = 1.0 / static_cast<double>(n_src);
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 v[16];
#pragma unroll
        for (int s = 0; s < 16; ++s)
            if (s < n_src) v[s] = reinterpret_cast<const float4*>(L.p[s])[i];
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
            if (s >= n_src) break;
            a0 = __dadd_rn(a0, static_cast<double>(v[s].x));
            a1 = __dadd_rn(a1, static_cast<double>(v[s].y));
            a2 = __dadd_rn(a2, static_cast<double>(v[s].z));
            a3 = __dadd_rn(a3, static_cast<double>(v[s].w));
        }
        const float4 r =
            make_float4(__double2float_rn(__dmul_rn(a0, inv)), __double2float_rn(__dmul_rn(a1, inv)),
                        __double2float_rn(__dmul_rn(a2, inv)), __double2float_rn(__dmul_rn(a3, inv)));
        reinterpret_cast<float4*>(out)[i] = r;
        if (slot >= 0) {  // the expert's bf16 GEMM operand copy, from the same values
            AdamSeg sg{};
            sg.kind = 1;
            sg.slot = slot;
            write_shadow4(sg, 4 * i, r, sh);
        }
    }
}

void owner_mean(const float* const* srcs, int n_src, int64_t n, float* out, cudaStream_t s,
                const Shadows* sh, int slot) {
    SrcList L{};
    bool aligned = n % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
    for (int i = 0; i < n_src && i < 16; ++i) {
        L.p[i] = srcs[i];
        aligned = aligned && reinterpret_cast<uintptr_t>(srcs[i]) % 16 == 0;
    }
    if (aligned) {
        const int blocks = static_cast<int>(std::min<int64_t>(cdiv(n / 4, 256), 148 * 8));
        owner_mean_list4_k<<<blocks, 256, 0, s>>>(L, n_src, n / 4, out, sh ? *sh : Shadows{},
                                                   sh ? slot : -1);
    } else {
        if (sh) throw std::logic_error("owner_mean: operand refresh needs 16-byte aligned rows");
        const int blocks = static_cast<int>(std::min<int64_t>(cdiv(n, 256), 148 * 16));
        owner_mean_list_k<<<blocks, 256, 0, s>>>(L, n_src, n, out);
    }
    count_launch();
}

// ---- the fused expert exchange of the sparse sync (one persistent kernel) ----
// Tasks are chunks of experts: first every owner-set mean this node is primary for (its
// co-owners' copies read in place over NVLink, fp64 sum in ascending node order,
// protocol.cpp:238-243), then every expert chunk it pulls from that expert's primary. Blocks
// claim tasks from a device counter in that order. When the last mean chunk of a layer is
// done, the node publishes flags[layer] = epoch (release, system scope); a pull chunk of a
// layer first waits until its primary's flag for the layer reaches the epoch (acquire). So a
// layer's pulls overlap the remaining means, here and on every peer, with no host barrier
// between the phases. No deadlock: a block only waits on a pull after every mean task of
// this node has been claimed by a running block, and peers progress independently.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int NS>  // sources per mean, at most
__global__ void __launch_bounds__(256, NS <= 2 ? 3 : 1) sync_exchange_k(const SyncTask* __restrict__ tasks,
                                                       int ntasks, int* __restrict__ ctr,
                                                       const int* __restrict__ layer_total, int L,
                                                       uint32_t* flags, uint32_t* const* peer_flags,
                                                       uint32_t epoch, Shadows sh) {
    __shared__ int s_task;
    if (blockIdx.x == 0 && threadIdx.x < L && layer_total[threadIdx.x] == 0)
        st_release_sys(flags + threadIdx.x, epoch);  // nothing to average in this layer
    for (;;) {
        if (threadIdx.x == 0) s_task = atomicAdd(ctr, 1);
        __syncthreads();
        const int ti = s_task;
        __syncthreads();
        if (ti >= ntasks) break;
        const SyncTask& t = tasks[ti];  // fields read as needed (L1-resident)
        if (t.nsrc == 0) {  // a pull: wait for the primary's means of this layer
            if (threadIdx.x == 0)
                while (ld_acquire_sys(peer_flags[t.primary] + t.layer) < epoch) __nanosleep(256);
            __syncthreads();
            (void)ld_acquire_sys(peer_flags[t.primary] + t.layer);
        }
        AdamSeg sg{};
        sg.kind = 1;
        sg.slot = t.slot;
        const int nsrc = t.nsrc == 0 ? 1 : t.nsrc;
        const double inv = 1.0 / static_cast<double>(nsrc);
        float4* dst = reinterpret_cast<float4*>(t.dst);
        if (t.nsrc == 0) {  // a pull: a plain copy with 8 float4 per thread in flight
            constexpr int PU = 8;
            const float4* src = reinterpret_cast<const float4*>(t.src[0]);
            for (int64_t i0 = threadIdx.x; i0 < t.n4; i0 += PU * blockDim.x) {
                float4 v[PU];
#pragma unroll
                for (int u = 0; u < PU; ++u) {
                    const int64_t i = i0 + u * blockDim.x;
                    if (i < t.n4) v[u] = src[i];
                }
#pragma unroll
                for (int u = 0; u < PU; ++u) {
                    const int64_t i = i0 + u * blockDim.x;
                    if (i < t.n4) {
                        dst[i] = v[u];
                        write_shadow4(sg, t.off + 4 * i, v[u], sh);
                    }
                }
            }
            continue;
        }
        constexpr int XU = 4;  // float4 groups per thread in flight, per source
        for (int64_t i0 = threadIdx.x; i0 < t.n4; i0 += XU * blockDim.x) {
            float4 v[NS][XU];
#pragma unroll
            for (int s2 = 0; s2 < NS; ++s2)
                if (s2 < nsrc)
#pragma unroll
                    for (int u = 0; u < XU; ++u) {
                        const int64_t i = i0 + u * blockDim.x;
                        if (i < t.n4) v[s2][u] = reinterpret_cast<const float4*>(t.src[s2])[i];
                    }
#pragma unroll
            for (int u = 0; u < XU; ++u) {
                const int64_t i = i0 + u * blockDim.x;
                if (i >= t.n4) break;
                float4 r = v[0][u];
                if (t.nsrc > 0) {  // owner-set mean, nodes ascending (a unique owner: copy)
                    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
                    for (int s2 = 0; s2 < NS; ++s2) {
                        if (s2 >= nsrc) break;
                        a0 = __dadd_rn(a0, static_cast<double>(v[s2][u].x));
                        a1 = __dadd_rn(a1, static_cast<double>(v[s2][u].y));
                        a2 = __dadd_rn(a2, static_cast<double>(v[s2][u].z));
                        a3 = __dadd_rn(a3, static_cast<double>(v[s2][u].w));
                    }
                    r = make_float4(__double2float_rn(__dmul_rn(a0, inv)),
                                    __double2float_rn(__dmul_rn(a1, inv)),
                                    __double2float_rn(__dmul_rn(a2, inv)),
                                    __double2float_rn(__dmul_rn(a3, inv)));
                }
                dst[i] = r;
                write_shadow4(sg, t.off + 4 * i, r, sh);
            }
        }
        if (t.nsrc > 0) {  // mean chunk done: the layer's flag once all its chunks are
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(ctr + 1 + t.layer, 1) + 1 == layer_total[t.layer]) {
                    __threadfence_system();
                    st_release_sys(flags + t.layer, epoch);
                }
            }
        }
    }
}

void sync_exchange(const SyncTask* tasks, int ntasks, int max_src, int* ctr,
                   const int* layer_total, int L, uint32_t* flags, uint32_t* const* peer_flags,
                   uint32_t epoch, Shadows sh, cudaStream_t s) {
    cudaMemsetAsync(ctr, 0, sizeof(int) * (1 + L), s);
    if (max_src <= 2)
        sync_exchange_k<2><<<148 * 3, 256, 0, s>>>(tasks, ntasks, ctr, layer_total, L, flags,
                                                   peer_flags, epoch, sh);
    else
        sync_exchange_k<SYNC_MAX_SRC><<<148 * 2, 256, 0, s>>>(tasks, ntasks, ctr, layer_total, L,
                                                              flags, peer_flags, epoch, sh);
    count_launch();
}


// ============================ merge: Gram + apply ============================
// Projection vector of expert j: D1 floats at vec_offs[j] (+ a second D1 run at
// +gap when two_parts: Concat source). Partial fp64 dot products per chunk.
// Gram partials: block = a contiguous element range; per tile of SUB elements the M
// vectors are staged in smem by float4 loads, then work items (pair, part) accumulate
// their share in fp64, several items per thread (independent chains). A block's partial of
// a pair = its parts summed in part order. Fixed grouping -> deterministic; vs the
// reference's sequential sum ~1e-12 relative (select_peers re-checks near-ties exactly).
constexpr int GRAM_ITEMS = 9;  // work items per thread (2080 pairs at M = 64)
__host__ __device__ inline int gram_sub(int M) { return 16384 / M; }  // tile: <= 64 KB smem
__host__ __device__ inline int gram_parts(int npairs) {
    int P = 1;
    while (npairs * P * 2 <= 768 && P < 16) P *= 2;
    return P;
}

__global__ void __launch_bounds__(256) gram_partial_k(const float* __restrict__ params,
                                                      const int64_t* __restrict__ vec_offs, int M,
                                                      int64_t D1, int64_t gap, int two_parts,
                                                      double* __restrict__ partial, int nchunks) {
    extern __shared__ __align__(16) float sv[];  // [M][sub], then [npairs * P] doubles
    const int sub = gram_sub(M), q4 = sub / 4;
    const int npairs = M * (M + 1) / 2, P = gram_parts(npairs), seg = sub / P;
    double* sitem = reinterpret_cast<double*>(sv + static_cast<int64_t>(M) * sub);
    const int64_t D = two_parts ? 2 * D1 : D1;
    const int64_t per = ((D + nchunks - 1) / nchunks + sub - 1) / sub * sub;
    const int64_t e0 = static_cast<int64_t>(blockIdx.x) * per, e1 = min(D, e0 + per);
    const int nitems = npairs * P;
    double acc[GRAM_ITEMS];
    int pa[GRAM_ITEMS], pb[GRAM_ITEMS], pp[GRAM_ITEMS];
#pragma unroll
    for (int u = 0; u < GRAM_ITEMS; ++u) {
        acc[u] = 0.0;
        const int item = threadIdx.x + u * 256;
        const int pidx = item / P;
        int a = 0, rem = pidx;
        if (item < nitems)
            while (rem >= M - a) {
                rem -= M - a;
                ++a;
            }
        pa[u] = a;
        pb[u] = a + rem;
        pp[u] = item % P;
    }
    for (int64_t b = e0; b < e1; b += sub) {
        __syncthreads();
        for (int i = threadIdx.x; i < M * q4; i += blockDim.x) {
            const int j = i / q4;
            const int64_t e = b + 4 * (i % q4);  // D1 and every bound are multiples of 4
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < e1) {
                const int64_t src = (two_parts && e >= D1) ? vec_offs[j] + gap + (e - D1) : vec_offs[j] + e;
                v = __ldg(reinterpret_cast<const float4*>(params + src));
            }
            reinterpret_cast<float4*>(sv + static_cast<int64_t>(j) * sub)[i % q4] = v;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < GRAM_ITEMS; ++u) {
            if (threadIdx.x + u * 256 < nitems) {
                const float* va = sv + pa[u] * sub + pp[u] * seg;
                const float* vb = sv + pb[u] * sub + pp[u] * seg;
                double s2 = acc[u];
                for (int i = 0; i < seg; ++i) s2 += static_cast<double>(va[i]) * vb[i];
                acc[u] = s2;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < GRAM_ITEMS; ++u)
        if (threadIdx.x + u * 256 < nitems) sitem[threadIdx.x + u * 256] = acc[u];
    __syncthreads();
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < P; ++q) t += sitem[p * P + q];
        partial[static_cast<int64_t>(blockIdx.x) * npairs + p] = t;
    }
}

// M <= 16 (rows padded to 16 with zeros): the 16 x 16 Gram as ten upper-triangle 4 x 4
// register tiles, warp w owning tiles w and w + 8; lane l takes elements l, l+32, ... of each
// staged tile (conflict-free LDS: all lanes on the same rows), 8 loads feed 16 fp64 FMAs;
// the lanes' sums meet in a fixed butterfly at the end. Deterministic.
constexpr int GRAM_SMALL_SUB = 1024;
__device__ __forceinline__ int gram_pair_index(int M, int a, int b) {  // a <= b
    int idx = 0;
    for (int i = 0; i < a; ++i) idx += M - i;
    return idx + (b - a);
}
__global__ void __launch_bounds__(256) gram_small_k(const float* __restrict__ params,
                                                    const int64_t* __restrict__ vec_offs, int M,
                                                    int64_t D1, int64_t gap, int two_parts,
                                                    double* __restrict__ partial, int nchunks) {
    extern __shared__ __align__(16) float sv[];  // [16][GRAM_SMALL_SUB]
    constexpr int SUB = GRAM_SMALL_SUB, Q4 = SUB / 4;
    const int npairs = M * (M + 1) / 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t D = two_parts ? 2 * D1 : D1;
    const int64_t per = ((D + nchunks - 1) / nchunks + SUB - 1) / SUB * SUB;
    const int64_t e0 = static_cast<int64_t>(blockIdx.x) * per, e1 = min(D, e0 + per);
    int bi[2] = {0, 0}, bj[2] = {0, 0}, nt = 0;
    for (int k = 0; k < 2; ++k) {
        int t = warp + 8 * k;
        if (t >= 10) break;
        int r = 0;
        while (t >= 4 - r) {
            t -= 4 - r;
            ++r;
        }
        bi[nt] = r;
        bj[nt] = r + t;
        ++nt;
    }
    double acc[2][4][4];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[k][r][c] = 0.0;
    for (int64_t b = e0; b < e1; b += SUB) {
        __syncthreads();
        for (int i = threadIdx.x; i < 16 * Q4; i += blockDim.x) {
            const int j = i / Q4;
            const int64_t e = b + 4 * (i % Q4);
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (j < M && e < e1) {
                const int64_t src = (two_parts && e >= D1) ? vec_offs[j] + gap + (e - D1) : vec_offs[j] + e;
                v = __ldg(reinterpret_cast<const float4*>(params + src));
            }
            reinterpret_cast<float4*>(sv + j * SUB)[i % Q4] = v;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            if (k >= nt) break;
            const float* ra = sv + 4 * bi[k] * SUB;
            const float* rb = sv + 4 * bj[k] * SUB;
            for (int i = lane; i < SUB; i += 32) {
                float xa[4], xb[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    xa[r] = ra[r * SUB + i];
                    xb[r] = rb[r * SUB + i];
                }
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        acc[k][r][c] += static_cast<double>(xa[r]) * static_cast<double>(xb[c]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (k >= nt) break;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const double t = warp_sum_d(acc[k][r][c]);
                const int a = 4 * bi[k] + r, bb = 4 * bj[k] + c;
                if (lane == 0 && a <= bb && bb < M)
                    partial[static_cast<int64_t>(blockIdx.x) * npairs + gram_pair_index(M, a, bb)] = t;
            }
    }
}

void gram_partials(const float* params, const int64_t* vec_offs, int M, int64_t D1, int64_t gap,
                   int two_parts, double* partial, int nchunks, cudaStream_t s) {
    const int npairs = M * (M + 1) / 2;
    if (M <= 16) {
        const size_t smem = sizeof(float) * 16 * GRAM_SMALL_SUB;
        cudaFuncSetAttribute(gram_small_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        gram_small_k<<<nchunks, 256, smem, s>>>(params, vec_offs, M, D1, gap, two_parts, partial,
                                               nchunks);
        count_launch();
        return;
    }
    const size_t smem = sizeof(float) * M * gram_sub(M) + sizeof(double) * npairs * gram_parts(npairs);
    cudaFuncSetAttribute(gram_partial_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gram_partial_k<<<nchunks, 256, smem, s>>>(params, vec_offs, M, D1, gap, two_parts, partial,
                                             nchunks);
    count_launch();
}

// sim[a][b] = dot/(norm_a*norm_b) (merging.hpp:55-82); zero norm -> 0. One warp per pair:
// the block partials of the pair and of both diagonals, lane-strided then a butterfly
// (fixed order, identical bits on every lane).
__global__ void gram_finish_k(const double* __restrict__ partial, int M, int nchunks,
                              double* __restrict__ sim) {
    const int npairs = M * (M + 1) / 2;
    const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (p >= npairs) return;
    int a = 0, rem = p;
    while (rem >= M - a) {
        rem -= M - a;
        ++a;
    }
    const int b = a + rem;
    auto diag_idx = [&](int j) {
        int idx = 0;
        for (int i = 0; i < j; ++i) idx += M - i;
        return idx;
    };
    const int da = diag_idx(a), db = diag_idx(b);
    double sp = 0.0, sa = 0.0, sb = 0.0;
    for (int c = lane; c < nchunks; c += 32) {
        const double* row = partial + static_cast<int64_t>(c) * npairs;
        sp += row[p];
        sa += row[da];
        sb += row[db];
    }
    sp = warp_sum_d(sp);
    sa = warp_sum_d(sa);
    sb = warp_sum_d(sb);
    if (lane == 0) {
        const double na = sqrt(sa), nb = sqrt(sb);
        double v = 0.0;
        if (na > 0.0 && nb > 0.0) v = sp / (na * nb);
        sim[a * M + b] = v;
        sim[b * M + a] = v;
    }
}

void gram_finish(const double* partial, int M, int nchunks, double* sim, cudaStream_t s) {
    const int npairs = M * (M + 1) / 2;
    gram_finish_k<<<static_cast<unsigned>((npairs + 7) / 8), 256, 0, s>>>(partial, M, nchunks, sim);
    count_launch();
}

// merge_experts (merging.hpp:97-136): w_j += coef_j * sum_q (w_peer_q - w_j), all experts
// from the same pre-merge snapshot, in fp64. Each thread snapshots element i of every expert
// into its own smem column (peers are data-dependent indices), converted to double once:
// 2 elements per thread for M <= 16 (double2 columns), else 1.
// VEC (1 or 2) consecutive parameters at offset o (even for VEC = 2) of expert slot `slot`
// -> its bf16 operand copy (a pair never straddles a 128-column block of W1)
template <int VEC>
__device__ __forceinline__ void write_shadow_n(int slot, int64_t o, const float* v,
                                               const Shadows& sh) {
    const uint32_t df = static_cast<uint32_t>(sh.d * sh.f), f = static_cast<uint32_t>(sh.f);
    const uint32_t o32 = static_cast<uint32_t>(o);
    bf16* dst;
    if (o32 < 2 * df) {
        const bool up = o32 >= df;
        const uint32_t oo = up ? o32 - df : o32;
        const uint32_t q = (f & (f - 1)) == 0 ? oo >> (__ffs(f) - 1) : oo / f;
        const uint32_t x = oo - q * f;
        dst = sh.w1 + static_cast<int64_t>(slot) * 2 * df + static_cast<int64_t>(q) * 2 * f +
              (up ? il_up(x) : il_gate(x));
    } else {
        dst = sh.w2 + static_cast<int64_t>(slot) * df + (o32 - 2 * df);
    }
    if (VEC == 2)
        *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(v[0], v[1]);
    else
        *dst = __float2bfloat16_rn(v[0]);
}

template <int VEC>
__global__ void __launch_bounds__(256) merge_apply_k(float* __restrict__ params,
                                                     const int64_t* __restrict__ expert_offs,
                                                     int M, int64_t per,
                                                     const int32_t* __restrict__ peers, int K,
                                                     const double* __restrict__ coef,
                                                     double* __restrict__ disp_partial, Shadows sh,
                                                     int slot0) {
    using F = typename std::conditional<VEC == 2, float2, float>::type;
    __shared__ int32_t sp[64 * 64];
    __shared__ double sc[64];
    __shared__ int64_t so[64];
    __shared__ double red[256];
    extern __shared__ __align__(16) double snap[];  // [M][256][VEC]
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) sp[i] = peers[i];
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
        sc[i] = coef[i];
        so[i] = expert_offs[i];
    }
    __syncthreads();
    double disp = 0.0;
    const int tid = threadIdx.x;
    const int64_t nv = per / VEC;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid; i < nv;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        constexpr int JU = VEC == 2 ? 16 : 8;  // loads in flight per batch
        for (int j0 = 0; j0 < M; j0 += JU) {
            F x[JU];
#pragma unroll
            for (int u = 0; u < JU; ++u)
                if (j0 + u < M) x[u] = *reinterpret_cast<const F*>(params + so[j0 + u] + i * VEC);
#pragma unroll
            for (int u = 0; u < JU; ++u) {
                if (j0 + u >= M) break;
                const float* xf = reinterpret_cast<const float*>(&x[u]);
#pragma unroll
                for (int c = 0; c < VEC; ++c)
                    snap[((j0 + u) * 256 + tid) * VEC + c] = static_cast<double>(xf[c]);
            }
        }
        for (int j = 0; j < M; ++j) {
            float outv[VEC];
#pragma unroll
            for (int c = 0; c < VEC; ++c) {
                const double self = snap[(j * 256 + tid) * VEC + c];
                double acc = 0.0;
                for (int q = 0; q < K; ++q)
                    acc = __dadd_rn(acc, __dsub_rn(snap[(sp[j * K + q] * 256 + tid) * VEC + c], self));
                const double delta = __dmul_rn(sc[j], acc);
                disp += delta * delta;
                outv[c] = __double2float_rn(__dadd_rn(self, delta));
            }
            *reinterpret_cast<F*>(params + so[j] + i * VEC) = *reinterpret_cast<const F*>(outv);
            if (slot0 >= 0) write_shadow_n<VEC>(slot0 + j, i * VEC, outv, sh);
        }
    }
    red[tid] = disp;
    __syncthreads();
    if (tid == 0) {
        double s2 = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) s2 += red[i];
        disp_partial[blockIdx.x] = s2;
    }
}

// M <= 16, K <= 8: two elements per thread as double2 snapshot columns, the peers' column
// offsets precomputed per block, the peer loop unrolled (same fp64 operations and order)
__global__ void __launch_bounds__(256) merge_apply_small_k(float* __restrict__ params,
                                                           const int64_t* __restrict__ expert_offs,
                                                           int M, int64_t per,
                                                           const int32_t* __restrict__ peers, int K,
                                                           const double* __restrict__ coef,
                                                           double* __restrict__ disp_partial,
                                                           Shadows sh, int slot0) {
    __shared__ int32_t spo[16 * 8];  // peer column offset (peer * 256)
    __shared__ double sc[16];
    __shared__ int64_t so[16];
    __shared__ double red[256];
    extern __shared__ __align__(16) double2 snap2[];  // [M][256]
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) spo[(i / K) * 8 + i % K] = peers[i] * 256;
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
        sc[i] = coef[i];
        so[i] = expert_offs[i];
    }
    __syncthreads();
    double disp = 0.0;
    const int tid = threadIdx.x;
    const int64_t nv = per / 2;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid; i < nv;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float2 x[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < M) x[j] = *reinterpret_cast<const float2*>(params + so[j] + 2 * i);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < M) snap2[j * 256 + tid] = make_double2(x[j].x, x[j].y);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (j >= M) break;
            const double2 self = snap2[j * 256 + tid];
            double ax = 0.0, ay = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q >= K) break;
                const double2 pv = snap2[spo[j * 8 + q] + tid];
                ax = __dadd_rn(ax, __dsub_rn(pv.x, self.x));
                ay = __dadd_rn(ay, __dsub_rn(pv.y, self.y));
            }
            const double dx = __dmul_rn(sc[j], ax), dy = __dmul_rn(sc[j], ay);
            disp += dx * dx;
            disp += dy * dy;
            const float outv[2] = {__double2float_rn(__dadd_rn(self.x, dx)),
                                   __double2float_rn(__dadd_rn(self.y, dy))};
            *reinterpret_cast<float2*>(params + so[j] + 2 * i) = make_float2(outv[0], outv[1]);
            if (slot0 >= 0) write_shadow_n<2>(slot0 + j, 2 * i, outv, sh);
        }
    }
    red[tid] = disp;
    __syncthreads();
    if (tid == 0) {
        double s2 = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) s2 += red[i];
        disp_partial[blockIdx.x] = s2;
    }
}

void merge_apply(float* params, const int64_t* expert_offs, int M, int64_t per,
                 const int32_t* peers, int K, const double* coef, double* disp_partial,
                 int nblocks, cudaStream_t s, const Shadows* sh, int slot0) {
    const Shadows shv = sh ? *sh : Shadows{};
    if (!sh) slot0 = -1;
    if (M <= 16 && K <= 8 && per % 2 == 0) {
        const size_t smem = sizeof(double2) * M * 256;
        cudaFuncSetAttribute(merge_apply_small_k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        merge_apply_small_k<<<nblocks, 256, smem, s>>>(params, expert_offs, M, per, peers, K, coef,
                                                       disp_partial, shv, slot0);
    } else if (M <= 16 && per % 2 == 0) {
        const size_t smem = sizeof(double) * 2 * M * 256;
        cudaFuncSetAttribute(merge_apply_k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        merge_apply_k<2><<<nblocks, 256, smem, s>>>(params, expert_offs, M, per, peers, K, coef,
                                                     disp_partial, shv, slot0);
    } else {
        const size_t smem = sizeof(double) * M * 256;
        cudaFuncSetAttribute(merge_apply_k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        merge_apply_k<1><<<nblocks, 256, smem, s>>>(params, expert_offs, M, per, peers, K, coef,
                                                     disp_partial, shv, slot0);
    }
    count_launch();
}

// ============================ split-K combine ============================
__global__ void splitk_reduce_k(const float4* __restrict__ part, int nsplit, int64_t n4,
                                float4* __restrict__ out) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float4 a = __ldg(part + i);
        int s = 1;
        for (; s + 8 <= nsplit; s += 8) {  // 8 loads in flight, added in split order
            float4 b[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) b[u] = __ldg(part + (s + u) * n4 + i);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                a.x += b[u].x;
                a.y += b[u].y;
                a.z += b[u].z;
                a.w += b[u].w;
            }
        }
        for (; s < nsplit; ++s) {
            const float4 b = __ldg(part + s * n4 + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        out[i] = a;
    }
}

__global__ void router_grad_reduce_k(const float* __restrict__ part, int nsplit, int64_t d, int M,
                                     float* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= d * M) return;
    const int64_t q = i / M, e = i % M;
    float a = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) a += __ldg(part + (sp * d + q) * 128 + e);
    out[i] = a;
}

void router_grad_reduce(const float* part, int nsplit, int64_t d, int M, float* out,
                        cudaStream_t s) {
    router_grad_reduce_k<<<static_cast<unsigned>(cdiv(d * M, 256)), 256, 0, s>>>(part, nsplit, d,
                                                                                M, out);
    count_launch();
}

void splitk_reduce(const float* part, int nsplit, int64_t n, float* out, cudaStream_t s) {
    const int64_t n4 = n / 4;
    const int blocks = static_cast<int>(std::min<int64_t>(cdiv(n4, 256), 148 * 8));
    splitk_reduce_k<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(part), nsplit, n4,
                                           reinterpret_cast<float4*>(out));
    count_launch();
}

// ============================ expf port probe ============================
__global__ void expf_port_k(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                            int variant) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        y[i] = variant ? spes_expf::expf_glibc<1>(x[i]) : spes_expf::expf_glibc<0>(x[i]);
}

void expf_port_device(const float* x, float* y, int64_t n, int variant, cudaStream_t s) {
    expf_port_k<<<148 * 16, 256, 0, s>>>(x, y, n, variant);
    count_launch();
}

}  // namespace spes_k

// Host-side launchers of the SPES device kernels (kernels.cu, gemm.cu).
// All launches go to the given stream; nothing here synchronizes.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "common.cuh"
#include "grouped_gemm.cuh"

namespace spes_k {

using bf16 = __nv_bfloat16;
using spes_dev::GemmGroup;

// Counts every kernel launch (for the bench's gpu_launches claim).
extern thread_local int64_t* g_launch_counter;
inline void count_launch(int n = 1) {
    if (g_launch_counter) *g_launch_counter += n;
}

// cudaFuncSetAttribute applies to the current device only: one bit per device records
// where a kernel's attributes are set (contexts on several GPUs may share a process).
inline bool first_use_on_device(std::atomic<uint64_t>& mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    return (mask.fetch_or(bit) & bit) == 0;
}

struct AdamSeg {
    int64_t param_off;  // offset in the fp32 parameter vector
    int64_t comp_off;   // offset in the compact (trainable-only) grad / m / v buffers
    int64_t len;
    int32_t kind;       // bf16 operand copy to refresh: 0 none, 1 expert (wg|wu|wd), 2 head
    int32_t slot;       // expert slot (layer*M + j) for kind 1
};

// ---- forward ----
void embed_gather(const float* emb, const int32_t* tokens, int64_t B, int64_t S, int64_t d,
                  int64_t V, float* h, int32_t* inputs, int32_t* targets, int32_t* err,
                  cudaStream_t s);
// normed (fp32) and normed_bf (bf16, the expert GEMM operand) are each optional.
// hrow (optional): row t of h is h + hrow[t] * d (layer 0 reads emb[inputs] in place).
// d: row width; dn: the rmsnorm mean's width (the model's hidden size; < d when rows carry
// zero padding)
void router_forward(const float* h, const int32_t* hrow, const float* gain, const float* router,
                    int64_t T, int64_t d, int64_t dn,
                    int M, int k, int renorm, float eps, int expf_variant, float* normed,
                    bf16* normed_bf, float* logits, float* probs, int32_t* topk_idx,
                    float* topk_w, float* lse, float* inv_rms, float* denom, cudaStream_t s);
// Deterministic counting sort of the (token, slot) pairs, expert-major and
// token-ascending (model.hpp:314-318), each expert padded to 128 rows; also
// builds the GEMM group tables of this layer on the device.
struct RoutePlan {
    int32_t* chunk_counts;  // [nchunks][M]
    int32_t* counts;        // [M]
    int32_t* pad_off;       // [M+1]
    float* lb_coeff;        // [M]
    int32_t* slot_row;      // [T][k]
    int32_t* row_token;     // [R_cap]  (-1 = padding)
    float* row_w;           // [R_cap]
    GemmGroup* groups;      // [6][M]: fwd1, fwd2, dH, dX, dW1, dW2
    int32_t* tiles;         // [6] total tiles per GEMM
};
struct GroupBases {  // output bases written into the group tables
    bf16* gu;
    float* y;
    bf16* dgu;
    float* dxp;
    float* grad_expert_base;       // compact grad buffer
    const int64_t* grad_off_layer; // [M]: offset of expert j of this layer in grads, -1 = frozen
    int64_t d, f;
    int bn_fwd2, bn_dh, bn_dx, bn_dw2;
    int tile_rows;  // 128 (1-CTA tiles) or 256 (cta_group::2 pair tiles); also the row padding
    // fused optimizer: dW groups address the parameters (param_expert_base + e*3df),
    // the compact Adam state (grad_off_layer[e]) and shadow slot slot0 + e
    float* param_expert_base;
    int32_t slot0;
    int32_t fused_adam;
};
void route_plan(const int32_t* topk_idx, const float* topk_w, int64_t T, int M, int k,
                int64_t R_cap, const RoutePlan& p, const GroupBases& gb, cudaStream_t s);
// Dispatch: Xp[slot_row[t][s]] = src[t] (bf16 rows of `cols`) by TMA bulk copies (one
// row load, k row stores per token); rows with row_token < 0 among the first *nrows_dev
// are zeroed (cols * 2 bytes must be a multiple of 16 and at most 16 KiB).
void permute_rows_tma(const bf16* src, int64_t cols, const int32_t* slot_row,
                      const int32_t* row_token, const int32_t* nrows_dev, int64_t T, int k,
                      bf16* dst, cudaStream_t s);
// h_next_bf (optional): bf16 copy of h_next (the head GEMM operand after the last layer);
// h_next may then be null (the final fp32 hidden state has no other consumer)
void combine_forward(const float* h, const int32_t* hrow, const float* y, const int32_t* slot_row,
                     const int32_t* topk_idx, const float* topk_w, int64_t T, int64_t d, int k,
                     float* h_next, bf16* h_next_bf, cudaStream_t s);
// CE + z on head logits; writes dlogits as bf16 (the head backward GEMM operand; padding
// rows zero) and the per-token terms.
// V: row width of logits / dlogits; Vt <= V: the model's vocabulary (columns >= Vt are zero
// padding: excluded from the softmax, zero gradient)
void head_ce(const float* logits, const int32_t* targets, int64_t T, int64_t T_pad, int64_t V,
             int64_t Vt, float g_s2, float g_ssum, bf16* dlogits, float* diff,
             float* lse, cudaStream_t s);
// Loss scalars (tolerance-level, deterministic tree order) -> out[0..4] (doubles), and
// the step's status word (sticky in *status, copied to out[5]; see spes_dev::loss_ok)
void losses_reduce(const float* diff, const float* lse_head, const float* lse_r,
                   const float* probs, const float* lb_coeff, int64_t T, int64_t Tstride, int L,
                   int M,
                   float inv_T, float inv_L, float c_ce, float c_lb, float c_mz, float c_z,
                   int32_t* status, double* part, double* out, cudaStream_t s);

// ---- backward ----
// slot_row / topk_w (optional): the token-major form (each token's gradient row read once)
void combine_backward(const float* gh, const float* y, const int32_t* row_token,
                      const float* row_w, const int32_t* R_total_dev, int64_t R_cap, int64_t d,
                      bf16* dyw, float* gw_part, cudaStream_t s, const int32_t* slot_row = nullptr,
                      const float* topk_w = nullptr, int64_t T = 0, int k = 0);
// Router backward in two halves: the per-token scalar chain (-> glog; needs only the
// forward's routing and the gate-weight gradients) and the normed gradient (needs dX; its
// per-slab rmsnorm dot partials go to dot_part for norm_router_grads)
void router_scalar_backward(const float* probs, const float* lse_r, const float* denom,
                            const int32_t* topk_idx, const int32_t* slot_row, const float* gw_row,
                            const float* lb_coeff, int64_t T, int M, int k, int renorm,
                            float g_lbsum, float g_s, float* glog, bf16* glog_bf,
                            cudaStream_t s);
void normed_grad(const float* h, const int32_t* hrow, const float* gain, const float* router,
                 const int32_t* slot_row, const float* dxp, int64_t T, int64_t d, int M, int k,
                 const float* glog, float* gnormed, float* dot_part, cudaStream_t s);
// token chunks of norm_router_grads ((d/128) x 37 blocks = whole waves of 2 per SM); its
// partial buffer holds kNormRouterChunks * d * (M + 1) floats
constexpr int kNormRouterChunks = 37;
// normed is recomputed exactly from h, inv_rms and the gain (not stored in forward)
// gh non-null: also applies the rmsnorm backward (dot from normed_grad's dot_part)
// M = 0: gain gradient and rmsnorm backward only (the router gradient runs on the tensor
// cores, router_grad_reduce)
void norm_router_grads(const float* h, const int32_t* hrow, const float* gain, const float* gnormed,
                       const float* glog, const float* inv_rms, int64_t T, int64_t d, int64_t dn,
                       int M,
                       float* partial, float* g_gain, float* g_router, const float* dot_part,
                       float* gh, cudaStream_t s);
// embedding gradient in two halves: the token bucketing by vocabulary id (needs only the
// inputs; scratch: 2V + 1 + T int32; false => no fast path (V > 1024 or no scratch), and
// embed_grad_apply does everything) and the gradient sums
bool embed_grad_plan(const int32_t* inputs, int64_t T, int64_t V, int32_t* scratch, cudaStream_t s);
void embed_grad_apply(const int32_t* inputs, const float* gh0, int64_t T, int64_t d, int64_t V,
                      float* g_emb, int32_t* scratch, cudaStream_t s);

// ---- optimizer / shadows ----
// bf16 GEMM operand copies written by the optimizer / refresh: W1 [slots][d][2f]
// (gate|up interleaved in 128-column blocks), W2 [slots][f][d] (= Wd), headB [d][V].
struct Shadows {
    bf16* w1;
    bf16* w2;
    bf16* headB;
    int64_t d, f;
};
// out = fp64 mean of the sources in order (the sources may be peer GPUs' memory); with sh,
// also the bf16 operand copy of expert slot `slot` (out is that expert's parameter block)
void owner_mean(const float* const* srcs, int n_src, int64_t n, float* out, cudaStream_t s,
                const Shadows* sh = nullptr, int slot = -1);
// one expert (per floats) from a peer's parameters into ours, plus its bf16 operand copy
// Fused expert exchange of the sparse sync (kernels.cu): owner-set means (nsrc >= 1 sources
// in ascending node order) then pulls from the primaries (nsrc == 0, src[0] = the primary's
// copy), gated per layer by the primaries' flags (flags / peer_flags: one uint32 per layer
// and node, IPC-mapped; epoch increases per sync). ctr: 1 + L ints (reset here).
constexpr int SYNC_MAX_SRC = 8;
struct SyncTask {
    const float* src[SYNC_MAX_SRC];
    float* dst;
    int64_t off;   // element offset of the chunk within its expert (bf16 copy addressing)
    int64_t n4;    // float4 groups in the chunk
    int32_t nsrc;  // owners averaged; 0 = a pull
    int32_t slot;  // expert slot (layer * M + j)
    int32_t layer;
    int32_t primary;
};
void sync_exchange(const SyncTask* tasks, int ntasks, int max_src, int* ctr,
                   const int* layer_total, int L, uint32_t* flags, uint32_t* const* peer_flags,
                   uint32_t epoch, Shadows sh, cudaStream_t s);
// Segment table of the compact optimizer layout: npsi leading segments (psi_len scalars in
// total) followed by expert segments of `per` scalars each.
struct SegTable {
    const AdamSeg* segs;
    int32_t npsi;
    int64_t psi_len, per;
};
// MaskedAdamW (or, a->sgd, SGD) step over the whole segments [seg0, seg0 + nseg) of the
// table; also writes the refreshed bf16 copies. No update while the step status is bad
// (spes_dev::loss_ok; loss_total may be null).
using spes_dev::AdamScalars;
void adamw(float* params, const float* grads, float* m, float* v, const SegTable& tab,
           int seg0, int nseg, const AdamScalars* a, Shadows sh, const double* loss_total,
           cudaStream_t s);
// The piece [off, off + len) of each of the segments [seg0, seg0 + nseg) (multiples of 4), as
// a background launch (short blocks, no smem: fits beside a GEMM CTA)
void adamw_pieces(float* params, const float* grads, float* m, float* v, const SegTable& tab,
                  int seg0, int nseg, int64_t off, int64_t len, const AdamScalars* a, Shadows sh,
                  const double* loss_total, cudaStream_t s);  // a: device memory (graph-replayable)
// shape of the background (adamw_pieces) launches: threads per block, tiles per chunk,
// blocks per SM over the launch (0: one chunk per block), float4 groups per thread (2 / 4)
void adamw_background_shape(int threads, int tiles, int per_sm, int u);
// Rewrite the bf16 copies of refresh-table scalars [0, total) from the fp32 parameters
// (after load / sync / merge).
void refresh_shadows(const float* params, const SegTable& tab, int64_t total, Shadows sh,
                     cudaStream_t s);

// batch tokens B x (S+1) from the HBM-resident corpus rows
void corpus_gather(const int32_t* corpus, const int64_t* rows, int64_t B, int64_t S1,
                   int32_t* tokens, cudaStream_t s);
// device corpus generation (corpus_dev.cu): n uniform doubles from the std::mt19937_64
// state (312 words, next position pos), then one Markov chain per sequence over the
// sources' prefix-sum tables cum [C][V+1][V]
void corpus_draws(const uint64_t* state, int pos, int64_t n, double* out, cudaStream_t s);
void corpus_chains(const double* cum, const double* u, int64_t sequences, int64_t seq, int V,
                   int C, int32_t* tokens, cudaStream_t s);

// ---- sync / merge ----
// DiLoCo outer step over this rank's slice (theta, n scalars): recv = the N nodes' local
// slices (stride ld, node order); kind 0 SGD, 1 Nesterov (buf: fp64 state); the new values
// go to theta and out
void outer_step(float* theta, const float* recv, int N, int64_t n, int64_t ld, int kind, double lr,
                double momentum, double* buf, float* out, cudaStream_t s);
void owner_mean_strided(const float* x, int n_src, int64_t stride, int64_t n, float* out,
                        cudaStream_t s);
void gram_partials(const float* params, const int64_t* vec_offs, int M, int64_t D1,
                   int64_t gap, int two_parts, double* partial, int nchunks, cudaStream_t s);
void gram_finish(const double* partial, int M, int nchunks, double* sim, cudaStream_t s);
void merge_apply(float* params, const int64_t* expert_offs, int M, int64_t per,
                 const int32_t* peers, int K, const double* coef, double* disp_partial,
                 int nblocks, cudaStream_t s, const Shadows* sh = nullptr, int slot0 = -1);

// ---- GEMMs (gemm.cu) ----
void gemm_swiglu(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                 const int32_t* tiles, int max_tiles, bf16* hact, int64_t f, cudaStream_t s);
// operand majors: KK (both K contiguous), KMN (B = row-major weight [K x N]),
// MNMN (weight-gradient form: A [K x M], B [K x N] row-major over K = tokens)
enum class GemmMajor { KK, KMN, MNMN };
void gemm_store_f32(int bn, GemmMajor mj, const CUtensorMap& a, const CUtensorMap& b,
                    const GemmGroup* g, int ng, const int32_t* tiles, int max_tiles,
                    cudaStream_t s);
// dSwiGLU epilogue variant: 0 direct loads; 1 / 2 TMA-staged 64-column pieces through the
// transpose slots with 1 / 2 buffers (needs gu_map: the GU buffer as {64 x 128}-box tensor
// map in device memory); 3 / 4 TMA-staged 32-column pieces written back in place by TMA with
// 2 / 3 buffers (needs inplace_maps: GU as {32 x 128} and dGU as {32 x 32} boxes, 64B
// swizzle, device memory). Pair tiles (BN = 256) only; otherwise the direct epilogue.
void gemm_dswiglu(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, const bf16* gu, int64_t f,
                  const CUtensorMap* gu_map, const CUtensorMap* inplace_maps, int variant,
                  cudaStream_t s);
// head forward (V == 256) with softmax-CE fused into the epilogue: writes bf16 dlogits
// ([T_pad x 256], padding rows zero), the per-token CE term and lse (head_ce semantics)
void gemm_head_ce(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, const int32_t* targets, int64_t T,
                  float g_s2, float g_ssum, bf16* dlog, float* diff, float* lse, cudaStream_t s);
void gemm_grad_w1(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                  const int32_t* tiles, int max_tiles, cudaStream_t s);
// dW GEMMs with MaskedAdamW fused into the epilogue (params, m, v and bf16 shadows are
// updated in place; no gradient is materialized)
struct AdamEpi {
    const AdamScalars* a;  // device memory
    float* m;
    float* v;
    bf16* w1;
    bf16* w2;
    int64_t d, f;
    const double* loss_total;
};
// Tensor maps of one layer's expert parameters and Adam moments for the TMA-staged fused
// optimizer (gemm.cu EpiAdamStaged): the layer's expert region of theta (all M experts) and
// of m / v (its owned experts, compact) viewed as rows of f floats (wg / wu blocks) and of d
// floats (wd blocks), boxes of 32 x 128 fp32 with the 128B swizzle. Device memory.
struct AdamMaps {
    CUtensorMap th_f, m_f, v_f, th_d, m_d, v_d;
    const float* th_base;   // theta of expert 0 of the layer
    int64_t mv_base;        // compact offset of the layer's first owned expert
};
// aw (optional, device memory, one per layer): with it the pair kernel stages theta / m / v
// by TMA and writes them back by TMA stores (EpiAdamStaged)
void gemm_adamw_w1(const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const AdamEpi& p, cudaStream_t s,
                   const AdamMaps* aw = nullptr, int M = 0);
void gemm_adamw_w2(int bn, const CUtensorMap& a, const CUtensorMap& b, const GemmGroup* g, int ng,
                   const int32_t* tiles, int max_tiles, const AdamEpi& p, cudaStream_t s,
                   const AdamMaps* aw = nullptr, int M = 0);
void gemm_prepare(int device);
// cta_group::2 cluster-pair GEMMs (256-row tiles) for the following launches on this thread
void gemm_set_pair_mode(bool on);
int num_sms();

// out[i] = sum over splits in order of part[s*n + i]   (deterministic split-K combine)
void splitk_reduce(const float* part, int nsplit, int64_t n, float* out, cudaStream_t s);
// g_router [d x M] = sum over splits (in order) of part [nsplit][d][128] (columns < M)
void router_grad_reduce(const float* part, int nsplit, int64_t d, int M, float* out,
                        cudaStream_t s);

// expf port checks
void expf_port_device(const float* x, float* y, int64_t n, int variant, cudaStream_t s);

}  // namespace spes_k

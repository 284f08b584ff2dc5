/*
 * spes_oracle.h -- CPU restatement of the SPES hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker: the product (libspes_b200.so) never
 * links or calls it. It restates, in plain C with the reference's exact fp32
 * operation order (no FMA, sequential reductions, glibc expf), the functions of
 * /root/reference/proj that SURVEY.md §8(a) lists; each function cites the
 * reference lines it follows. It is pinned bit-for-bit against the reference
 * itself (oracle/_ref/libspes_ref.so, built from the reference sources by
 * oracle/Makefile) in tests/test_oracle_pinning.py.
 */
#ifndef SPES_ORACLE_H
#define SPES_ORACLE_H

#include <stdint.h>

#include "../include/spes_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Intermediates of one forward/backward (any pointer may be NULL). T = B*S. */
typedef struct {
    float* normed;      /* [L][T][d]   rmsnorm output                          */
    float* logits;      /* [L][T][M]   router logits                           */
    float* probs;       /* [L][T][M]   router softmax                          */
    int32_t* topk_idx;  /* [L][T][k]   selected experts, ascending            */
    float* topk_w;      /* [L][T][k]   gate weights (renormalized if enabled) */
    int32_t* counts;    /* [L][M]      tokens per expert                       */
    int32_t* perm;      /* [L][T*k]    token of each routed row, expert-major  */
    float* h;           /* [L+1][T][d] residual stream into layer l / final   */
    float* head_logits; /* [T][V]                                              */
    float* grad_h;      /* [L+1][T][d] d total / d h_l                         */
} oracle_trace;

int64_t oracle_param_count(const spes_model_cfg* c);
/* offsets of: emb, head, norm[l], router[l], e[l][j].{wg,wu,wd} */
int64_t oracle_off_emb(const spes_model_cfg* c);
int64_t oracle_off_head(const spes_model_cfg* c);
int64_t oracle_off_norm(const spes_model_cfg* c, int l);
int64_t oracle_off_router(const spes_model_cfg* c, int l);
int64_t oracle_off_expert(const spes_model_cfg* c, int l, int j); /* wg; wu = +d*f; wd = +2*d*f */

/* rmsnorm -> router matmul -> softmax -> route_from_logits for T rows. */
void oracle_router_forward(const spes_model_cfg* c, const float* h, const float* gain,
                           const float* router, int64_t T, float* normed, float* logits,
                           float* probs, int32_t* topk_idx, float* topk_w, int32_t* counts,
                           int32_t* perm);

/* build_loss + GraphT::backward for one batch. trainable_expert[M] (shared blocks
 * are always trainable). grads: full parameter layout, zeros on frozen blocks.
 * losses[5] = total, ce, lb, moe_z, z. Returns 0, or 2 on a bad token id. */
int oracle_forward_backward(const spes_model_cfg* c, const float* params, const int32_t* tokens,
                            int64_t B, int64_t S, const uint8_t* trainable_expert, float* grads,
                            double* losses, oracle_trace* trace);

/* MaskedAdamW::step over the trainable blocks; m, v have the full parameter layout. */
void oracle_adamw_step(const spes_model_cfg* c, float* params, const float* grads, float* m,
                       float* v, const uint8_t* trainable_expert, const spes_adamw_cfg* opt,
                       int64_t step);

void oracle_adamw_array(float* theta, const float* g, float* m, float* v, int64_t n,
                        const spes_adamw_cfg* opt, int64_t step);

/* local_round (AdamW, fresh state) over H batches; lr[h] per step; losses[H][5].
 * Returns 0, 2 (bad token), or 3 + h when step h has a non-finite loss. */
int oracle_local_round(const spes_model_cfg* c, float* params, const int32_t* tokens, int64_t B,
                       int64_t S, int32_t H, const double* lr, const spes_adamw_cfg* opt,
                       const uint8_t* trainable_expert, double* losses);

/* Server::aggregate generalized to owner sets: psi <- fp64 node-order mean over all
 * N node copies; expert e <- fp64 mean over owners (ascending node id); experts
 * without owners keep global_in. node_params: N x P. owners via CSR node -> experts. */
void oracle_outer_step(int32_t kind, double lr, double momentum, float* theta,
                       const float* locals, int32_t N, int64_t n, double* buf);
void oracle_aggregate(const spes_model_cfg* c, int32_t n_nodes, const float* node_params,
                      const int32_t* node_offsets, const int32_t* experts,
                      const float* global_in, float* global_out);

void oracle_similarity(const spes_model_cfg* c, const float* params, int32_t layer,
                       int32_t source, double* sim);
/* returns |peers| */
int32_t oracle_select_peers(const double* sim, int32_t M, int32_t j, int32_t K, int32_t* peers);
/* merge_model; events[L], peers[L][M][K]; returns number of events */
int32_t oracle_merge_model(const spes_model_cfg* c, float* params, const spes_merge_sched* s,
                           int32_t round, spes_merge_event* events, int32_t* peers);

double oracle_lr_at(double peak, double min_frac, int64_t warmup, int64_t total, int64_t step);
void oracle_param_partition(int32_t M, int32_t N, int32_t* node_offsets, int32_t* experts);

/* glibc expf / logf on the calling host, for device-port checks. */
void oracle_expf_array(const float* x, float* y, int64_t n);
/* exhaustive comparison helper: counts mismatches between expf(x) and y over n */
int64_t oracle_expf_mismatches(const float* x, const float* y, int64_t n);
/* bitwise range sweep: for all float bit patterns in [lo, hi] compare expf with y[i-lo] */
int64_t oracle_expf_range_mismatches(uint32_t lo_bits, uint32_t hi_bits, const float* y);

#ifdef __cplusplus
}
#endif

#endif

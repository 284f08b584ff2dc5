/*
 * spes_b200.h -- C ABI of the B200-native SPES hot path.
 *
 * SPES (Sparse Expert Synchronization, arXiv 2602.11543): every node trains the
 * shared parameters psi plus its owned experts Phi_i, keeps the other experts
 * frozen, and every H steps synchronizes psi over all nodes and each expert over
 * its owner set; early rounds additionally blend similar experts (merge warm-up).
 *
 * One context = one node = one GPU. All parameters live on the device in the
 * reference's canonical block order (enumerate_blocks, proj/include/spes/model.hpp:95-111),
 * so spes_load_params / spes_read_params are plain fp32 copies of that layout.
 *
 * Every entry point below names the reference interface it replaces.
 * Errors: a non-zero spes_status whose class mirrors the reference's exception
 * type (proj/include/spes/*.hpp); spes_last_error() returns the
 * message (thread-local).
 */
#ifndef SPES_B200_H
#define SPES_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPES_B200_ABI_VERSION 1

typedef enum {
    SPES_OK = 0,
    SPES_INVALID_ARGUMENT = 1, /* std::invalid_argument                       */
    SPES_OUT_OF_RANGE = 2,     /* std::out_of_range (token id, layer)          */
    SPES_LOGIC_ERROR = 3,      /* std::logic_error (step on frozen block, tied) */
    SPES_RUNTIME_ERROR = 4,    /* std::runtime_error (non-finite loss)         */
    SPES_CUDA_ERROR = 5,       /* device / driver failure                      */
    SPES_NCCL_ERROR = 6,       /* collective failure                           */
    SPES_PROTOCOL_ERROR = 7    /* ProtocolError (proj/include/spes/wire.hpp:23-47) */
} spes_status;

/* ModelConfig + LossCoeffs (proj/include/spes/model.hpp:14-41). */
typedef struct {
    int64_t vocab;
    int64_t hidden;       /* d */
    int64_t intermediate; /* f */
    int32_t layers;       /* L */
    int32_t experts_total;  /* M */
    int32_t experts_active; /* k */
    int32_t renormalize_after_topk;
    int32_t tied_head; /* must be 0: the reference throws logic_error (model.hpp:361) */
    int32_t _pad;
    double coeff_ce, coeff_lb, coeff_moe_z, coeff_z; /* defaults 1, 0.01, 0.001, 1e-5 */
    float rms_eps;                                    /* default 1e-5 */
    float _pad2;
} spes_model_cfg;

/* AdamWConfig (proj/include/spes/trainer.hpp:45-51). */
typedef struct {
    double lr, beta1, beta2, eps, weight_decay;
} spes_adamw_cfg;

/* MergeSchedule (proj/include/spes/merging.hpp:14-25). source: 0 Gate, 1 Up, 2 Concat. */
typedef struct {
    int32_t warmup_rounds;
    int32_t interval;
    double alpha0;
    int32_t peers;
    int32_t source;
} spes_merge_sched;

/* LossBundle (proj/include/spes/model.hpp:376-378). */
typedef struct {
    double total, ce, lb, moe_z, z;
} spes_losses;

/* MergeEvent (proj/include/spes/merging.hpp:97-102); peers: experts_total x peers_k. */
typedef struct {
    int32_t layer;
    int32_t peers_k; /* |Q_j| (identical for every j) */
    double alpha;
    double displacement_sq;
} spes_merge_event;

typedef struct {
    double psi_bytes_in;    /* bytes received for the shared mean               */
    double expert_bytes_in; /* bytes received for owner-set means + gather       */
    double ms;              /* device time of the whole sync (CUDA events)       */
} spes_sync_stats;

typedef struct spes_ctx spes_ctx;

/* ---- configuration helpers (pure host) ---- */

/* ModelConfig::validate (model.hpp:33-40) plus the B200 tiling constraints. */
spes_status spes_validate_cfg(const spes_model_cfg* cfg);
/* sum of numel over enumerate_blocks(cfg) (model.hpp:95-111, 138-149). */
int64_t spes_param_count(const spes_model_cfg* cfg);
/* offsets (in floats) of every block in enumerate_blocks order; n_blocks_out may be NULL. */
spes_status spes_block_offsets(const spes_model_cfg* cfg, int64_t* offsets, int32_t* n_blocks_out);
/* param_partition (model.hpp:466-477): CSR node -> experts (node_offsets has N+1 entries). */
spes_status spes_param_partition(const spes_model_cfg* cfg, int32_t n_nodes,
                                 int32_t* node_offsets, int32_t* experts);
/* Sync plan of spes_sync for an ownership map: primary owner per expert (-1: unowned)
 * and whether the primaries form contiguous balanced slices (in-place all-gather). */
spes_status spes_sync_plan(int32_t experts_total, int32_t n_nodes, const int32_t* node_offsets,
                           const int32_t* experts, int32_t* primary_out, int32_t* balanced_out);
/* LrSchedule::at (proj/src/experiment.cpp:32-41). */
double spes_lr_at(double peak, double min_frac, int64_t warmup_steps, int64_t total_steps,
                  int64_t step);
/* MergeSchedule::merge_at / alpha_at (merging.hpp:21-33). */
int32_t spes_merge_at(const spes_merge_sched* s, int32_t round);
spes_status spes_alpha_at(const spes_merge_sched* s, int32_t round, double* alpha);

/* ---- context ---- */

/* One node. nccl_id: 128-byte ncclUniqueId shared by all nodes (NULL iff n_nodes == 1).
 * Replaces Worker construction + HELLO/ASSIGN (proj/src/protocol.cpp:109-136, 276-292). */
spes_status spes_create(const spes_model_cfg* cfg, int32_t node, int32_t n_nodes,
                        int32_t cuda_device, const void* nccl_id, spes_ctx** out);
void spes_destroy(spes_ctx* ctx);
/* ncclGetUniqueId, for the launcher to broadcast (128 bytes). */
spes_status spes_nccl_unique_id(void* out128);

/* Ownership map, CSR node -> sorted expert ids, identical on every node; any
 * replication r >= 1 (the reference's param_partition is the r = 1 case).
 * TrainMask (trainer.hpp:15-30) of this node is derived from it. */
spes_status spes_set_ownership(spes_ctx* ctx, const int32_t* node_offsets,
                               const int32_t* experts);

/* Full fp32 parameter vector in enumerate_blocks order (host memory). */
spes_status spes_load_params(spes_ctx* ctx, const float* host, int64_t n);
spes_status spes_read_params(spes_ctx* ctx, float* host, int64_t n);
/* Same as spes_load_params from a device buffer of this context's GPU (e.g. a model
 * initialized on the device; no host round trip for multi-GB models). */
spes_status spes_load_params_device(spes_ctx* ctx, const float* dev, int64_t n);

/* Start a local round: fresh MaskedAdamW state (trainer.hpp:151-156) unless carry_state. */
spes_status spes_round_begin(spes_ctx* ctx, int32_t carry_state);

/* One local step (build_loss + backward + MaskedAdamW::step; trainer.hpp:161-206)
 * on host tokens B x (S+1). losses may be NULL (then the step does not synchronize).
 * lr is the already-scheduled learning rate for this step. */
spes_status spes_local_step(spes_ctx* ctx, const int32_t* tokens, int64_t B, int64_t S,
                            const spes_adamw_cfg* opt, spes_losses* losses);
/* Same with device-resident tokens (int32, B x (S+1)). */
spes_status spes_local_step_device(spes_ctx* ctx, const int32_t* d_tokens, int64_t B, int64_t S,
                                   const spes_adamw_cfg* opt, spes_losses* losses);

/* local_round (trainer.hpp:143-222): H steps over H host batches laid out
 * contiguously (H x B x (S+1)); lr[h] per step; per_step[h] receives losses.
 * Throws runtime_error semantics on a non-finite loss (reports the step). */
spes_status spes_local_round(spes_ctx* ctx, const int32_t* tokens, int64_t B, int64_t S,
                             int32_t H, const double* lr, const spes_adamw_cfg* opt,
                             int32_t carry_state, spes_losses* per_step);

/* Sparse synchronization (Server::aggregate, proj/src/protocol.cpp:197-251):
 * psi <- fp64 node-order mean over all nodes; each expert <- fp64 mean over its
 * owner set in ascending node order (== verbatim copy when r = 1); every node
 * ends with the identical global model. Collective: all nodes must call. */
spes_status spes_sync(spes_ctx* ctx, spes_sync_stats* stats);

/* DiLoCo baseline: full-model outer synchronization, Server::aggregate's
 * diloco branch (protocol.cpp:199-213) with OuterOptimizer::step (trainer.hpp:228-271):
 * theta <- OuterOpt(theta, mean_i(local_i - theta)) in fp64 with the nodes in order, kind
 * 0 = SGD, 1 = Nesterov (state persists across calls). spes_outer_begin snapshots the
 * round-start global model (call it once after loading the initial parameters); each
 * spes_outer_sync then replaces every node's parameters with the new global model and keeps
 * it as the next round's theta. Collective: all nodes call it. Bit-exact with the reference. */
spes_status spes_outer_begin(spes_ctx* ctx);
spes_status spes_outer_sync(spes_ctx* ctx, int32_t kind, double lr, double momentum,
                            spes_sync_stats* stats);

/* merge_model (merging.hpp:138-150) on this node's (global) model. events must
 * hold `layers` entries and peers `layers * experts_total * peers` ints (either may be NULL).
 * Returns the number of merged layers in *n_events (0 when the schedule is inactive). */
spes_status spes_merge(spes_ctx* ctx, const spes_merge_sched* sched, int32_t round0,
                       spes_merge_event* events, int32_t* peers, int32_t* n_events);
/* similarity_matrix (merging.hpp:55-82) of one layer, M x M doubles. */
spes_status spes_similarity(spes_ctx* ctx, int32_t layer, int32_t source, double* sim_out);

/* ---- synthetic corpus and batch streams (proj/src/corpus.cpp) ----
 * Host generators bit-identical with the reference (same std::mt19937_64 / libstdc++
 * distributions and draw order): gen_corpus (corpus.cpp:49-79; tokens: sequences x (S+1),
 * source_id may be NULL), shard_corpus (:107-128; order + N+1 node offsets), and the index
 * stream of make_batch_provider (:130-149). The corpus is uploaded to HBM once; a step then
 * transfers only its B row indices and gathers the batch on the device. */
typedef struct spes_batch_stream spes_batch_stream;
spes_status spes_gen_corpus(int64_t vocab, int64_t seq, int32_t sources, int64_t sequences,
                            uint64_t seed, double skew, int32_t* tokens, int32_t* source_id);
spes_status spes_shard_corpus(const int32_t* source_id, int64_t sequences, int32_t nodes,
                              int32_t by_source, uint64_t seed, int64_t* order,
                              int64_t* node_offsets);
spes_status spes_batch_stream_create(const int64_t* shard, int64_t n, int64_t batch, uint64_t seed,
                                     spes_batch_stream** out);
spes_status spes_batch_stream_next(spes_batch_stream* s, int64_t* rows);
void spes_batch_stream_destroy(spes_batch_stream* s);
/* corpus -> HBM (token ids validated once) */
spes_status spes_corpus_load(spes_ctx* ctx, const int32_t* tokens, int64_t sequences, int64_t seq);
/* gen_corpus (corpus.cpp:49-79) generated straight into this context's HBM corpus: the
 * Markov sources are built on the host (make_source's rejection-sampled normals), then the
 * device replays the engine and samples every sequence's chain; the same tokens as
 * spes_gen_corpus bit for bit. vocab <= the model's vocabulary. tokens_out (sequences x
 * (seq+1)) and source_id_out (sequences) may be NULL. */
spes_status spes_corpus_generate(spes_ctx* ctx, int64_t vocab, int64_t seq, int32_t sources,
                                 int64_t sequences, uint64_t seed, double skew,
                                 int32_t* tokens_out, int32_t* source_id_out);
/* local step / round over corpus rows (rows: B, resp. H x B indices) */
spes_status spes_local_step_rows(spes_ctx* ctx, const int64_t* rows, int64_t B,
                                 const spes_adamw_cfg* opt, spes_losses* losses);
spes_status spes_local_round_rows(spes_ctx* ctx, const int64_t* rows, int64_t B, int32_t H,
                                  const double* lr, const spes_adamw_cfg* opt, int32_t carry_state,
                                  spes_losses* per_step);

/* ---- CommLedger (protocol.hpp:29-52) ----
 * The reference's transport-agnostic byte accounting for a run of `rounds` SPES rounds
 * over n_nodes, as its Server records it (protocol.cpp:56-175): every frame is its payload
 * plus an 18-byte header; HELLO is counted under node -1 (the connection has no node yet),
 * then ASSIGN, the GLOBAL_MODEL broadcasts of rounds 1..rounds+1, each node's LOCAL_UPDATE
 * (shared blocks + owned experts; the whole model with diloco) and ROUND_DONE, and the BYE
 * exchange at round rounds+1. The B200 nodes move these parameters over NCCL instead; this
 * keeps the reference's accounting (and its metrics.csv bytes_up / bytes_down columns).
 * Ownership: CSR map as spes_set_ownership, or NULL for param_partition (the reference's
 * server assignment). Entries in (node, round) order; up to cap are written, *n_entries
 * is the total; totals = {total_up, total_down, pushes, broadcasts}. */
typedef struct {
    int32_t node, round;
    uint64_t up, down;
} spes_ledger_entry;
spes_status spes_comm_ledger(const spes_model_cfg* cfg, int32_t n_nodes,
                             const int32_t* node_offsets, const int32_t* experts, int32_t rounds,
                             int32_t diloco, spes_ledger_entry* entries, int32_t cap,
                             int32_t* n_entries, uint64_t* totals);
/* RoundMetrics (protocol.hpp:132-137) -> the text of an experiment's metrics.csv
 * (experiment.cpp:376-385: same header, columns and number formatting). tokens_seen =
 * tokens_per_round * round (nodes * H * batch * seq_len per round in the reference);
 * wall_ms may be NULL (0.0). *len = the text's length; up to cap bytes are written. */
typedef struct {
    int32_t round;
    double mean_total, mean_ce, mean_lb, mean_moe_z, mean_z, merge_displacement_sq;
    uint64_t bytes_up, bytes_down;
} spes_round_metrics;
spes_status spes_metrics_csv(const spes_round_metrics* rows, int32_t n, int64_t tokens_per_round,
                             const double* wall_ms, char* out, int64_t cap, int64_t* len);

/* ---- upcycling ----
 * upcycle_from_dense (model.hpp:415-460): a dense model (experts_total == 1) -> an m-expert
 * model: embedding / norms / head copied, routers widened by replicating their column,
 * every expert a copy of the dense FFN with a noise_frac subset of its elements perturbed
 * by N(0, noise_std) draws (std::mt19937_64(seed), libstdc++ distributions, the reference's
 * draw order => bit-identical), renormalize_after_topk = 1. out_cfg may be NULL; out_params
 * holds spes_param_count(out_cfg) floats. invalid_argument: dense M != 1, m < 2. */
spes_status spes_upcycle_from_dense(const spes_model_cfg* dense_cfg, const float* dense_params,
                                    int32_t m, double noise_frac, double noise_std, uint64_t seed,
                                    spes_model_cfg* out_cfg, float* out_params);

/* ---- wire / checkpoint format (proj/src/wire.cpp) ----
 * Byte-identical to the reference: encode_blocks(model_to_blocks(params)) is the
 * GLOBAL_MODEL payload (wire.cpp:96-115,154-159); a checkpoint is that payload followed by
 * the u64 round (write_checkpoint / read_checkpoint, wire.cpp:212-236). Decoding validates
 * exactly like decode_blocks + blocks_into_model (wire.cpp:117-176): SPES_PROTOCOL_ERROR
 * with the reference's ProtoError name as message prefix ("[Truncated] ..."). */
/* payload bytes of a model (-1 on an invalid config) */
int64_t spes_model_payload_bytes(const spes_model_cfg* cfg);
/* host-only codec over a flat fp32 parameter vector (enumerate_blocks order) */
spes_status spes_encode_model_host(const spes_model_cfg* cfg, const float* params, uint8_t* out,
                                   int64_t cap);
spes_status spes_decode_model_host(const spes_model_cfg* cfg, const uint8_t* payload, int64_t len,
                                   float* params);
/* the context's device parameters (device -> host export / host -> device import; the
 * bf16 GEMM operand copies are refreshed on import) */
spes_status spes_encode_model(spes_ctx* ctx, uint8_t* out, int64_t cap);
spes_status spes_decode_model(spes_ctx* ctx, const uint8_t* payload, int64_t len);
spes_status spes_write_checkpoint(spes_ctx* ctx, const char* path, uint64_t round);
spes_status spes_read_checkpoint(spes_ctx* ctx, const char* path, uint64_t* round);

/* ---- introspection (tests / benchmarks) ---- */

/* Counters: optimizer-state scalars (2(|psi|+|Phi_i|)), gradient scalars, step count. */
spes_status spes_counts(spes_ctx* ctx, int64_t* opt_state_scalars, int64_t* grad_scalars,
                        int64_t* adam_step);
/* Read a named device buffer of the last step into host (bytes >= the buffer's size):
 *   "h" (layer l's input; layer 0 rebuilt from the current embedding), "logits", "probs",
 *   "topk_idx", "topk_w", "counts", "pad_off", "row_token", "slot_row", "perm", "y",
 *   "grad_h0" (gradient w.r.t. the layer-0 input), "head_logits" (V != 256 only),
 *   "w1" / "w2" (layer l's bf16 expert operand copies: [M][d][2f] gate|up interleaved in
 *   128-column blocks, [M][f][d]). Unknown names: invalid_argument. */
spes_status spes_debug_read(spes_ctx* ctx, const char* name, int32_t layer, void* host,
                            int64_t bytes);
/* Gradient of the last step, full parameter layout (zeros for frozen blocks). Needs the
 * unfused optimizer for owned experts (logic_error otherwise, see below). */
spes_status spes_read_grads(spes_ctx* ctx, float* host, int64_t n);
/* Optimizer placement. 1: the owned experts' MaskedAdamW runs inside the dW GEMM
 * epilogue and their gradients are never materialized (read_grads then throws
 * logic_error). 0 (default): gradients are materialized and one standalone optimizer
 * pass runs after the backward. Both give identical bits. */
spes_status spes_set_fused_optimizer(spes_ctx* ctx, int32_t on);
/* Inner optimizer of the local steps (LocalRoundConfig::inner, trainer.hpp:116-121):
 * 0 = MaskedAdamW (default), 1 = SGD (theta -= float(lr) * g on the trainable blocks,
 * trainer.hpp:197-204; no optimizer state, the fused placement does not apply).
 * invalid_argument for other kinds. */
spes_status spes_set_inner_optimizer(spes_ctx* ctx, int32_t kind);
/* Stream layout of the local step. 1 (default): off-critical-path work (embedding-gradient
 * bucketing, loss scalars, the router's scalar backward, the owned experts' AdamW) runs on
 * a low-priority second stream beside the GEMMs; 0: one stream. Identical bits either way. */
spes_status spes_set_stream_overlap(spes_ctx* ctx, int32_t on);
/* Live per-kernel-family timing: CUDA events bracket every launch family on the
 * context stream while enabled; totals accumulate until spes_profile_reset. */
spes_status spes_profile(spes_ctx* ctx, int32_t enable);
spes_status spes_profile_reset(spes_ctx* ctx);
int32_t spes_profile_count(spes_ctx* ctx);
spes_status spes_profile_get(spes_ctx* ctx, int32_t index, char* name64, double* total_ms,
                             int64_t* launches);
/* The CUDA stream all work of this context is issued on (cudaStream_t). */
void* spes_stream(spes_ctx* ctx);
/* Number of kernels this context launched since creation. */
int64_t spes_kernel_launches(spes_ctx* ctx);
const char* spes_last_error(void);

/* ---- kernel-level entry points for bit-exact parity on identical inputs ---- */

/* Router forward (rmsnorm -> logits -> softmax -> top-k) on host arrays. */
spes_status spes_kernel_router(const spes_model_cfg* cfg, const float* h, const float* gain,
                               const float* router, int64_t T, float* normed, float* logits,
                               float* probs, int32_t* topk_idx, float* topk_w, int32_t* counts,
                               int32_t* perm, int32_t cuda_device);
/* MaskedAdamW element update on host arrays (trainer.hpp:85-92); step = optimizer step count. */
spes_status spes_kernel_adamw(float* theta, const float* grad, float* m, float* v, int64_t n,
                              const spes_adamw_cfg* opt, int64_t step, int32_t cuda_device);
/* Owner-set fp64 node-order mean: x is n_owners x n (ascending node order). */
spes_status spes_kernel_owner_mean(const float* x, int32_t n_owners, int64_t n, float* out,
                                   int32_t cuda_device);
/* glibc-compatible expf port evaluated on the device / on the host (variant: 0 auto). */
spes_status spes_kernel_expf(const float* x, float* y, int64_t n, int32_t cuda_device);
void spes_host_expf_port(const float* x, float* y, int64_t n, int32_t variant);
int32_t spes_host_expf_variant(void);

#ifdef __cplusplus
}
#endif

#endif /* SPES_B200_H */

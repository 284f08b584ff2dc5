/*
 * spes_oracle.c -- CPU restatement of the SPES hot path. TEST INFRASTRUCTURE ONLY
 * (see spes_oracle.h). Plain C11, fp32 with the reference's operation order:
 *   - built without FMA contraction (-ffp-contract=off, no -mfma), like the
 *     reference's -O3 build (proj/CMakeLists.txt:6-8 has no -march);
 *   - sequential reductions exactly where the reference has them;
 *   - expf/logf/sqrtf from glibc, as std::exp/std::log/std::sqrt on float.
 * Citations are to /root/reference/proj/.
 */
#include "spes_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IDX(r, c, ld) ((int64_t)(r) * (int64_t)(ld) + (int64_t)(c))

/* ---------------- layout: enumerate_blocks (include/spes/model.hpp:95-111) ---------------- */

int64_t oracle_off_emb(const spes_model_cfg* c) { (void)c; return 0; }
int64_t oracle_off_head(const spes_model_cfg* c) { return c->vocab * c->hidden; }
static int64_t shared_layer_base(const spes_model_cfg* c) {
    return c->vocab * c->hidden + c->hidden * c->vocab;
}
int64_t oracle_off_norm(const spes_model_cfg* c, int l) {
    return shared_layer_base(c) + (int64_t)l * (c->hidden + c->hidden * c->experts_total);
}
int64_t oracle_off_router(const spes_model_cfg* c, int l) {
    return oracle_off_norm(c, l) + c->hidden;
}
static int64_t expert_base(const spes_model_cfg* c) {
    return shared_layer_base(c) + (int64_t)c->layers * (c->hidden + c->hidden * c->experts_total);
}
int64_t oracle_off_expert(const spes_model_cfg* c, int l, int j) {
    return expert_base(c) +
           ((int64_t)l * c->experts_total + j) * 3 * c->hidden * c->intermediate;
}
int64_t oracle_param_count(const spes_model_cfg* c) {
    return oracle_off_expert(c, c->layers, 0);
}

/* ---------------- kernels (include/spes/kernels.hpp) ---------------- */

/* matmul_serial (kernels.hpp:27-38): C = A[m x k] B[k x n], row by row, p outer. */
static void mm(const float* a, const float* b, float* c, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static) if (m > 1)
    for (int64_t i = 0; i < m; ++i) {
        float* crow = c + i * n;
        for (int64_t j = 0; j < n; ++j) crow[j] = 0.f;
        for (int64_t p = 0; p < k; ++p) {
            float av = a[i * k + p];
            const float* brow = b + p * n;
            for (int64_t j = 0; j < n; ++j) crow[j] += av * brow[j];
        }
    }
}

/* matmul_nt_acc (kernels.hpp:62-75): C[m x n] += A[m x k] B[n x k]^T. */
static void mm_nt_acc(const float* a, const float* b, float* c, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static) if (m > 1)
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            float s = 0.f;
            const float* arow = a + i * k;
            const float* brow = b + j * k;
            for (int64_t p = 0; p < k; ++p) s += arow[p] * brow[p];
            c[i * n + j] += s;
        }
}

/* matmul_tn_acc (kernels.hpp:77-88): C[k x n] += A[m x k]^T B[m x n]. */
static void mm_tn_acc(const float* a, const float* b, float* c, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(static) if (k > 1)
    for (int64_t i = 0; i < k; ++i)
        for (int64_t j = 0; j < n; ++j) {
            float s = 0.f;
            for (int64_t p = 0; p < m; ++p) s += a[p * k + i] * b[p * n + j];
            c[i * n + j] += s;
        }
}

/* sigmoid (kernels.hpp:92-97) */
static float sigmoidf_ref(float z) {
    if (z >= 0.f) return 1.f / (1.f + expf(-z));
    float e = expf(z);
    return e / (1.f + e);
}

/* rmsnorm_forward (kernels.hpp:117-128) */
static void rmsnorm_fwd(const float* x, const float* g, float* y, int64_t rows, int64_t d,
                        float eps) {
#pragma omp parallel for schedule(static) if (rows > 1)
    for (int64_t r = 0; r < rows; ++r) {
        const float* xr = x + r * d;
        float* yr = y + r * d;
        float ms = 0.f;
        for (int64_t j = 0; j < d; ++j) ms += xr[j] * xr[j];
        float inv = 1.f / sqrtf(ms / (float)d + eps);
        for (int64_t j = 0; j < d; ++j) yr[j] = xr[j] * inv * g[j];
    }
}

/* rmsnorm_backward_acc (kernels.hpp:130-152), serial over rows */
static void rmsnorm_bwd_acc(const float* x, const float* g, const float* gy, float* gx, float* gg,
                            int64_t rows, int64_t d, float eps) {
    for (int64_t r = 0; r < rows; ++r) {
        const float* xr = x + r * d;
        const float* gyr = gy + r * d;
        float ms = 0.f;
        for (int64_t j = 0; j < d; ++j) ms += xr[j] * xr[j];
        float m = ms / (float)d + eps;
        float inv = 1.f / sqrtf(m);
        float dot = 0.f;
        for (int64_t j = 0; j < d; ++j) dot += gyr[j] * g[j] * xr[j];
        float coef = dot * inv * inv * inv / (float)d;
        if (gx) {
            float* gxr = gx + r * d;
            for (int64_t j = 0; j < d; ++j) gxr[j] += gyr[j] * g[j] * inv - coef * xr[j];
        }
        if (gg)
            for (int64_t j = 0; j < d; ++j) gg[j] += gyr[j] * xr[j] * inv;
    }
}

/* softmax_rows (kernels.hpp:156-172) */
static void softmax_rows(const float* x, float* y, int64_t rows, int64_t cols) {
#pragma omp parallel for schedule(static) if (rows > 1)
    for (int64_t r = 0; r < rows; ++r) {
        const float* xr = x + r * cols;
        float* yr = y + r * cols;
        float mx = xr[0];
        for (int64_t j = 1; j < cols; ++j) mx = (mx < xr[j]) ? xr[j] : mx; /* std::max(mx, x) */
        float sum = 0.f;
        for (int64_t j = 0; j < cols; ++j) {
            yr[j] = expf(xr[j] - mx);
            sum += yr[j];
        }
        float inv = 1.f / sum;
        for (int64_t j = 0; j < cols; ++j) yr[j] *= inv;
    }
}

/* logsumexp_rows (kernels.hpp:174-185) */
static void logsumexp_rows(const float* x, float* lse, int64_t rows, int64_t cols) {
#pragma omp parallel for schedule(static) if (rows > 1)
    for (int64_t r = 0; r < rows; ++r) {
        const float* xr = x + r * cols;
        float mx = xr[0];
        for (int64_t j = 1; j < cols; ++j) mx = (mx < xr[j]) ? xr[j] : mx;
        float sum = 0.f;
        for (int64_t j = 0; j < cols; ++j) sum += expf(xr[j] - mx);
        lse[r] = mx + logf(sum);
    }
}

/* ---------------- routing (model.hpp:185-216, 314-318) ---------------- */

/* Stable descending sort by prob (ties keep lower index), first k, then ascending. */
static void topk_stable(const float* p, int32_t M, int32_t k, int32_t* out) {
    /* insertion sort over indices == std::stable_sort with comparator p[a] > p[b] */
    int32_t idx[1024];
    for (int32_t i = 0; i < M; ++i) idx[i] = i;
    for (int32_t i = 1; i < M; ++i) {
        int32_t v = idx[i];
        int32_t j = i - 1;
        while (j >= 0 && p[v] > p[idx[j]]) {
            idx[j + 1] = idx[j];
            --j;
        }
        idx[j + 1] = v;
    }
    for (int32_t i = 0; i < k; ++i) out[i] = idx[i];
    /* std::sort ascending (distinct ints) */
    for (int32_t i = 1; i < k; ++i) {
        int32_t v = out[i];
        int32_t j = i - 1;
        while (j >= 0 && out[j] > v) {
            out[j + 1] = out[j];
            --j;
        }
        out[j + 1] = v;
    }
}

static void route_rows(const spes_model_cfg* c, const float* probs, int64_t T, int32_t* idx,
                       float* w, int32_t* counts, int32_t* perm) {
    const int32_t M = c->experts_total, k = c->experts_active;
    for (int64_t t = 0; t < T; ++t) {
        topk_stable(probs + t * M, M, k, idx + t * k);
        float denom = 0.f;
        for (int32_t s = 0; s < k; ++s) denom += probs[t * M + idx[t * k + s]];
        for (int32_t s = 0; s < k; ++s) {
            float wv = probs[t * M + idx[t * k + s]];
            if (c->renormalize_after_topk) wv /= denom;
            if (w) w[t * k + s] = wv;
        }
    }
    if (counts || perm) {
        int32_t* cnt = (int32_t*)calloc((size_t)M, sizeof(int32_t));
        for (int64_t t = 0; t < T; ++t)
            for (int32_t s = 0; s < k; ++s) cnt[idx[t * k + s]]++;
        if (counts) memcpy(counts, cnt, (size_t)M * sizeof(int32_t));
        if (perm) {
            int64_t* pos = (int64_t*)malloc((size_t)M * sizeof(int64_t));
            int64_t acc = 0;
            for (int32_t j = 0; j < M; ++j) {
                pos[j] = acc;
                acc += cnt[j];
            }
            for (int64_t t = 0; t < T; ++t)
                for (int32_t s = 0; s < k; ++s) perm[pos[idx[t * k + s]]++] = (int32_t)t;
            free(pos);
        }
        free(cnt);
    }
}

void oracle_router_forward(const spes_model_cfg* c, const float* h, const float* gain,
                           const float* router, int64_t T, float* normed, float* logits,
                           float* probs, int32_t* topk_idx, float* topk_w, int32_t* counts,
                           int32_t* perm) {
    const int64_t d = c->hidden, M = c->experts_total;
    rmsnorm_fwd(h, gain, normed, T, d, c->rms_eps);        /* model.hpp:292 */
    mm(normed, router, logits, T, d, M);                    /* model.hpp:294 */
    softmax_rows(logits, probs, T, M);                      /* model.hpp:295 */
    route_rows(c, probs, T, topk_idx, topk_w, counts, perm); /* model.hpp:297 */
}

/* ---------------- forward + backward (model.hpp:252-374, graph.hpp:340-348) ---------------- */

typedef struct {
    int32_t n;        /* rows routed to this expert */
    int32_t* rows;    /* token ids, ascending (model.hpp:314-318) */
    float *gp, *gate, *up, *hm, *y; /* [n x f] x4, [n x d] */
} expert_act;

typedef struct {
    float *h, *normed, *logits, *probs, *lse_r, *denom;
    int32_t* idx;
    int32_t counts[1024];
    expert_act* ex;
} layer_act;

int oracle_forward_backward(const spes_model_cfg* c, const float* P, const int32_t* tokens,
                            int64_t B, int64_t S, const uint8_t* trainable_expert, float* G,
                            double* losses, oracle_trace* tr) {
    const int64_t V = c->vocab, d = c->hidden, f = c->intermediate;
    const int32_t L = c->layers, M = c->experts_total, k = c->experts_active;
    const int64_t T = B * S;
    const int renorm = c->renormalize_after_topk;
    const float eps = c->rms_eps;
    const int64_t NP = oracle_param_count(c);

    int32_t* inputs = (int32_t*)malloc((size_t)T * sizeof(int32_t));
    int32_t* targets = (int32_t*)malloc((size_t)T * sizeof(int32_t));
    for (int64_t b = 0; b < B; ++b)
        for (int64_t s = 0; s < S; ++s) {
            int32_t tin = tokens[b * (S + 1) + s], tout = tokens[b * (S + 1) + s + 1];
            if (tin < 0 || tin >= V || tout < 0 || tout >= V) { /* model.hpp:280-281 */
                free(inputs);
                free(targets);
                return 2;
            }
            inputs[b * S + s] = tin;
            targets[b * S + s] = tout;
        }

    memset(G, 0, (size_t)NP * sizeof(float));
    layer_act* la = (layer_act*)calloc((size_t)L, sizeof(layer_act));

    /* h0 = gather_rows(emb, inputs) (model.hpp:286) */
    float* h = (float*)malloc((size_t)(T * d) * sizeof(float));
    for (int64_t t = 0; t < T; ++t)
        memcpy(h + t * d, P + oracle_off_emb(c) + (int64_t)inputs[t] * d, (size_t)d * sizeof(float));

    float moe_z_sum = 0.f, lb_sum = 0.f;
    float inv_T = 1.f / (float)(T); /* GraphT::mean: T(1)/numel */

    for (int32_t l = 0; l < L; ++l) {
        layer_act* A = &la[l];
        const float* gain = P + oracle_off_norm(c, l);
        const float* R = P + oracle_off_router(c, l);
        A->h = h;
        A->normed = (float*)malloc((size_t)(T * d) * sizeof(float));
        A->logits = (float*)malloc((size_t)(T * M) * sizeof(float));
        A->probs = (float*)malloc((size_t)(T * M) * sizeof(float));
        A->idx = (int32_t*)malloc((size_t)(T * k) * sizeof(int32_t));
        A->lse_r = (float*)malloc((size_t)T * sizeof(float));
        A->denom = renorm ? (float*)malloc((size_t)T * sizeof(float)) : NULL;
        rmsnorm_fwd(h, gain, A->normed, T, d, eps);  /* model.hpp:292 */
        mm(A->normed, R, A->logits, T, d, M);         /* model.hpp:294 */
        softmax_rows(A->logits, A->probs, T, M);      /* model.hpp:295 */
        float* wtmp = (float*)malloc((size_t)(T * k) * sizeof(float));
        route_rows(c, A->probs, T, A->idx, wtmp, NULL, NULL); /* model.hpp:297 */
        if (tr && tr->normed) memcpy(tr->normed + (int64_t)l * T * d, A->normed, (size_t)(T * d) * 4);
        if (tr && tr->logits) memcpy(tr->logits + (int64_t)l * T * M, A->logits, (size_t)(T * M) * 4);
        if (tr && tr->probs) memcpy(tr->probs + (int64_t)l * T * M, A->probs, (size_t)(T * M) * 4);
        if (tr && tr->topk_idx) memcpy(tr->topk_idx + (int64_t)l * T * k, A->idx, (size_t)(T * k) * 4);
        if (tr && tr->topk_w) memcpy(tr->topk_w + (int64_t)l * T * k, wtmp, (size_t)(T * k) * 4);
        free(wtmp);
        /* renormalization denominator: add chain of gather_cols (model.hpp:301-312) */
        if (renorm)
            for (int64_t t = 0; t < T; ++t) {
                float dn = A->probs[t * M + A->idx[t * k + 0]];
                for (int32_t s = 1; s < k; ++s) dn = dn + A->probs[t * M + A->idx[t * k + s]];
                A->denom[t] = dn;
            }
        /* groups (model.hpp:314-318) */
        memset(A->counts, 0, sizeof(A->counts));
        for (int64_t t = 0; t < T * k; ++t) A->counts[A->idx[t]]++;
        A->ex = (expert_act*)calloc((size_t)M, sizeof(expert_act));
        for (int32_t j = 0; j < M; ++j) {
            A->ex[j].n = A->counts[j];
            A->ex[j].rows = (int32_t*)malloc((size_t)(A->counts[j] + 1) * sizeof(int32_t));
            A->ex[j].n = 0;
        }
        for (int64_t t = 0; t < T; ++t)
            for (int32_t s = 0; s < k; ++s) {
                expert_act* E = &A->ex[A->idx[t * k + s]];
                E->rows[E->n++] = (int32_t)t;
            }
        if (tr && tr->counts) memcpy(tr->counts + (int64_t)l * M, A->counts, (size_t)M * 4);
        if (tr && tr->perm) {
            int64_t q = 0;
            for (int32_t j = 0; j < M; ++j)
                for (int32_t r = 0; r < A->ex[j].n; ++r) tr->perm[(int64_t)l * T * k + q++] = A->ex[j].rows[r];
        }

        /* experts (model.hpp:322-337) */
        float* moe_out = (float*)calloc((size_t)(T * d), sizeof(float));
        int have_out = 0;
        for (int32_t j = 0; j < M; ++j) {
            expert_act* E = &A->ex[j];
            const int64_t n = E->n;
            if (n == 0) continue;
            const float* wg = P + oracle_off_expert(c, l, j);
            const float* wu = wg + d * f;
            const float* wd = wg + 2 * d * f;
            float* xj = (float*)malloc((size_t)(n * d) * sizeof(float));
            for (int64_t r = 0; r < n; ++r)
                memcpy(xj + r * d, A->normed + (int64_t)E->rows[r] * d, (size_t)d * 4);
            E->gp = (float*)malloc((size_t)(n * f) * 4);
            E->gate = (float*)malloc((size_t)(n * f) * 4);
            E->up = (float*)malloc((size_t)(n * f) * 4);
            E->hm = (float*)malloc((size_t)(n * f) * 4);
            E->y = (float*)malloc((size_t)(n * d) * 4);
            /* swiglu_expert (graph.hpp:391-400) */
            mm(xj, wg, E->gp, n, d, f);
            for (int64_t i = 0; i < n * f; ++i) E->gate[i] = E->gp[i] * sigmoidf_ref(E->gp[i]);
            mm(xj, wu, E->up, n, d, f);
            for (int64_t i = 0; i < n * f; ++i) E->hm[i] = E->gate[i] * E->up[i];
            mm(E->hm, wd, E->y, n, f, d);
            free(xj);
            /* wfull = gather_cols(probs, j) [/ denom]; wj = select_rows; rowwise_mul; scatter; add */
            for (int64_t r = 0; r < n; ++r) {
                int64_t t = E->rows[r];
                float wv = A->probs[t * M + j];
                if (renorm) wv = wv / A->denom[t];
                for (int64_t q = 0; q < d; ++q) {
                    float contrib = 0.f + E->y[r * d + q] * wv; /* scatter into zeros */
                    if (have_out)
                        moe_out[t * d + q] = moe_out[t * d + q] + contrib;
                    else
                        moe_out[t * d + q] = contrib;
                }
            }
            if (!have_out) {
                /* tokens not routed to the first expert: the contrib tensor is zero there */
                have_out = 1;
            }
        }
        float* hn = (float*)malloc((size_t)(T * d) * sizeof(float));
        for (int64_t i = 0; i < T * d; ++i) hn[i] = have_out ? h[i] + moe_out[i] : h[i];
        free(moe_out);
        /* moe_z: mean(square(logsumexp_rows(logits))) (model.hpp:341) */
        logsumexp_rows(A->logits, A->lse_r, T, M);
        float s = 0.f;
        for (int64_t t = 0; t < T; ++t) s += A->lse_r[t] * A->lse_r[t];
        moe_z_sum = moe_z_sum + s * inv_T;
        /* lb (model.hpp:344-358) */
        {
            int64_t assignments = T * k;
            float coeff[1024];
            for (int32_t j = 0; j < M; ++j) {
                double f_j = (double)A->counts[j] / (double)assignments;
                coeff[j] = (float)((double)M * f_j / (double)T);
            }
            float ls = 0.f;
            for (int64_t t = 0; t < T; ++t)
                for (int32_t j = 0; j < M; ++j) ls += A->probs[t * M + j] * coeff[j];
            lb_sum = lb_sum + ls;
        }
        if (tr && tr->h) memcpy(tr->h + (int64_t)l * T * d, h, (size_t)(T * d) * 4);
        h = hn;
    }
    if (tr && tr->h) memcpy(tr->h + (int64_t)L * T * d, h, (size_t)(T * d) * 4);

    /* head + CE + z (model.hpp:362-373, graph.hpp:410-423) */
    const float* head = P + oracle_off_head(c);
    float* ol = (float*)malloc((size_t)(T * V) * 4);
    mm(h, head, ol, T, d, V);
    if (tr && tr->head_logits) memcpy(tr->head_logits, ol, (size_t)(T * V) * 4);
    float* lse = (float*)malloc((size_t)T * 4);
    logsumexp_rows(ol, lse, T, V);
    float ssum = 0.f, s2 = 0.f;
    for (int64_t t = 0; t < T; ++t) {
        float picked = ol[t * V + targets[t]];
        float neg = picked * -1.f;
        ssum += lse[t] + neg;
    }
    for (int64_t t = 0; t < T; ++t) s2 += lse[t] * lse[t];
    const float ce = ssum * inv_T;
    const float z = s2 * inv_T;
    const float inv_L = 1.f / (float)L;
    const float moe_z = moe_z_sum * inv_L;
    const float lb = lb_sum * inv_L;
    const float c_ce = (float)c->coeff_ce, c_lb = (float)c->coeff_lb, c_mz = (float)c->coeff_moe_z,
                c_z = (float)c->coeff_z;
    const float total = (ce * c_ce + lb * c_lb) + (moe_z * c_mz + z * c_z);
    losses[0] = total;
    losses[1] = ce;
    losses[2] = lb;
    losses[3] = moe_z;
    losses[4] = z;

    /* ---------------- backward: reverse tape order (graph.hpp:340-348) ---------------- */
    /* scalar chain */
    const float g_a3 = 1.f, g_a6 = 1.f;
    const float g_z = c_z * g_a6;
    const float g_mz = c_mz * g_a6;
    const float g_lb = c_lb * g_a3;
    const float g_ce = c_ce * g_a3;
    const float g_lbsum = inv_L * g_lb;
    const float g_mzsum = inv_L * g_mz;
    const float g_s2 = inv_T * g_z;
    const float g_ssum = inv_T * g_ce;

    float* gol = (float*)calloc((size_t)(T * V), 4); /* d out_logits */
    float* glse = (float*)calloc((size_t)T, 4);
    for (int64_t t = 0; t < T; ++t) {
        glse[t] += g_s2 * lse[t]; /* mul(lse,lse): a then b */
        glse[t] += g_s2 * lse[t];
        glse[t] += g_ssum;          /* add(lse, neg) */
        float gpick = -1.f * g_ssum; /* scale(picked, -1) */
        gol[t * V + targets[t]] += gpick; /* gather_cols */
    }
    {
        float* p = (float*)malloc((size_t)(T * V) * 4);
        softmax_rows(ol, p, T, V); /* logsumexp backward recomputes softmax (graph.hpp:196-203) */
        for (int64_t t = 0; t < T; ++t)
            for (int64_t j = 0; j < V; ++j) gol[t * V + j] += glse[t] * p[t * V + j];
        free(p);
    }
    float* gh = (float*)calloc((size_t)(T * d), 4);
    mm_nt_acc(gol, head, gh, T, V, d);                     /* d h_L */
    mm_tn_acc(h, gol, G + oracle_off_head(c), T, d, V);    /* d head */
    if (tr && tr->grad_h) memcpy(tr->grad_h + (int64_t)L * T * d, gh, (size_t)(T * d) * 4);
    free(ol);
    free(lse);
    free(glse);
    free(gol);
    free(h);

    for (int32_t l = L - 1; l >= 0; --l) {
        layer_act* A = &la[l];
        const float* gain = P + oracle_off_norm(c, l);
        const float* R = P + oracle_off_router(c, l);
        float* gprobs = (float*)calloc((size_t)(T * M), 4);
        float* glog = (float*)calloc((size_t)(T * M), 4);
        /* lb: mul(probs, cmat) (nodes 16-18) */
        {
            int64_t assignments = T * k;
            for (int32_t j = 0; j < M; ++j) {
                double f_j = (double)A->counts[j] / (double)assignments;
                float cj = (float)((double)M * f_j / (double)T);
                for (int64_t t = 0; t < T; ++t) gprobs[t * M + j] += g_lbsum * cj;
            }
        }
        /* moe_z: logsumexp backward (nodes 10-14) */
        {
            const float g_s = inv_T * g_mzsum;
            for (int64_t t = 0; t < T; ++t) {
                float gl = 0.f;
                gl += g_s * A->lse_r[t];
                gl += g_s * A->lse_r[t];
                for (int32_t j = 0; j < M; ++j) glog[t * M + j] += gl * A->probs[t * M + j];
            }
        }
        /* h_{l+1} = add(h_l, moe_out): grad passes to both (node 9) */
        float* gnext = gh; /* complete d h_{l+1} */
        float* gh_l = (float*)calloc((size_t)(T * d), 4);
        for (int64_t i = 0; i < T * d; ++i) gh_l[i] += gnext[i];
        float* gnormed = (float*)calloc((size_t)(T * d), 4);
        float* gdenom = renorm ? (float*)calloc((size_t)T, 4) : NULL;
        /* experts, descending (node 8) */
        for (int32_t j = M - 1; j >= 0; --j) {
            expert_act* E = &A->ex[j];
            const int64_t n = E->n;
            if (n == 0) continue;
            const int owned = trainable_expert[j] != 0;
            const float* wg = P + oracle_off_expert(c, l, j);
            const float* wu = wg + d * f;
            const float* wd = wg + 2 * d * f;
            float* Gwg = G + oracle_off_expert(c, l, j);
            float* Gwu = Gwg + d * f;
            float* Gwd = Gwg + 2 * d * f;
            float* gy = (float*)calloc((size_t)(n * d), 4);
            float* gwj = (float*)calloc((size_t)n, 4);
            for (int64_t r = 0; r < n; ++r) {
                int64_t t = E->rows[r];
                float wv = A->probs[t * M + j];
                if (renorm) wv = wv / A->denom[t];
                float acc = 0.f;
                for (int64_t q = 0; q < d; ++q) {
                    float g = gnext[t * d + q]; /* scatter_rows backward */
                    gy[r * d + q] += g * wv;
                    acc += g * E->y[r * d + q];
                }
                gwj[r] += acc;
            }
            /* select_rows(wfull) backward, div backward, gather_cols backward */
            for (int64_t r = 0; r < n; ++r) {
                int64_t t = E->rows[r];
                float gw = gwj[r]; /* wfull.grad[t] (0 + gwj) */
                if (renorm) {
                    float a = A->probs[t * M + j], b = A->denom[t];
                    float gwf = 0.f;
                    gwf += gw / b;
                    gdenom[t] -= gw * a / (b * b);
                    gprobs[t * M + j] += gwf;
                } else {
                    gprobs[t * M + j] += gw;
                }
            }
            /* yj = matmul(hm, wd) */
            float* ghm = (float*)calloc((size_t)(n * f), 4);
            mm_nt_acc(gy, wd, ghm, n, d, f);
            if (owned) mm_tn_acc(E->hm, gy, Gwd, n, f, d);
            /* hm = mul(gate, up) */
            float* ggate = (float*)calloc((size_t)(n * f), 4);
            float* gup = (float*)calloc((size_t)(n * f), 4);
            for (int64_t i = 0; i < n * f; ++i) {
                ggate[i] += ghm[i] * E->up[i];
                gup[i] += ghm[i] * E->gate[i];
            }
            /* up = matmul(xj, wu) */
            float* xj = (float*)malloc((size_t)(n * d) * 4);
            for (int64_t r = 0; r < n; ++r)
                memcpy(xj + r * d, A->normed + (int64_t)E->rows[r] * d, (size_t)d * 4);
            float* gx = (float*)calloc((size_t)(n * d), 4);
            mm_nt_acc(gup, wu, gx, n, f, d);
            if (owned) mm_tn_acc(xj, gup, Gwu, n, d, f);
            /* gate = silu(gp) (kernels.hpp:105-113) */
            float* ggp = (float*)calloc((size_t)(n * f), 4);
            for (int64_t i = 0; i < n * f; ++i) {
                float s = sigmoidf_ref(E->gp[i]);
                ggp[i] += ggate[i] * s * (1.f + E->gp[i] * (1.f - s));
            }
            /* gp = matmul(xj, wg) */
            mm_nt_acc(ggp, wg, gx, n, f, d);
            if (owned) mm_tn_acc(xj, ggp, Gwg, n, d, f);
            /* xj = select_rows(normed) */
            for (int64_t r = 0; r < n; ++r) {
                int64_t t = E->rows[r];
                for (int64_t q = 0; q < d; ++q) gnormed[t * d + q] += gx[r * d + q];
            }
            free(gy); free(gwj); free(ghm); free(ggate); free(gup); free(xj); free(gx); free(ggp);
        }
        /* renorm denominator chain (node 7): slots descending */
        if (renorm)
            for (int64_t t = 0; t < T; ++t)
                for (int32_t s = k - 1; s >= 0; --s) gprobs[t * M + A->idx[t * k + s]] += gdenom[t];
        /* softmax backward (graph.hpp:172-183) */
        for (int64_t t = 0; t < T; ++t) {
            const float* p = A->probs + t * M;
            const float* gy = gprobs + t * M;
            float dot = 0.f;
            for (int32_t j = 0; j < M; ++j) dot += gy[j] * p[j];
            for (int32_t j = 0; j < M; ++j) glog[t * M + j] += p[j] * (gy[j] - dot);
        }
        /* router matmul backward */
        mm_nt_acc(glog, R, gnormed, T, M, d);
        mm_tn_acc(A->normed, glog, G + oracle_off_router(c, l), T, d, M);
        /* rmsnorm backward */
        rmsnorm_bwd_acc(A->h, gain, gnormed, gh_l, G + oracle_off_norm(c, l), T, d, eps);
        if (tr && tr->grad_h) memcpy(tr->grad_h + (int64_t)l * T * d, gh_l, (size_t)(T * d) * 4);
        free(gprobs); free(glog); free(gnormed); free(gdenom);
        free(gh);
        gh = gh_l;
    }
    /* embedding: gather_rows backward, rows ascending (graph.hpp:220-229) */
    {
        float* Ge = G + oracle_off_emb(c);
        for (int64_t t = 0; t < T; ++t) {
            float* dst = Ge + (int64_t)inputs[t] * d;
            for (int64_t q = 0; q < d; ++q) dst[q] += gh[t * d + q];
        }
    }
    free(gh);
    /* frozen expert blocks never get a gradient (graph.hpp:56-63): already zero */
    for (int32_t l = 0; l < L; ++l) {
        layer_act* A = &la[l];
        for (int32_t j = 0; j < M; ++j) {
            expert_act* E = &A->ex[j];
            free(E->rows); free(E->gp); free(E->gate); free(E->up); free(E->hm); free(E->y);
        }
        free(A->ex);
        if (l > 0) free(A->h);
        free(A->normed); free(A->logits); free(A->probs); free(A->idx); free(A->lse_r);
        free(A->denom);
    }
    free(la[0].h);
    free(la);
    free(inputs);
    free(targets);
    return 0;
}

/* ---------------- MaskedAdamW::step (trainer.hpp:68-94) ---------------- */

static void adamw_range(float* theta, const float* g, float* m, float* v, int64_t n, float lr,
                        float b1, float b2, float eps, float wd, float bc1, float bc2) {
    for (int64_t i = 0; i < n; ++i) {
        float gi = g[i];
        m[i] = b1 * m[i] + (1.f - b1) * gi;
        v[i] = b2 * v[i] + (1.f - b2) * gi * gi;
        float mhat = m[i] / bc1;
        float vhat = v[i] / bc2;
        theta[i] -= lr * (mhat / (sqrtf(vhat) + eps) + wd * theta[i]);
    }
}

void oracle_adamw_step(const spes_model_cfg* c, float* P, const float* G, float* m, float* v,
                       const uint8_t* trainable_expert, const spes_adamw_cfg* o, int64_t step) {
    float bc1 = 1.f - (float)pow(o->beta1, (double)step);
    float bc2 = 1.f - (float)pow(o->beta2, (double)step);
    const float lr = (float)o->lr, b1 = (float)o->beta1, b2 = (float)o->beta2,
                eps = (float)o->eps, wd = (float)o->weight_decay;
    int64_t eb = expert_base(c);
    adamw_range(P, G, m, v, eb, lr, b1, b2, eps, wd, bc1, bc2); /* all shared blocks */
    const int64_t per = 3 * c->hidden * c->intermediate;
    for (int32_t l = 0; l < c->layers; ++l)
        for (int32_t j = 0; j < c->experts_total; ++j) {
            if (!trainable_expert[j]) continue;
            int64_t o0 = oracle_off_expert(c, l, j);
            adamw_range(P + o0, G + o0, m + o0, v + o0, per, lr, b1, b2, eps, wd, bc1, bc2);
        }
}

/* Flat-array form of the same element update (for kernel-level parity). */
void oracle_adamw_array(float* theta, const float* g, float* m, float* v, int64_t n,
                        const spes_adamw_cfg* o, int64_t step) {
    float bc1 = 1.f - (float)pow(o->beta1, (double)step);
    float bc2 = 1.f - (float)pow(o->beta2, (double)step);
    adamw_range(theta, g, m, v, n, (float)o->lr, (float)o->beta1, (float)o->beta2, (float)o->eps,
                (float)o->weight_decay, bc1, bc2);
}

/* ---------------- local_round (trainer.hpp:143-222), AdamW, fresh state ---------------- */

int oracle_local_round(const spes_model_cfg* c, float* P, const int32_t* tokens, int64_t B,
                       int64_t S, int32_t H, const double* lr, const spes_adamw_cfg* opt,
                       const uint8_t* trainable_expert, double* losses) {
    const int64_t NP = oracle_param_count(c);
    float* G = (float*)malloc((size_t)NP * 4);
    float* m = (float*)calloc((size_t)NP, 4);
    float* v = (float*)calloc((size_t)NP, 4);
    int rc = 0;
    for (int32_t h = 0; h < H; ++h) {
        rc = oracle_forward_backward(c, P, tokens + (int64_t)h * B * (S + 1), B, S,
                                     trainable_expert, G, losses + 5 * h, NULL);
        if (rc) break;
        if (!isfinite(losses[5 * h])) { /* trainer.hpp:166-167 */
            rc = 3 + h;
            break;
        }
        spes_adamw_cfg o = *opt;
        o.lr = lr ? lr[h] : opt->lr;
        oracle_adamw_step(c, P, G, m, v, trainable_expert, &o, h + 1);
    }
    free(G);
    free(m);
    free(v);
    return rc;
}

/* ---------------- OuterOptimizer::step (trainer.hpp:228-266), DiLoCo baseline ----------------
 * theta <- OuterOpt(theta, mean_i(local_i - theta)) per element in fp64: delta accumulates
 * (local_i - theta) * (1/N) over the locals in order; SGD: theta = float(theta + lr*delta);
 * Nesterov: g = -delta, b = momentum*b + g, theta = float(theta - lr*(g + momentum*b)).
 * buf (n doubles, zero before the first step) is the Nesterov state; locals is N x n. */
void oracle_outer_step(int32_t kind, double lr, double momentum, float* theta,
                       const float* locals, int32_t N, int64_t n, double* buf) {
    const double inv_n = 1.0 / (double)N;
    for (int64_t j = 0; j < n; ++j) {
        double delta = 0.0;
        for (int32_t i = 0; i < N; ++i)
            delta += ((double)locals[(int64_t)i * n + j] - (double)theta[j]) * inv_n;
        if (kind == 0) {
            theta[j] = (float)((double)theta[j] + lr * delta);
        } else {
            const double g = -delta;
            buf[j] = momentum * buf[j] + g;
            theta[j] = (float)((double)theta[j] - lr * (g + momentum * buf[j]));
        }
    }
}

/* ---------------- Server::aggregate (protocol.cpp:197-251), owner-set form ---------------- */

void oracle_aggregate(const spes_model_cfg* c, int32_t N, const float* node_params,
                      const int32_t* node_offsets, const int32_t* experts,
                      const float* global_in, float* global_out) {
    const int64_t NP = oracle_param_count(c);
    const int64_t eb = expert_base(c);
    memcpy(global_out, global_in, (size_t)NP * 4);
    /* psi: acc(double) += x_n in node-id order; float(acc * (1.0/N)) (protocol.cpp:238-243) */
    double inv_n = 1.0 / (double)N;
    for (int64_t i = 0; i < eb; ++i) {
        double acc = 0.0;
        for (int32_t n = 0; n < N; ++n) acc += (double)node_params[(int64_t)n * NP + i];
        global_out[i] = (float)(acc * inv_n);
    }
    /* experts: mean over owners in ascending node id (r = 1: verbatim, protocol.cpp:229-236) */
    const int32_t M = c->experts_total;
    const int64_t per = 3 * c->hidden * c->intermediate;
    int32_t* own = (int32_t*)malloc((size_t)N * sizeof(int32_t));
    for (int32_t j = 0; j < M; ++j) {
        int32_t no = 0;
        for (int32_t n = 0; n < N; ++n)
            for (int32_t q = node_offsets[n]; q < node_offsets[n + 1]; ++q)
                if (experts[q] == j) own[no++] = n;
        if (no == 0) continue;
        double inv_o = 1.0 / (double)no;
        for (int32_t l = 0; l < c->layers; ++l) {
            int64_t o0 = oracle_off_expert(c, l, j);
            for (int64_t i = 0; i < per; ++i) {
                double acc = 0.0;
                for (int32_t q = 0; q < no; ++q) acc += (double)node_params[(int64_t)own[q] * NP + o0 + i];
                global_out[o0 + i] = (float)(acc * inv_o);
            }
        }
    }
    free(own);
}

/* ---------------- merging (merging.hpp) ---------------- */

static double* projection(const spes_model_cfg* c, const float* P, int l, int j, int32_t src,
                          int64_t* len) {
    const int64_t df = c->hidden * c->intermediate;
    const float* wg = P + oracle_off_expert(c, l, j);
    const float* wu = wg + df;
    int64_t n = (src == 2) ? 2 * df : df;
    double* w = (double*)malloc((size_t)n * sizeof(double));
    int64_t q = 0;
    if (src == 0 || src == 2)
        for (int64_t i = 0; i < df; ++i) w[q++] = (double)wg[i];
    if (src == 1 || src == 2)
        for (int64_t i = 0; i < df; ++i) w[q++] = (double)wu[i];
    *len = n;
    return w;
}

/* similarity_matrix (merging.hpp:55-82) */
void oracle_similarity(const spes_model_cfg* c, const float* P, int32_t l, int32_t src,
                       double* sim) {
    const int32_t M = c->experts_total;
    double** w = (double**)malloc((size_t)M * sizeof(double*));
    double* norm = (double*)malloc((size_t)M * sizeof(double));
    int64_t len = 0;
    for (int32_t j = 0; j < M; ++j) {
        w[j] = projection(c, P, l, j, src, &len);
        double n2 = 0.0;
        for (int64_t i = 0; i < len; ++i) n2 += w[j][i] * w[j][i];
        norm[j] = sqrt(n2);
    }
#pragma omp parallel for schedule(dynamic)
    for (int32_t j = 0; j < M; ++j)
        for (int32_t k = j; k < M; ++k) {
            double v = 0.0;
            if (norm[j] > 0.0 && norm[k] > 0.0) {
                double dot = 0.0;
                for (int64_t i = 0; i < len; ++i) dot += w[j][i] * w[k][i];
                v = dot / (norm[j] * norm[k]);
            }
            sim[(int64_t)j * M + k] = v;
            sim[(int64_t)k * M + j] = v;
        }
    for (int32_t j = 0; j < M; ++j) free(w[j]);
    free(w);
    free(norm);
}

/* select_peers (merging.hpp:85-95) */
int32_t oracle_select_peers(const double* sim, int32_t M, int32_t j, int32_t K, int32_t* peers) {
    int32_t idx[1024];
    int32_t n = 0;
    for (int32_t i = 0; i < M; ++i)
        if (i != j) idx[n++] = i;
    for (int32_t i = 1; i < n; ++i) { /* stable: insert after equal keys */
        int32_t v = idx[i];
        int32_t q = i - 1;
        while (q >= 0 && sim[(int64_t)j * M + v] > sim[(int64_t)j * M + idx[q]]) {
            idx[q + 1] = idx[q];
            --q;
        }
        idx[q + 1] = v;
    }
    if (n > K) n = K;
    for (int32_t i = 1; i < n; ++i) {
        int32_t v = idx[i];
        int32_t q = i - 1;
        while (q >= 0 && idx[q] > v) {
            idx[q + 1] = idx[q];
            --q;
        }
        idx[q + 1] = v;
    }
    for (int32_t i = 0; i < n; ++i) peers[i] = idx[i];
    return n;
}

static int merge_at(const spes_merge_sched* s, int32_t round) {
    return s->warmup_rounds > 0 && round < s->warmup_rounds && s->interval > 0 &&
           round % s->interval == 0;
}

static double alpha_at(const spes_merge_sched* s, int32_t round) {
    if (s->warmup_rounds <= 0) return 0.0;
    double frac = 1.0 - (double)round / (double)s->warmup_rounds;
    return s->alpha0 * (frac > 0.0 ? frac : 0.0);
}

/* merge_experts + merge_model (merging.hpp:106-150) */
int32_t oracle_merge_model(const spes_model_cfg* c, float* P, const spes_merge_sched* s,
                           int32_t round, spes_merge_event* events, int32_t* peers_out) {
    if (!merge_at(s, round)) return 0;
    double alpha = alpha_at(s, round);
    if (alpha <= 0.0) return 0;
    const int32_t M = c->experts_total;
    const int64_t df = c->hidden * c->intermediate;
    const int64_t per = 3 * df;
    int32_t K = s->peers < M - 1 ? s->peers : M - 1;
    double* sim = (double*)malloc((size_t)M * M * sizeof(double));
    float* snap = (float*)malloc((size_t)(M * per) * 4);
    int32_t* peers = (int32_t*)malloc((size_t)M * (K > 0 ? K : 1) * sizeof(int32_t));
    for (int32_t l = 0; l < c->layers; ++l) {
        oracle_similarity(c, P, l, s->source, sim);
        for (int32_t j = 0; j < M; ++j)
            memcpy(snap + (int64_t)j * per, P + oracle_off_expert(c, l, j), (size_t)per * 4);
        double disp = 0.0;
        int32_t nk = 0;
        for (int32_t j = 0; j < M; ++j) {
            nk = oracle_select_peers(sim, M, j, K, peers + (int64_t)j * K);
            double coef = alpha / (double)nk;
            float* dst = P + oracle_off_expert(c, l, j);
            const float* self = snap + (int64_t)j * per;
            for (int64_t i = 0; i < per; ++i) { /* wg, wu, wd back to back */
                double acc = 0.0;
                for (int32_t q = 0; q < nk; ++q)
                    acc += (double)snap[(int64_t)peers[j * K + q] * per + i] - (double)self[i];
                double delta = coef * acc;
                disp += delta * delta;
                dst[i] = (float)((double)self[i] + delta);
            }
        }
        if (events) {
            events[l].layer = l;
            events[l].peers_k = nk;
            events[l].alpha = alpha;
            events[l].displacement_sq = disp;
        }
        if (peers_out) memcpy(peers_out + (int64_t)l * M * K, peers, (size_t)M * K * sizeof(int32_t));
    }
    free(sim);
    free(snap);
    free(peers);
    return c->layers;
}

/* ---------------- misc ---------------- */

/* LrSchedule::at (experiment.cpp:32-41) */
double oracle_lr_at(double peak, double min_frac, int64_t warmup, int64_t total, int64_t step) {
    if (warmup > 0 && step < warmup) return peak * (double)(step + 1) / (double)warmup;
    double lo = peak * min_frac;
    int64_t span = total - warmup;
    if (span <= 0) return peak;
    double progress = (double)(step - warmup) / (double)span;
    progress = progress < 0.0 ? 0.0 : (progress > 1.0 ? 1.0 : progress);
    return lo + (peak - lo) * 0.5 * (1.0 + cos(M_PI * progress));
}

/* param_partition (model.hpp:466-477) */
void oracle_param_partition(int32_t M, int32_t N, int32_t* node_offsets, int32_t* experts) {
    int32_t base = M / N, extra = M % N, next = 0;
    node_offsets[0] = 0;
    for (int32_t i = 0; i < N; ++i) {
        int32_t take = base + (i < extra ? 1 : 0);
        for (int32_t j = 0; j < take; ++j) experts[next] = next, ++next;
        node_offsets[i + 1] = next;
    }
}

void oracle_expf_array(const float* x, float* y, int64_t n) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) y[i] = expf(x[i]);
}

int64_t oracle_expf_mismatches(const float* x, const float* y, int64_t n) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t i = 0; i < n; ++i) {
        float e = expf(x[i]);
        if (memcmp(&e, &y[i], 4) != 0) ++bad;
    }
    return bad;
}

int64_t oracle_expf_range_mismatches(uint32_t lo, uint32_t hi, const float* y) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t b = (int64_t)lo; b <= (int64_t)hi; ++b) {
        uint32_t bits = (uint32_t)b;
        float x;
        memcpy(&x, &bits, 4);
        float e = expf(x);
        if (memcmp(&e, &y[b - lo], 4) != 0) ++bad;
    }
    return bad;
}

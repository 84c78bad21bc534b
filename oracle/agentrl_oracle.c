/*
 * agentrl_oracle.c -- plain, slow, fp64 CPU ORACLE for the AgentRL hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2510_04206_b200/csrc); neither side includes or links the other.
 *
 * What it computes (PAPER.md = arxiv 2510.04206 LaTeX source):
 *   step 1  validate                       -- DESIGN.md readings R14, R16
 *   step 2  counts n_g, K_j                -- token set of Eq.1, P:548-569 (sec 3.2)
 *   step 3  GRPO group advantage           -- P:1263 (App. B.2 GRPO objective),
 *                                             P:1121-1125 (App. A Eq. for A_i)
 *   step 4  per-task token mean / std      -- P:572-578 (sec 3.2 Eq.1)
 *   step 5  apply Eq.1 and broadcast       -- P:572-576
 *   step 6  token log-prob via the LM head -- P:1182-1190 (App. B.1 factorisation)
 *           PPO-clip term, token-level mean -- P:1230-1241 (App. B.2 PPO objective),
 *                                             P:1132-1141 (DAPO token-level 1/sum|o|,
 *                                             decoupled eps_low/eps_high)
 *   step 7  exact gradients of step 6 w.r.t. hidden and W_head (derivative of
 *           the above; no paper passage spells it out -- see DESIGN.md R10).
 *
 * Every floating-point quantity is fp64.  Inputs hidden / W_head are given as
 * doubles (the caller passes the bf16-rounded values, which fp64 holds exactly).
 * Sums are plain left-to-right loops; the only parallelism (OpenMP) is across
 * independent outputs (tokens or vocabulary rows), which changes no summation
 * order.  Two-pass mean/variance everywhere.
 *
 * Readings of silent / ambiguous points are numbered R1..R18 in DESIGN.md and
 * quoted at the line that applies them.
 *
 * Parity pins: see tests/test_oracle_*.py.  Parity unpinned: none of the
 * functions below is without a pin, but readings R1, R3, R5, R7 and R12 are
 * conventions (SPEC / north_star), not paper values -- DESIGN.md lists them.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_ERR_ARG (-1)

/* data-dependent status bits (same meaning as the product's device word, but
 * defined here independently, from DESIGN.md's table) */
#define ORS_BAD_TARGET 1
#define ORS_NONFINITE 2
#define ORS_BAD_OFFSETS 4
#define ORS_GROUP_SPANS_TASKS 8
#define ORS_GROUP_TOO_SMALL 16
#define ORS_NO_TOKENS 32

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------------ */
/* Step 1: validation (R14 group size >= 2 per SPEC S:140; R16 empty batch)  */
/* ------------------------------------------------------------------------ */
int oracle_validate(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks,
                    const int64_t* traj_offsets, const int32_t* task_id,
                    const int32_t* group_id) {
    int status = 0;
    if (traj_offsets[0] != 0 || traj_offsets[n_traj] != T) status |= ORS_BAD_OFFSETS;
    for (int32_t g = 0; g < n_traj; ++g)
        if (traj_offsets[g + 1] < traj_offsets[g]) status |= ORS_BAD_OFFSETS;
    int32_t* grp_task = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_groups > 0 ? n_groups : 1));
    int32_t* grp_size = (int32_t*)calloc((size_t)(n_groups > 0 ? n_groups : 1), sizeof(int32_t));
    for (int32_t j = 0; j < n_groups; ++j) grp_task[j] = -1;
    for (int32_t g = 0; g < n_traj; ++g) {
        int32_t j = group_id[g];
        if (j < 0 || j >= n_groups || task_id[g] < 0 || task_id[g] >= n_tasks) {
            status |= ORS_GROUP_SPANS_TASKS;
            continue;
        }
        grp_size[j] += 1;
        if (grp_task[j] < 0) grp_task[j] = task_id[g];
        else if (grp_task[j] != task_id[g]) status |= ORS_GROUP_SPANS_TASKS;
    }
    for (int32_t j = 0; j < n_groups; ++j)
        if (grp_size[j] == 1) status |= ORS_GROUP_TOO_SMALL;
    free(grp_task);
    free(grp_size);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Step 2: counts.  n_g = number of loss-masked (assistant) tokens of       */
/* trajectory g: the tokens y_{t,k} of actions a_t, k <= L_t.   */
/* R4: only mask != 0 tokens are action tokens; R18: any nonzero byte = 1.  */
/* ------------------------------------------------------------------------ */
void oracle_counts(int32_t n_traj, int32_t n_groups, const int64_t* traj_offsets,
                   const int32_t* group_id, const uint8_t* loss_mask,
                   int64_t* n_g /*[n_traj]*/, int32_t* K_j /*[n_groups]*/) {
    for (int32_t g = 0; g < n_traj; ++g) {
        int64_t c = 0;
        for (int64_t t = traj_offsets[g]; t < traj_offsets[g + 1]; ++t)
            if (loss_mask[t] != 0) c += 1;
        n_g[g] = c;
    }
    for (int32_t j = 0; j < n_groups; ++j) K_j[j] = 0;
    for (int32_t g = 0; g < n_traj; ++g) K_j[group_id[g]] += 1;
}

/* ------------------------------------------------------------------------ */
/* Step 3: GRPO group-relative advantage:                            */
/*   A_hat_{i,j,g} = (R_{i,j,g} - mean(R_{i,j})) / std(R_{i,j})              */
/* R1: population std (divide by K).  R2: if every reward of the group is    */
/* exactly equal, A_hat = 0 exactly; otherwise the denominator is            */
/* max(std, eps).  Two-pass mean, then variance.                */
/* ------------------------------------------------------------------------ */
void oracle_group_advantage(int32_t n_traj, int32_t n_groups, const int32_t* group_id,
                            const float* rewards, double eps_std,
                            double* adv_hat /*[n_traj]*/) {
    for (int32_t j = 0; j < n_groups; ++j) {
        double K = 0.0, sum = 0.0;
        int have = 0;
        double rmax = 0.0, rmin = 0.0;
        for (int32_t g = 0; g < n_traj; ++g) {
            if (group_id[g] != j) continue;
            double r = (double)rewards[g];
            if (!have) { rmax = r; rmin = r; have = 1; }
            if (r > rmax) rmax = r;
            if (r < rmin) rmin = r;
            K += 1.0;
            sum += r;
        }
        if (!have) continue;
        if (rmax == rmin) { /* R2: all-equal group -> exactly zero */
            for (int32_t g = 0; g < n_traj; ++g)
                if (group_id[g] == j) adv_hat[g] = 0.0;
            continue;
        }
        double mean = sum / K;
        double ss = 0.0;
        for (int32_t g = 0; g < n_traj; ++g)
            if (group_id[g] == j) {
                double dlt = (double)rewards[g] - mean;
                ss += dlt * dlt;
            }
        double sd = sqrt(ss / K); /* R1 population */
        double den = sd > eps_std ? sd : eps_std;
        for (int32_t g = 0; g < n_traj; ++g)
            if (group_id[g] == j) adv_hat[g] = ((double)rewards[g] - mean) / den;
    }
}

/* ------------------------------------------------------------------------ */
/* Step 4: per-task moments of the token-level advantage set A_i^tok        */
/* (P:557-569): every masked token of trajectory g carries A_hat_g, so       */
/*   N_i  = sum_{g in i} n_g                                                 */
/*   mu_i = mean(A_i^tok)  = sum_{g in i} n_g A_hat_g / N_i     */
/*   sig_i = std(A_i^tok)  = sqrt(sum n_g (A_hat_g - mu_i)^2 / N_i)  */
/* R1 population std; R5 each token counts once; R6 "batch" = the global     */
/* batch (the caller passes the whole batch); R16 N_i = 0 -> (0,0,0).        */
/* ------------------------------------------------------------------------ */
void oracle_task_moments(int32_t n_traj, int32_t n_tasks, const int32_t* task_id,
                         const int64_t* n_g, const double* adv_hat,
                         double* task_stats /*[n_tasks*3]: N_i, mu_i, sigma_i*/) {
    for (int32_t i = 0; i < n_tasks; ++i) {
        double N = 0.0, S = 0.0;
        for (int32_t g = 0; g < n_traj; ++g)
            if (task_id[g] == i) {
                N += (double)n_g[g];
                S += (double)n_g[g] * adv_hat[g];
            }
        if (N == 0.0) {
            task_stats[3 * i + 0] = 0.0;
            task_stats[3 * i + 1] = 0.0;
            task_stats[3 * i + 2] = 0.0;
            continue;
        }
        double mu = S / N;
        double Q = 0.0;
        for (int32_t g = 0; g < n_traj; ++g)
            if (task_id[g] == i) {
                double dlt = adv_hat[g] - mu;
                Q += (double)n_g[g] * dlt * dlt;
            }
        task_stats[3 * i + 0] = N;
        task_stats[3 * i + 1] = mu;
        task_stats[3 * i + 2] = sqrt(Q / N);
    }
}

/* ------------------------------------------------------------------------ */
/* Step 5: Eq.1:  A_tilde = (A_hat - mu_i) / sigma_i, with the   */
/* denominator floored at eps (R2), broadcast to the masked tokens (R4).     */
/* Also the stable compaction list of masked token positions.               */
/* ------------------------------------------------------------------------ */
void oracle_apply(int64_t T, int32_t n_traj, const int64_t* traj_offsets,
                  const int32_t* task_id, const uint8_t* loss_mask, const double* adv_hat,
                  const double* task_stats, double eps_std,
                  double* adv_tilde /*[n_traj]*/, double* adv_tok /*[T]*/,
                  int64_t* idx /*[T] (first n_mask used) or NULL*/, int64_t* n_mask) {
    for (int32_t g = 0; g < n_traj; ++g) {
        int32_t i = task_id[g];
        double mu = task_stats[3 * i + 1], sd = task_stats[3 * i + 2];
        double den = sd > eps_std ? sd : eps_std;
        adv_tilde[g] = (adv_hat[g] - mu) / den;
    }
    int64_t m = 0;
    for (int32_t g = 0; g < n_traj; ++g)
        for (int64_t t = traj_offsets[g]; t < traj_offsets[g + 1]; ++t) {
            if (loss_mask[t] != 0) {
                adv_tok[t] = adv_tilde[g];
                if (idx) idx[m] = t;
                m += 1;
            } else {
                adv_tok[t] = 0.0;
            }
        }
    (void)T;
    *n_mask = m;
}

/* Steps 1-5 in the paper's order (R3: group -> broadcast -> task). */
int oracle_task_adv_norm(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks,
                         const int64_t* traj_offsets, const int32_t* task_id,
                         const int32_t* group_id, const float* rewards,
                         const uint8_t* loss_mask, double eps_std,
                         /* outputs */
                         int64_t* n_g, int32_t* K_j, double* adv_hat, double* adv_tilde,
                         double* task_stats, double* adv_tok, int64_t* idx,
                         int64_t* n_mask) {
    if (T < 0 || n_traj < 0 || n_groups < 0 || n_tasks <= 0 || !(eps_std > 0.0))
        return OR_ERR_ARG;
    int status = oracle_validate(T, n_traj, n_groups, n_tasks, traj_offsets, task_id, group_id);
    if (status & (ORS_BAD_OFFSETS | ORS_GROUP_SPANS_TASKS)) return status;
    oracle_counts(n_traj, n_groups, traj_offsets, group_id, loss_mask, n_g, K_j);
    oracle_group_advantage(n_traj, n_groups, group_id, rewards, eps_std, adv_hat);
    oracle_task_moments(n_traj, n_tasks, task_id, n_g, adv_hat, task_stats);
    oracle_apply(T, n_traj, traj_offsets, task_id, loss_mask, adv_hat, task_stats, eps_std,
                 adv_tilde, adv_tok, idx, n_mask);
    if (*n_mask == 0) status |= ORS_NO_TOKENS;
    return status;
}

/* ------------------------------------------------------------------------ */
/* Step 6: one token's logits, log-prob and PPO-clip term.                  */
/*   z_v   = s * sum_k h_k W_{v,k}                  (LM head;   */
/*                                                    s = logit_scale, R12)  */
/*   lse   = m + log sum_v exp(z_v - m),  m = max_v z_v                      */
/*   logp  = z_y - lse                  (token log-prob)        */
/*   rho   = exp(logp - old_logp)       (ratio)                 */
/*   term  = min(rho*A, clip(rho, 1-eps_lo, 1+eps_hi)*A)  (P:1230-1233,      */
/*                                                    P:1141 decoupled eps)  */
/*   c     = clipped ? 0 : rho*A/N      (d(-term/N)/dlogp = -c; R10)          */
/* ------------------------------------------------------------------------ */
typedef struct {
    double lse, logp, rho, term, coef;
    int clipped;
} oracle_token_t;

static void token_logits(int32_t d, int32_t V, const double* h, const double* W, double s,
                         double* z /*[V]*/) {
    for (int32_t v = 0; v < V; ++v) {
        double acc = 0.0;
        const double* w = W + (size_t)v * (size_t)d;
        for (int32_t k = 0; k < d; ++k) acc += h[k] * w[k];
        z[v] = s * acc;
    }
}

static oracle_token_t token_loss(int32_t V, const double* z, int32_t y, double A, double old,
                                 double eps_lo, double eps_hi, double N) {
    oracle_token_t r;
    double m = z[0];
    for (int32_t v = 1; v < V; ++v)
        if (z[v] > m) m = z[v];
    double se = 0.0;
    for (int32_t v = 0; v < V; ++v) se += exp(z[v] - m);
    r.lse = m + log(se);
    r.logp = z[y] - r.lse;
    r.rho = exp(r.logp - old);
    double lo = 1.0 - eps_lo, hi = 1.0 + eps_hi;
    double rc = r.rho < lo ? lo : (r.rho > hi ? hi : r.rho);
    double u = r.rho * A, c = rc * A;
    r.term = u < c ? u : c;
    /* R10: the gradient is zero only where the clip is strictly active. */
    r.clipped = (A > 0.0 && r.rho > hi) || (A < 0.0 && r.rho < lo);
    r.coef = r.clipped ? 0.0 : r.rho * A / N;
    return r;
}

/*
 * Full loss + gradients over all masked tokens (step 6 + step 7).
 *   loss       = -(1/N) sum_{t masked} term_t               (R7, R8)
 *   G_{t,v}    = c_t (p_{t,v} - [v = y_t]),  p = exp(z - lse)
 *   grad_h_t   = s * sum_v G_{t,v} W_v                      (0 on unmasked rows)
 *   grad_W_v   = s * sum_t G_{t,v} h_t
 * N = n_mask_global (the global masked-token count, R6).  Tokens are taken in
 * blocks of 64 so that the G block stays small (an allocation choice: each
 * sum above is still accumulated in plain index order).
 * Returns the status bits (ORS_BAD_TARGET / ORS_NONFINITE / ORS_NO_TOKENS).
 */
int oracle_policy_loss_fwd_bwd(int64_t T, int32_t d, int32_t V, const double* hidden,
                               const double* W, const int32_t* target, const double* adv_tok,
                               const double* old_logp, const uint8_t* loss_mask,
                               double eps_lo, double eps_hi, double logit_scale,
                               int64_t n_mask_global,
                               /* outputs (any may be NULL except loss) */
                               double* loss, double* logp_out /*[T]*/,
                               double* grad_hidden /*[T*d]*/, double* grad_W /*[V*d]*/,
                               double* loss_stats /*[4]*/) {
    if (T < 0 || d <= 0 || V <= 0 || eps_lo < 0 || eps_lo >= 1 || eps_hi < 0 ||
        !(logit_scale > 0))
        return OR_ERR_ARG;
    int status = 0;
    for (int64_t t = 0; t < T; ++t)
        if (loss_mask[t] && (target[t] < 0 || target[t] >= V)) status |= ORS_BAD_TARGET;
    if (status) return status;
    const double s = logit_scale;
    const double N = (double)n_mask_global;
    if (grad_hidden) memset(grad_hidden, 0, sizeof(double) * (size_t)T * (size_t)d);
    if (grad_W) memset(grad_W, 0, sizeof(double) * (size_t)V * (size_t)d);
    if (logp_out)
        for (int64_t t = 0; t < T; ++t) logp_out[t] = 0.0;
    *loss = 0.0;
    if (loss_stats) memset(loss_stats, 0, 4 * sizeof(double));
    if (n_mask_global <= 0) return ORS_NO_TOKENS;

    /* masked token list in stream order */
    int64_t nm = 0;
    for (int64_t t = 0; t < T; ++t) nm += loss_mask[t] != 0;
    int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nm > 0 ? nm : 1));
    nm = 0;
    for (int64_t t = 0; t < T; ++t)
        if (loss_mask[t]) rows[nm++] = t;

    const int64_t B = 64;
    double* Gb = (double*)malloc(sizeof(double) * (size_t)B * (size_t)V);
    oracle_token_t* tok = (oracle_token_t*)malloc(sizeof(oracle_token_t) * (size_t)B);
    double loss_acc = 0.0, n_clip = 0.0, sum_rho = 0.0, sum_logp = 0.0;

    for (int64_t b0 = 0; b0 < nm; b0 += B) {
        int64_t nb = nm - b0 < B ? nm - b0 : B;
        /* forward + G rows for this block of tokens (independent per token) */
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t q = 0; q < nb; ++q) {
            int64_t t = rows[b0 + q];
            double* z = Gb + (size_t)q * (size_t)V;
            token_logits(d, V, hidden + (size_t)t * (size_t)d, W, s, z);
            tok[q] = token_loss(V, z, target[t], adv_tok[t], old_logp[t], eps_lo, eps_hi, N);
            /* z -> G in place: G = c (exp(z - lse) - onehot) */
            double c = tok[q].coef, lse = tok[q].lse;
            for (int32_t v = 0; v < V; ++v) z[v] = c * exp(z[v] - lse);
            z[target[t]] -= c;
        }
        for (int64_t q = 0; q < nb; ++q) {
            int64_t t = rows[b0 + q];
            loss_acc += tok[q].term;
            n_clip += tok[q].clipped ? 1.0 : 0.0;
            sum_rho += tok[q].rho;
            sum_logp += tok[q].logp;
            if (logp_out) logp_out[t] = tok[q].logp;
        }
        /* grad_hidden rows: s * sum_v G_tv W_v */
        if (grad_hidden) {
#pragma omp parallel for schedule(dynamic, 1)
            for (int64_t q = 0; q < nb; ++q) {
                int64_t t = rows[b0 + q];
                double* gh = grad_hidden + (size_t)t * (size_t)d;
                const double* G = Gb + (size_t)q * (size_t)V;
                for (int32_t v = 0; v < V; ++v) {
                    double gv = G[v];
                    const double* w = W + (size_t)v * (size_t)d;
                    for (int32_t k = 0; k < d; ++k) gh[k] += gv * w[k];
                }
                for (int32_t k = 0; k < d; ++k) gh[k] *= s;
            }
        }
        /* grad_W rows: accumulate s * G_tv h_t over tokens in stream order */
        if (grad_W) {
#pragma omp parallel for schedule(static)
            for (int32_t v = 0; v < V; ++v) {
                double* gw = grad_W + (size_t)v * (size_t)d;
                for (int64_t q = 0; q < nb; ++q) {
                    double gv = s * Gb[(size_t)q * (size_t)V + (size_t)v];
                    const double* h = hidden + (size_t)rows[b0 + q] * (size_t)d;
                    for (int32_t k = 0; k < d; ++k) gw[k] += gv * h[k];
                }
            }
        }
    }
    *loss = -loss_acc / N;
    if (!isfinite(*loss)) status |= ORS_NONFINITE;
    if (loss_stats && nm > 0) {
        loss_stats[0] = n_clip / (double)nm;
        loss_stats[1] = sum_rho / (double)nm;
        loss_stats[2] = sum_logp / (double)nm;
        loss_stats[3] = (double)nm;
    }
    free(rows);
    free(Gb);
    free(tok);
    return status;
}

/*
 * Per-token spot rows (for full-size parity): for each listed token t (masked
 * or not) return lse, logp, rho, term, coef, clipped, and optionally the
 * grad_hidden row.  Each needs only its own hidden row plus N and A_t.
 * Same arithmetic as oracle_policy_loss_fwd_bwd, restricted to those rows.
 * out_row[6*q + {0..5}] = lse, logp, rho, term, coef, clipped.
 */
int oracle_policy_loss_rows(int32_t d, int32_t V, const double* hidden_rows /*[n,d]*/,
                            const double* W, const int32_t* target_rows,
                            const double* adv_rows, const double* old_rows, int64_t n_rows,
                            double eps_lo, double eps_hi, double logit_scale,
                            int64_t n_mask_global, double* out_row /*[n*6]*/,
                            double* grad_hidden_rows /*[n*d] or NULL*/) {
    if (d <= 0 || V <= 0 || !(logit_scale > 0) || n_mask_global <= 0) return OR_ERR_ARG;
    const double s = logit_scale, N = (double)n_mask_global;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < n_rows; ++q) {
        double* z = (double*)malloc(sizeof(double) * (size_t)V);
        const double* h = hidden_rows + (size_t)q * (size_t)d;
        token_logits(d, V, h, W, s, z);
        oracle_token_t r = token_loss(V, z, target_rows[q], adv_rows[q], old_rows[q], eps_lo,
                                      eps_hi, N);
        out_row[6 * q + 0] = r.lse;
        out_row[6 * q + 1] = r.logp;
        out_row[6 * q + 2] = r.rho;
        out_row[6 * q + 3] = r.term;
        out_row[6 * q + 4] = r.coef;
        out_row[6 * q + 5] = (double)r.clipped;
        if (grad_hidden_rows) {
            double* gh = grad_hidden_rows + (size_t)q * (size_t)d;
            for (int32_t k = 0; k < d; ++k) gh[k] = 0.0;
            for (int32_t v = 0; v < V; ++v) {
                double gv = r.coef * (exp(z[v] - r.lse) - (v == target_rows[q] ? 1.0 : 0.0));
                const double* w = W + (size_t)v * (size_t)d;
                for (int32_t k = 0; k < d; ++k) gh[k] += gv * w[k];
            }
            for (int32_t k = 0; k < d; ++k) gh[k] *= s;
        }
        free(z);
    }
    return 0;
}

/*
 * Forward-only log-probs (logp_t = z_{y_t} - lse_t) for every masked token;
 * unmasked tokens get 0.  Used by tests to build behaviour log-probs
 * old_logp = logp + delta (DESIGN.md input recipe) without touching the GPU.
 */
int oracle_logprob(int64_t T, int32_t d, int32_t V, const double* hidden, const double* W,
                   const int32_t* target, const uint8_t* loss_mask, double logit_scale,
                   double* logp_out /*[T]*/) {
    if (T < 0 || d <= 0 || V <= 0 || !(logit_scale > 0)) return OR_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < T; ++t) {
        if (!loss_mask[t]) { logp_out[t] = 0.0; continue; }
        double* z = (double*)malloc(sizeof(double) * (size_t)V);
        token_logits(d, V, hidden + (size_t)t * (size_t)d, W, logit_scale, z);
        double m = z[0];
        for (int32_t v = 1; v < V; ++v)
            if (z[v] > m) m = z[v];
        double se = 0.0;
        for (int32_t v = 0; v < V; ++v) se += exp(z[v] - m);
        logp_out[t] = z[target[t]] - (m + log(se));
        free(z);
    }
    return 0;
}

/*
 * Fused step (steps 1-7): task advantage normalization followed by the loss,
 * with A_t = A_tilde of the token's trajectory and N = this batch's masked
 * count.  adv_tok_out receives the fp64 token advantages.
 */
int oracle_grpo_step(int64_t T, int32_t n_traj, int32_t n_groups, int32_t n_tasks,
                     const int64_t* traj_offsets, const int32_t* task_id,
                     const int32_t* group_id, const float* rewards, const uint8_t* loss_mask,
                     double eps_std, int32_t d, int32_t V, const double* hidden,
                     const double* W, const int32_t* target, const double* old_logp,
                     double eps_lo, double eps_hi, double logit_scale,
                     /* outputs */
                     double* adv_tok_out, double* task_stats, double* loss, double* logp_out,
                     double* grad_hidden, double* grad_W, double* loss_stats) {
    int64_t* n_g = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_traj + 1));
    int32_t* K_j = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_groups + 1));
    double* ah = (double*)malloc(sizeof(double) * (size_t)(n_traj + 1));
    double* at = (double*)malloc(sizeof(double) * (size_t)(n_traj + 1));
    int64_t n_mask = 0;
    int st = oracle_task_adv_norm(T, n_traj, n_groups, n_tasks, traj_offsets, task_id, group_id,
                                  rewards, loss_mask, eps_std, n_g, K_j, ah, at, task_stats,
                                  adv_tok_out, NULL, &n_mask);
    if (st >= 0 && !(st & (ORS_BAD_OFFSETS | ORS_GROUP_SPANS_TASKS))) {
        int st2 = oracle_policy_loss_fwd_bwd(T, d, V, hidden, W, target, adv_tok_out, old_logp,
                                             loss_mask, eps_lo, eps_hi, logit_scale, n_mask,
                                             loss, logp_out, grad_hidden, grad_W, loss_stats);
        st = st2 < 0 ? st2 : (st | st2);
    }
    free(n_g);
    free(K_j);
    free(ah);
    free(at);
    return st;
}

/*
 * Forward-only log-prob and entropy of every masked token (the token
 * distribution of P:1186-1190).  Plain definitions in fp64:
 *   p_v = exp(z_v - lse),  logp_t = z_y - lse,  H_t = -sum_v p_v log p_v = -sum_v p_v (z_v - lse)
 * Unmasked tokens get 0.
 */
int oracle_logprob_entropy(int64_t T, int32_t d, int32_t V, const double* hidden,
                           const double* W, const int32_t* target, const uint8_t* loss_mask,
                           double logit_scale, double* logp_out /*[T]*/,
                           double* ent_out /*[T]*/) {
    if (T < 0 || d <= 0 || V <= 0 || !(logit_scale > 0)) return OR_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < T; ++t) {
        if (!loss_mask[t]) {
            logp_out[t] = 0.0;
            ent_out[t] = 0.0;
            continue;
        }
        double* z = (double*)malloc(sizeof(double) * (size_t)V);
        token_logits(d, V, hidden + (size_t)t * (size_t)d, W, logit_scale, z);
        double m = z[0];
        for (int32_t v = 1; v < V; ++v)
            if (z[v] > m) m = z[v];
        double se = 0.0;
        for (int32_t v = 0; v < V; ++v) se += exp(z[v] - m);
        const double lse = m + log(se);
        double H = 0.0;
        for (int32_t v = 0; v < V; ++v) {
            const double lp = z[v] - lse;
            H -= exp(lp) * lp;
        }
        logp_out[t] = z[target[t]] - lse;
        ent_out[t] = H;
        free(z);
    }
    return 0;
}

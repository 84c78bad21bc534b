/*
 * oracle_variants.c -- fp64 CPU ORACLE for the loss variants.
 * TEST INFRASTRUCTURE ONLY (same rules as agentrl_oracle.c; compiled into liboracle.so).
 *
 * Generalised per-token objective, in the paper's notation:
 *   term_t = min(rho_t A_t, clip(rho_t, 1-eps_lo, 1+eps_hi) A_t)
 *   KL_t   = exp(ref_t - logp_t) - (ref_t - logp_t) - 1                the "- beta D_KL" of
 *            (k3 estimator of D_KL(pi_theta || pi_ref), >= 0)         P:1103 / P:1119 (R11b)
 *   loss   = sum_{t masked} w_t ( -term_t + beta KL_t )
 *   w_t    = weights[t] if given, else 1/N (token-level mean, R7)
 * and the group-level aggregation of the GRPO objective:
 *   L_GRPO = E_{i,j} [ 1/K_{i,j} sum_{g=1}^{K_{i,j}} min(rho_{i,j,g} A, clip(..) A) ]
 *   read with token-level ratios (R7b): the per-trajectory term is the mean of term_t over
 *   the trajectory's n_g masked tokens (0 when n_g = 0), E_{i,j} is the mean over the G
 *   groups of the (global) batch that have at least one trajectory, and K_{i,j} counts every
 *   member of the group (also members without masked tokens), so
 *   w_t    = 1 / (G * K_{j(t)} * n_{g(t)}).
 * Exact gradient: d loss / d logp_t = -w_t [unclipped] rho A + w_t beta (1 - exp(ref - logp)),
 * so G_{t,v} = c_t (p_{t,v} - [v = y_t]) with c_t = w_t ([unclipped] rho A - beta (1 -
 * exp(ref_t - logp_t)));  grad_h = s G W,  grad_W = s G^T h.  Plain loops, fp64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORV_ERR_ARG (-1)
#define ORV_BAD_TARGET 1
#define ORV_NONFINITE 2
#define ORV_NO_TOKENS 32

/* w_t of the GRPO group-level aggregation (reading R7b); unmasked tokens get
 * 0.  Plain loops in the paper's order: K_j = #members of group j, n_g = #masked tokens of
 * trajectory g, G = #groups with K_j >= 1.  Returns G (or -1 on a group id outside
 * [0, n_groups)). */
int64_t oracle_grpo_group_weights(int64_t T, int32_t n_traj, int32_t n_groups,
                                  const int64_t* traj_offsets, const int32_t* group_id,
                                  const uint8_t* loss_mask, double* w_out /*[T]*/) {
    int64_t* K = (int64_t*)calloc((size_t)(n_groups > 0 ? n_groups : 1), sizeof(int64_t));
    if (!K) return -1;
    for (int32_t g = 0; g < n_traj; ++g) {
        if (group_id[g] < 0 || group_id[g] >= n_groups) {
            free(K);
            return -1;
        }
        K[group_id[g]] += 1;
    }
    int64_t G = 0;
    for (int32_t j = 0; j < n_groups; ++j) G += K[j] >= 1;
    for (int64_t t = 0; t < T; ++t) w_out[t] = 0.0;
    for (int32_t g = 0; g < n_traj; ++g) {
        int64_t n = 0;
        for (int64_t t = traj_offsets[g]; t < traj_offsets[g + 1]; ++t) n += loss_mask[t] != 0;
        for (int64_t t = traj_offsets[g]; t < traj_offsets[g + 1]; ++t)
            if (loss_mask[t])
                w_out[t] = 1.0 / ((double)G * (double)K[group_id[g]] * (double)n);
    }
    free(K);
    return G;
}

/* loss_stats[5]: clip fraction, mean rho, mean logp, masked tokens, mean KL */
int oracle_policy_loss_ex(int64_t T, int32_t d, int32_t V, const double* hidden, const double* W,
                          const int32_t* target, const double* adv_tok, const double* old_logp,
                          const uint8_t* loss_mask, double eps_lo, double eps_hi,
                          double logit_scale, int64_t n_mask_global, double kl_beta,
                          const double* ref_logp /*[T] or NULL*/,
                          const double* weights /*[T] or NULL*/, double* loss,
                          double* logp_out /*[T]*/, double* grad_hidden /*[T*d] or NULL*/,
                          double* grad_W /*[V*d] or NULL*/, double* loss_stats /*[5]*/) {
    if (T < 0 || d <= 0 || V <= 0 || eps_lo < 0 || eps_lo >= 1 || eps_hi < 0 ||
        !(logit_scale > 0) || kl_beta < 0 || (kl_beta > 0 && !ref_logp))
        return ORV_ERR_ARG;
    for (int64_t t = 0; t < T; ++t)
        if (loss_mask[t] && (target[t] < 0 || target[t] >= V)) return ORV_BAD_TARGET;
    const double s = logit_scale, N = (double)n_mask_global;
    if (grad_hidden) memset(grad_hidden, 0, sizeof(double) * (size_t)T * (size_t)d);
    if (grad_W) memset(grad_W, 0, sizeof(double) * (size_t)V * (size_t)d);
    for (int64_t t = 0; t < T; ++t) logp_out[t] = 0.0;
    *loss = 0.0;
    if (loss_stats) memset(loss_stats, 0, 5 * sizeof(double));
    if (n_mask_global <= 0 && !weights) return ORV_NO_TOKENS;

    double* z = (double*)malloc(sizeof(double) * (size_t)V);
    double* c = (double*)calloc((size_t)T, sizeof(double));
    double* lse_t = (double*)calloc((size_t)T, sizeof(double));
    double L = 0.0, n_clip = 0.0, s_rho = 0.0, s_logp = 0.0, s_kl = 0.0, nm = 0.0;
    /* forward + coefficients, token by token */
    for (int64_t t = 0; t < T; ++t) {
        if (!loss_mask[t]) continue;
        const double* h = hidden + (size_t)t * (size_t)d;
        for (int32_t v = 0; v < V; ++v) {
            double acc = 0.0;
            for (int32_t k = 0; k < d; ++k) acc += h[k] * W[(size_t)v * (size_t)d + (size_t)k];
            z[v] = s * acc;
        }
        double m = z[0];
        for (int32_t v = 1; v < V; ++v)
            if (z[v] > m) m = z[v];
        double se = 0.0;
        for (int32_t v = 0; v < V; ++v) se += exp(z[v] - m);
        const double lse = m + log(se);
        const double logp = z[target[t]] - lse;
        const double A = adv_tok[t], rho = exp(logp - old_logp[t]);
        const double lo = 1.0 - eps_lo, hi = 1.0 + eps_hi;
        const double rc = rho < lo ? lo : (rho > hi ? hi : rho);
        const double term = rho * A < rc * A ? rho * A : rc * A;
        const int clipped = (A > 0.0 && rho > hi) || (A < 0.0 && rho < lo);
        const double w = weights ? weights[t] : 1.0 / N;
        double kl = 0.0, dkl = 0.0;
        if (kl_beta > 0.0) {
            const double r = ref_logp[t] - logp;
            kl = exp(r) - r - 1.0;
            dkl = 1.0 - exp(r); /* d KL / d logp */
        }
        L += w * (-term + kl_beta * kl);
        c[t] = w * ((clipped ? 0.0 : rho * A) - kl_beta * dkl);
        lse_t[t] = lse;
        logp_out[t] = logp;
        n_clip += clipped ? 1.0 : 0.0;
        s_rho += rho;
        s_logp += logp;
        s_kl += kl;
        nm += 1.0;
    }
    /* backward: G_tv = c_t (p_tv - [v=y]) */
    for (int64_t t = 0; t < T; ++t) {
        if (!loss_mask[t] || (!grad_hidden && !grad_W)) continue;
        const double* h = hidden + (size_t)t * (size_t)d;
        for (int32_t v = 0; v < V; ++v) {
            double acc = 0.0;
            for (int32_t k = 0; k < d; ++k) acc += h[k] * W[(size_t)v * (size_t)d + (size_t)k];
            const double p = exp(s * acc - lse_t[t]);
            const double G = c[t] * (p - (v == target[t] ? 1.0 : 0.0));
            for (int32_t k = 0; k < d; ++k) {
                if (grad_hidden)
                    grad_hidden[(size_t)t * (size_t)d + (size_t)k] +=
                        s * G * W[(size_t)v * (size_t)d + (size_t)k];
                if (grad_W) grad_W[(size_t)v * (size_t)d + (size_t)k] += s * G * h[k];
            }
        }
    }
    *loss = L;
    if (loss_stats && nm > 0) {
        loss_stats[0] = n_clip / nm;
        loss_stats[1] = s_rho / nm;
        loss_stats[2] = s_logp / nm;
        loss_stats[3] = nm;
        loss_stats[4] = s_kl / nm;
    }
    free(z);
    free(c);
    free(lse_t);
    return isfinite(L) ? 0 : ORV_NONFINITE;
}

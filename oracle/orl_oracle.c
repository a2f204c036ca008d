/*
 * orl_oracle.c -- the fp64 CPU oracle for the PPO/RLVR "logits -> training
 * signal" path of OpenRLHF (arXiv 2405.11143).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2405_11143_b200/, liborl.so) never links, loads or
 * calls it, and this file includes no header of the product path.
 *
 * Every function is the paper's definition written out as plain loops in
 * double precision (App. C; SPEC.md ppo-core
 * S:153-222).  No blocking, fusion or reordering beyond what the definition
 * states.  Readings where the paper is silent are the Z-numbers of
 * DESIGN.md section 3 (= SURVEY.md 8(c).2).
 *
 * Citation key:  P:n = /root/reference/PAPER.md line n,
 *                S:n = /root/reference/SPEC.md line n.
 *
 * Pins (tests/test_oracle_pins.py): every function below is checked against
 * values fixed by the paper or by mathematics (closed forms, worked examples
 * in tests/golden/, 50-digit mpmath brute force, exact enumeration,
 * independent algorithms).  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_DTYPE_BF16 0
#define ORACLE_DTYPE_F32 1
#define ORACLE_DTYPE_F64 2 /* test inputs (finite differences) */

/* bf16 -> fp64 is exact: a bf16 is the top 16 bits of an IEEE fp32. */
static double bf16_bits_to_double(uint16_t h)
{
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

static double load_logit(const void *logits, int dtype, int64_t off)
{
    if (dtype == ORACLE_DTYPE_BF16)
        return bf16_bits_to_double(((const uint16_t *)logits)[off]);
    if (dtype == ORACLE_DTYPE_F64)
        return ((const double *)logits)[off];
    return (double)((const float *)logits)[off];
}

/* ------------------------------------------------------------------------
 * S1  log-softmax over the full vocabulary, gather, entropy.
 *     P:191 "records action log-probabilities log pi_theta(y_i|x_i)";
 *     P:193 reference log-probabilities; "S[pi_theta](s_t) is the
 *     entropy of the policy distribution"; S:76-84 sequence_logprobs.
 *     Z2: x = inv_temp * logit.  Z3: entropy = -sum_v p_v ln p_v (nats).
 *
 *     lse  = M + ln sum_v exp(x_v - M),  M = max_v x_v   (max-subtraction,
 *            S:116, does not change the result)
 *     logp = x_y - lse
 *     H    = -sum_v p_v ln p_v,  p_v = exp(x_v - lse),  ln p_v = x_v - lse
 *            (terms with p_v = 0 contribute 0, the limit of p ln p)
 * Returns 0, or 1 if the result is non-finite.
 * ---------------------------------------------------------------------- */
int oracle_row_logsoftmax(const double *x, int64_t V, int64_t y,
                          double *lse_out, double *logp_out, double *ent_out)
{
    double M = -INFINITY;
    for (int64_t v = 0; v < V; ++v)
        if (x[v] > M)
            M = x[v];
    double Z = 0.0;
    for (int64_t v = 0; v < V; ++v)
        Z += exp(x[v] - M);
    double lse = M + log(Z);
    double H = 0.0;
    for (int64_t v = 0; v < V; ++v) {
        double lp = x[v] - lse;
        double p = exp(lp);
        if (p > 0.0)
            H -= p * lp;
        else if (isnan(p))
            H = NAN;
    }
    double logp = x[y] - lse;
    *lse_out = lse;
    *logp_out = logp;
    *ent_out = H;
    return !(isfinite(lse) && isfinite(logp) && isfinite(H));
}

/*
 * S1 over a rank-local batch of B right-padded responses (Z10: valid iff
 * t < lengths[b]).  Logits row (b,t) starts at element b*stride_b + t*stride_t
 * (Z1: response-aligned), unit stride along V.  Per-token outputs are [B,T]
 * row-major; masked positions are exactly 0.0 and the logits there are never
 * read.  An out-of-vocabulary token (input error) gives NaN outputs and
 * is counted in *n_token_range; a non-finite result is counted in
 * *n_nonfinite.  Any output pointer may be NULL.
 */
void oracle_logprobs(const void *logits, int dtype, int64_t B, int64_t T, int64_t V,
                     int64_t stride_b, int64_t stride_t, const int32_t *tokens,
                     const int32_t *lengths, double inv_temp, double *logp,
                     double *entropy, double *lse, double *gathered,
                     int64_t *n_token_range, int64_t *n_nonfinite)
{
    double *x = (double *)malloc((size_t)(V > 0 ? V : 1) * sizeof(double));
    for (int64_t b = 0; b < B; ++b) {
        for (int64_t t = 0; t < T; ++t) {
            int64_t i = b * T + t;
            if (t >= lengths[b]) {
                if (logp) logp[i] = 0.0;
                if (entropy) entropy[i] = 0.0;
                if (lse) lse[i] = 0.0;
                if (gathered) gathered[i] = 0.0;
                continue;
            }
            int64_t y = tokens[i];
            if (y < 0 || y >= V) {
                if (n_token_range) *n_token_range += 1;
                if (logp) logp[i] = NAN;
                if (entropy) entropy[i] = NAN;
                if (lse) lse[i] = NAN;
                if (gathered) gathered[i] = NAN;
                continue;
            }
            int64_t base = b * stride_b + t * stride_t;
            for (int64_t v = 0; v < V; ++v)
                x[v] = inv_temp * load_logit(logits, dtype, base + v);
            double l, lp, h;
            int bad = oracle_row_logsoftmax(x, V, y, &l, &lp, &h);
            if (bad && n_nonfinite) *n_nonfinite += 1;
            if (logp) logp[i] = lp;
            if (entropy) entropy[i] = h;
            if (lse) lse[i] = l;
            if (gathered) gathered[i] = load_logit(logits, dtype, base + y);
        }
    }
    free(x);
}

/* ------------------------------------------------------------------------
 * S2  KL estimators, d = logp - logp_ref (Z6):
 *     k1 = d,  k2 = d^2/2,  k3 = exp(-d) - 1 + d.
 *     P:94 "we use k_2 as the loss function"; P:195 KL[pi_theta||pi_ref].
 * ---------------------------------------------------------------------- */
double oracle_kl(double d, int kind)
{
    if (kind == 1) return d;
    if (kind == 2) return 0.5 * d * d;
    if (kind == 3) return exp(-d) - 1.0 + d;
    return NAN;
}

/* derivative dk/dd, used for the KL-in-loss gradient (8(c).1 step 7) */
double oracle_kl_grad(double d, int kind)
{
    if (kind == 1) return 1.0;
    if (kind == 2) return d;
    if (kind == 3) return 1.0 - exp(-d);
    return NAN;
}

/* ------------------------------------------------------------------------
 * S2+S3  KL-shaped reward, "r'_t = r_t - beta KL[pi_theta||pi_ref]".
 *     Z4: shaping uses d = logp_a - logp_b with (a,b) = (old, ref).
 *     Z7: the scalar reward R_b sits on the last response token t = L_b-1
 *     (S:245).  kl_out[b,t] = k(d), r_out[b,t] = [t=L_b-1] R_b - beta k.
 *     Masked positions are 0.
 * ---------------------------------------------------------------------- */
void oracle_shape_rewards(int64_t B, int64_t T, const int32_t *lengths,
                          const double *logp_a, const double *logp_b, int kind,
                          double beta, const double *seq_reward, double *kl_out,
                          double *r_out)
{
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t) {
            int64_t i = b * T + t;
            if (t >= lengths[b]) {
                if (kl_out) kl_out[i] = 0.0;
                if (r_out) r_out[i] = 0.0;
                continue;
            }
            double k = oracle_kl(logp_a[i] - logp_b[i], kind);
            double r = (t == lengths[b] - 1) ? seq_reward[b] : 0.0;
            if (kl_out) kl_out[i] = k;
            if (r_out) r_out[i] = r - beta * k;
        }
}

/* ------------------------------------------------------------------------
 * S4  GAE, written as the paper's sum:
 *     delta_t = r_t + gamma V(s_{t+1}) - V(s_t)
 *     A_t     = sum_{l>=0} (gamma lambda)^l delta_{t+l}
 *     R_t     = A_t + V(s_t)
 *     Z8: the sum is truncated at the response end and V(s_{L_b}) = 0
 *     (S:176).  O(T^2) per response, on purpose: this is the
 *     definition, not the backward recursion the GPU scans with.
 * ---------------------------------------------------------------------- */
void oracle_gae(int64_t B, int64_t T, const int32_t *lengths, const double *r,
                const double *values, double gamma, double lambda, double *adv,
                double *ret)
{
    for (int64_t b = 0; b < B; ++b) {
        int64_t L = lengths[b];
        const double *rb = r + b * T;
        const double *Vb = values + b * T;
        for (int64_t t = 0; t < T; ++t) {
            int64_t i = b * T + t;
            if (t >= L) {
                adv[i] = 0.0;
                if (ret) ret[i] = 0.0;
                continue;
            }
            double A = 0.0, w = 1.0; /* w = (gamma lambda)^l */
            for (int64_t s = t; s < L; ++s) {
                double Vnext = (s + 1 < L) ? Vb[s + 1] : 0.0;
                double delta = rb[s] + gamma * Vnext - Vb[s];
                A += w * delta;
                w *= gamma * lambda;
            }
            adv[i] = A;
            if (ret) ret[i] = A + Vb[t];
        }
    }
}

/* ------------------------------------------------------------------------
 * S4'  REINFORCE++ return (north star; reading Z23):
 *     G_t = sum_{s=t}^{L_b-1} gamma^{s-t} r'_s.   O(T^2), the definition.
 * ---------------------------------------------------------------------- */
void oracle_discounted_returns(int64_t B, int64_t T, const int32_t *lengths,
                               const double *r, double gamma, double *out)
{
    for (int64_t b = 0; b < B; ++b) {
        int64_t L = lengths[b];
        for (int64_t t = 0; t < T; ++t) {
            int64_t i = b * T + t;
            if (t >= L) { out[i] = 0.0; continue; }
            double G = 0.0, w = 1.0;
            for (int64_t s = t; s < L; ++s) {
                G += w * r[b * T + s];
                w *= gamma;
            }
            out[i] = G;
        }
    }
}

/* ------------------------------------------------------------------------
 * S5  GRPO group advantages (P:102 name; Z20):
 *     groups are G contiguous sequences; mu = mean, sigma = population std
 *     (two-pass); A_b = (R_b - mu)/(sigma + 1e-8); a constant group
 *     (max == min) gives exactly 0.  keep[g] = (max - min >= 1e-12)
 *     is the DAPO dynamic-sampling keep flag (NEXT-2).
 *     Returns 0, or 1 if B is not a multiple of G.
 * ---------------------------------------------------------------------- */
int oracle_group_advantages(int64_t B, int64_t G, const double *R, double *adv_seq,
                            uint8_t *keep)
{
    if (G <= 0 || B % G != 0) return 1;
    for (int64_t g = 0; g < B / G; ++g) {
        const double *Rg = R + g * G;
        double mx = Rg[0], mn = Rg[0], sum = 0.0;
        for (int64_t j = 0; j < G; ++j) {
            if (Rg[j] > mx) mx = Rg[j];
            if (Rg[j] < mn) mn = Rg[j];
            sum += Rg[j];
        }
        double mu = sum / (double)G;
        double ss = 0.0;
        for (int64_t j = 0; j < G; ++j) ss += (Rg[j] - mu) * (Rg[j] - mu);
        double sigma = sqrt(ss / (double)G);
        for (int64_t j = 0; j < G; ++j)
            adv_seq[g * G + j] = (mx == mn) ? 0.0 : (Rg[j] - mu) / (sigma + 1e-8);
        if (keep) keep[g] = (mx - mn >= 1e-12) ? 1 : 0;
    }
    return 0;
}

/* REINFORCE++-baseline (Z23): R_b <- R_b - mean_g(R).  Returns 1 on bad G. */
int oracle_group_mean_subtract(int64_t B, int64_t G, const double *R, double *out)
{
    if (G <= 0 || B % G != 0) return 1;
    for (int64_t g = 0; g < B / G; ++g) {
        double sum = 0.0;
        for (int64_t j = 0; j < G; ++j) sum += R[g * G + j];
        double mu = sum / (double)G;
        for (int64_t j = 0; j < G; ++j) out[g * G + j] = R[g * G + j] - mu;
    }
    return 0;
}

/* broadcast a per-sequence value to the valid tokens of [B,T] (0 elsewhere) */
void oracle_broadcast_seq(int64_t B, int64_t T, const int32_t *lengths,
                          const double *per_seq, double *out)
{
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t)
            out[b * T + t] = (t < lengths[b]) ? per_seq[b] : 0.0;
}

/* ------------------------------------------------------------------------
 * S6  advantage whitening ("advantage normalization"; S:183-191;
 *     Z18, Z19, Z21): over the n valid advantages of the GLOBAL batch,
 *     mu = mean, sigma = population std (two-pass), A' = (A-mu)/(sigma+1e-8).
 *     n < 2 is a no-op (A' = A) and returns 1 (the warning flag).
 * ---------------------------------------------------------------------- */
int oracle_whiten_moments(const double *a, int64_t n, double *mean, double *std)
{
    if (n < 2) { *mean = 0.0; *std = 0.0; return 1; }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i];
    double mu = s / (double)n;
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) ss += (a[i] - mu) * (a[i] - mu);
    *mean = mu;
    *std = sqrt(ss / (double)n);
    return 0;
}

double oracle_whiten_value(double a, double mean, double std)
{
    return (a - mean) / (std + 1e-8);
}

/* ------------------------------------------------------------------------
 * S7-S9  PPO losses over the valid tokens of one rank-local batch
 *     (Z11-Z17, Z22).  Per token (b,t) with t < L_b:
 *       rho     = exp(logp_new - logp_old)
 *       obj     = min(rho A', clip(rho, 1-eps_low, 1+eps_high) A')
 *       clipped = [clip(rho) A' < rho A']  (strict, Z16)
 *       vl      = max((Vn-R)^2, (Vo + clip(Vn-Vo, -eps_v, eps_v) - R)^2)
 *                 if eps_v > 0, else (Vn-R)^2                       (Z13)
 *       H, k(new,ref) with the loss estimator, k3(old-new), rho
 *     sums[] (fp64, this batch):
 *       0 n  1 sum obj  2 sum vl  3 sum H  4 sum k(new,ref)  5 n clipped
 *       6 n value-clipped  7 sum k3(logp_old - logp_new)  8 sum rho
 *       9 n guard (|logp_new - logp_old| > ratio_guard, Z22)  10 n non-finite
 *     Per-token derivatives of the minimised total (8(c).1 step 7, Z17):
 *       dlogp = (-[not clipped] rho A' + [kl_in_loss] beta k'(d_ref)) / N
 *       dv    = c1 * dvl/dVn / N,  dvl/dVn = 2(Vn-R) on the unclipped branch
 *               (ties), else 2(Vc-R)[|Vn-Vo| < eps_v]
 *     clipped_out[b,t] (optional) holds the token's decisions as bits:
 *       0 clipped, 1 value-clipped (the clipped branch strictly wins, Z13),
 *       2 ratio guard (Z22), 3 a non-finite loss term; masked positions 0.
 *     N = n_global (all ranks' valid tokens, Z11).  A' = adv_w, already
 *     whitened by the caller when whitening is on.  Optional arrays may be
 *     NULL (no critic: v_new == NULL; no reference: logp_ref == NULL).
 *     NEXT-2 sequence-mean aggregation (Z31): sums[11..14] hold the
 *     per-sequence-mean sums  sum_t obj/L_b, vl/L_b, H/L_b, k(new,ref)/L_b
 *     (always); with seq_mean = 1 the derivatives are divided by
 *     n_seq * L_b instead of N (n_seq = all ranks' sequences with L_b > 0).
 * ---------------------------------------------------------------------- */
void oracle_ppo_loss(int64_t B, int64_t T, const int32_t *lengths,
                     const double *logp_new, const double *logp_old,
                     const double *logp_ref, const double *adv_w,
                     const double *ret, const double *v_new, const double *v_old,
                     const double *entropy, double eps_low, double eps_high,
                     double eps_v, double c1, double beta_loss, int kl_est,
                     int kl_in_loss, double ratio_guard, double n_global,
                     int seq_mean, double n_seq,
                     double *sums, double *obj_out, uint8_t *clipped_out,
                     double *vl_out, double *dlogp_out, double *dv_out)
{
    for (int k = 0; k < 15; ++k) sums[k] = 0.0;
    for (int64_t b = 0; b < B; ++b)
        for (int64_t t = 0; t < T; ++t) {
            int64_t i = b * T + t;
            if (t >= lengths[b]) {
                if (obj_out) obj_out[i] = 0.0;
                if (clipped_out) clipped_out[i] = 0;
                if (vl_out) vl_out[i] = 0.0;
                if (dlogp_out) dlogp_out[i] = 0.0;
                if (dv_out) dv_out[i] = 0.0;
                continue;
            }
            double A = adv_w[i];
            double dold = logp_new[i] - logp_old[i];
            double rho = exp(dold);
            double rho_c = rho;
            if (rho_c < 1.0 - eps_low) rho_c = 1.0 - eps_low;
            if (rho_c > 1.0 + eps_high) rho_c = 1.0 + eps_high;
            double unclipped = rho * A, clipped_term = rho_c * A;
            int clipped = clipped_term < unclipped;
            double obj = clipped ? clipped_term : unclipped;

            double vl = 0.0, dvl = 0.0;
            int vclipped = 0;
            if (v_new) {
                double e1 = v_new[i] - ret[i];
                if (eps_v > 0.0) {
                    double dv = v_new[i] - v_old[i];
                    double dvc = dv < -eps_v ? -eps_v : (dv > eps_v ? eps_v : dv);
                    double e2 = v_old[i] + dvc - ret[i];
                    vclipped = (e2 * e2) > (e1 * e1);
                    vl = vclipped ? e2 * e2 : e1 * e1;
                    dvl = vclipped ? 2.0 * e2 * (fabs(dv) < eps_v ? 1.0 : 0.0) : 2.0 * e1;
                } else {
                    vl = e1 * e1;
                    dvl = 2.0 * e1;
                }
            }

            double kref = 0.0, dkref = 0.0;
            if (logp_ref) {
                double dref = logp_new[i] - logp_ref[i];
                kref = oracle_kl(dref, kl_est);
                dkref = oracle_kl_grad(dref, kl_est);
            }
            double k3old = oracle_kl(logp_old[i] - logp_new[i], 3);
            double H = entropy ? entropy[i] : 0.0;

            sums[0] += 1.0;
            sums[1] += obj;
            sums[2] += vl;
            sums[3] += H;
            sums[4] += kref;
            sums[5] += clipped ? 1.0 : 0.0;
            sums[6] += vclipped ? 1.0 : 0.0;
            sums[7] += k3old;
            sums[8] += rho;
            int guard = fabs(dold) > ratio_guard;
            int nonfinite = !(isfinite(obj) && isfinite(vl) && isfinite(H) && isfinite(kref));
            if (guard) sums[9] += 1.0;
            if (nonfinite) sums[10] += 1.0;
            double Lb = (double)lengths[b];
            sums[11] += obj / Lb;
            sums[12] += vl / Lb;
            sums[13] += H / Lb;
            sums[14] += kref / Lb;

            double denom = seq_mean ? n_seq * Lb : n_global;
            if (obj_out) obj_out[i] = obj;
            if (clipped_out)
                clipped_out[i] = (uint8_t)(clipped | (vclipped << 1) | (guard << 2) | (nonfinite << 3));
            if (vl_out) vl_out[i] = vl;
            if (dlogp_out)
                dlogp_out[i] = ((clipped ? 0.0 : -rho * A) +
                                (kl_in_loss ? beta_loss * dkref : 0.0)) / denom;
            if (dv_out) dv_out[i] = c1 * dvl / denom;
        }
}

/* ------------------------------------------------------------------------
 * S9-S10  statistics from the global sums (Z11, Z12, Z27):
 *   out: 0 n_tokens 1 policy_loss = -sum obj/N 2 value_loss 3 entropy
 *        4 kl (loss estimator, new vs ref) 5 approx_kl_old (k3, old vs new)
 *        6 clip_frac 7 value_clip_frac 8 ratio_mean
 *        9 total = policy + c1 value - c2 entropy + [kl_in_loss] beta kl
 *   seq_mean = 1 (NEXT-2, Z31): policy_loss, value_loss, entropy and kl are
 *   means over the n_seq sequences of the per-sequence token means,
 *   e.g. policy_loss = -(1/n_seq) sum_b (1/L_b) sum_t obj; the shares and
 *   ratio_mean stay token means.
 *   N = 0 returns 1 (ORL_E_EMPTY_BATCH) and leaves out[] at 0.
 * ---------------------------------------------------------------------- */
int oracle_stats(const double *sums, double c1, double c2, double beta_loss,
                 int kl_in_loss, int seq_mean, double n_seq, double *out)
{
    for (int k = 0; k < 10; ++k) out[k] = 0.0;
    double N = sums[0];
    if (!(N > 0.0)) return 1;
    out[0] = N;
    out[1] = seq_mean ? -sums[11] / n_seq : -sums[1] / N;
    out[2] = seq_mean ? sums[12] / n_seq : sums[2] / N;
    out[3] = seq_mean ? sums[13] / n_seq : sums[3] / N;
    out[4] = seq_mean ? sums[14] / n_seq : sums[4] / N;
    out[5] = sums[7] / N;
    out[6] = sums[5] / N;
    out[7] = sums[6] / N;
    out[8] = sums[8] / N;
    out[9] = out[1] + c1 * out[2] - c2 * out[3] + (kl_in_loss ? beta_loss * out[4] : 0.0);
    return 0;
}

/* ------------------------------------------------------------------------
 * NEXT-1  gradient of the minimised total (Z12) w.r.t. the actor's raw
 *     logits, for one valid row ("gradient computation"):
 *       z = inv_temp x,  p = softmax(z),  ln p_v = z_v - lse,
 *       H = -sum_v p_v ln p_v,
 *       dL/dz_v = w (delta_vy - p_v) + a p_v (ln p_v + H),   a = c2/N
 *       dL/dx_v = inv_temp dL/dz_v
 *     w = dL/dlogp_new (the per-token derivative of oracle_ppo_loss).  The
 *     entropy part is the derivative of -c2 mean(H), present only when the
 *     loss has that term (a != 0: with c2 = 0 a -inf logit, p_v = 0, gets
 *     the gradient -w p_v = 0, not 0 * (-inf); DESIGN Z39); the policy and
 *     KL-loss parts reach the logits only through logp_new = z_y - lse.
 * ---------------------------------------------------------------------- */
void oracle_logits_grad_row(const double *x, int64_t V, int64_t y, double inv_temp, double w,
                            double a, double *grad)
{
    double *z = (double *)calloc((size_t)(V > 0 ? V : 1), sizeof(double));
    for (int64_t v = 0; v < V; ++v) z[v] = inv_temp * x[v];
    double lse, logp, H;
    oracle_row_logsoftmax(z, V, y, &lse, &logp, &H);
    for (int64_t v = 0; v < V; ++v) {
        double lp = z[v] - lse;
        double p = exp(lp);
        double dz = w * ((v == y ? 1.0 : 0.0) - p);
        if (a != 0.0) dz += a * p * (lp + H);  /* c2 = 0: no entropy term in the loss (Z39) */
        grad[v] = inv_temp * dz;
    }
    free(z);
}

/* ------------------------------------------------------------------------
 * NEXT-3  adaptive KL coefficient and early stop:
 *   beta <- beta (1 + clip(observed/target - 1, -0.5, 0.5) / horizon)
 *   early_stop = observed > max_kl
 * ---------------------------------------------------------------------- */
int oracle_kl_controller_step(double *beta, double target, double horizon, double observed,
                              double max_kl)
{
    double e = observed / target - 1.0;
    if (e < -0.5) e = -0.5;
    if (e > 0.5) e = 0.5;
    *beta = *beta * (1.0 + e / horizon);
    return observed > max_kl;
}

/* ------------------------------------------------------------------------
 * NEXT-4  LM head + S1 ("the actor model ...
 * forward", P:191/P:193 log-probabilities):
 *     z_{r,v} = sum_k h_{r,k} W_{v,k}          (the LM-head logits, fp64)
 *     then S1 of row r on x = inv_temp * z_r, target y_r (oracle_row_logsoftmax).
 * h is [R, d] with row pitch ld_h, W is [V, d] with row pitch ld_w, both bf16
 * bit patterns (exact in fp64).  y_r < 0 marks a row that is not computed
 * (outputs 0); y_r >= V gives NaN outputs (token range).  gathered_z = z_{r,y}.
 * Returns the number of non-finite rows.
 * ---------------------------------------------------------------------- */
int64_t oracle_lmhead_rows(const uint16_t *h, int64_t ld_h, const uint16_t *W, int64_t ld_w,
                           int64_t R, int64_t d, int64_t V, const int32_t *y, double inv_temp,
                           double *logp, double *entropy, double *lse, double *gathered_z)
{
    int64_t bad = 0;
    double *z = (double *)malloc((size_t)(V > 0 ? V : 1) * sizeof(double));
    double *x = (double *)malloc((size_t)(V > 0 ? V : 1) * sizeof(double));
    for (int64_t r = 0; r < R; ++r) {
        logp[r] = entropy[r] = lse[r] = gathered_z[r] = 0.0;
        if (y[r] < 0)
            continue;
        if (y[r] >= V) {
            logp[r] = entropy[r] = lse[r] = gathered_z[r] = NAN;
            continue;
        }
        for (int64_t v = 0; v < V; ++v) {
            double acc = 0.0;
            for (int64_t k = 0; k < d; ++k)
                acc += bf16_bits_to_double(h[r * ld_h + k]) * bf16_bits_to_double(W[v * ld_w + k]);
            z[v] = acc;
            x[v] = inv_temp * acc;
        }
        bad += oracle_row_logsoftmax(x, V, y[r], &lse[r], &logp[r], &entropy[r]);
        gathered_z[r] = z[y[r]];
    }
    free(z);
    free(x);
    return bad;
}

/* ------------------------------------------------------------------------
 * NEXT-2 / Z10  attention mask -> response lengths ("attention masks";
 *     S:240 masked positions).  The path's masks are right-padded prefixes:
 *     lengths[b] = number of leading nonzero entries of mask row b, i.e. the
 *     first t with mask[b,t] == 0 (T if none).  A row with a nonzero entry
 *     after its first zero is not a prefix mask (Z10: ORL_E_MASK); it keeps its
 *     leading-prefix length and is counted.  Returns the number of such rows.
 * ---------------------------------------------------------------------- */
int64_t oracle_lengths_from_mask(int64_t B, int64_t T, const uint8_t *mask, int32_t *lengths)
{
    int64_t bad = 0;
    for (int64_t b = 0; b < B; ++b) {
        int64_t L = T;
        for (int64_t t = 0; t < T; ++t)
            if (mask[b * T + t] == 0) { L = t; break; }
        int hole = 0;
        for (int64_t t = L; t < T; ++t)
            if (mask[b * T + t] != 0) hole = 1;
        lengths[b] = (int32_t)L;
        bad += hole;
    }
    return bad;
}

/* ------------------------------------------------------------------------
 * NEXT-2  DAPO dynamic sampling ("DAPO"): the indices of the
 *     kept groups (keep[g] != 0, the flag oracle_group_advantages writes), in
 *     increasing order, into idx[0..count).  Returns count.
 * ---------------------------------------------------------------------- */
int64_t oracle_keep_compact(int64_t n_groups, const uint8_t *keep, int32_t *idx)
{
    int64_t count = 0;
    for (int64_t g = 0; g < n_groups; ++g)
        if (keep[g] != 0) idx[count++] = (int32_t)g;
    return count;
}

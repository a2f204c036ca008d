/*
 * orl.h -- C ABI of liborl.so: the B200 (sm_100a) hot path that turns rollout
 * logits into PPO / GRPO / REINFORCE++ training signal, after the PPO workflow
 * of OpenRLHF (arXiv 2405.11143), Appendix C, lines 189-201.
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n (the CPU spec
 * written from the paper; used here for interfaces and error semantics),
 * Z-numbers = the readings listed in DESIGN.md section 3.
 *
 * One iteration on one rank (one process per GPU), in this order:
 *
 *   orl_begin_iteration                          reset accumulators/counters
 *   for each micro-batch: orl_logprobs(old)      S1
 *   for each micro-batch: orl_logprobs(ref,      S1+S2+S3
 *                               partner = old logp)
 *   orl_advantages                               S4 / S4' / S5
 *   orl_whiten_stats                             S6 + collective C1
 *   for each micro-batch: orl_ppo_loss           S1+S7+S8+S9
 *   orl_finalize                                 S10 + collective C2
 * C1/C2 run over NCCL or, after orl_peer_open, as single peer-memory kernels;
 * orl_finalize_async + orl_stats_decode split S10 for CUDA-graph capture;
 * NEXT-1 (orl_logits_grad, orl_ppo_loss_and_grad), NEXT-3
 * (orl_kl_controller_step) and NEXT-4 (orl_lmhead_*) are declared below.
 *
 * Conventions shared by every call
 *  - Pointers are DEVICE pointers on the context's device unless a comment
 *    says "host".  The caller owns every buffer; the library never frees or
 *    retains a caller pointer after a call returns.
 *  - Every call is asynchronous and stream-ordered on `stream` (a
 *    cudaStream_t passed as void*; NULL = legacy default stream), except
 *    orl_finalize, which synchronises `stream` before returning.
 *  - Per-token arrays are row-major [B_total, T] over the RANK-LOCAL batch of
 *    B_total responses, 4-byte aligned (ORL_E_ALIGN otherwise).  Position
 *    (b,t) is valid iff t < lengths[b] (right-padded prefix mask, Z10).
 *    Outputs at masked positions are written as exactly 0.0f; inputs there
 *    (logits included) are never read.  lengths[b] == 0 is allowed.
 *  - A micro-batch is the sequence range [seq_offset, seq_offset + B) of the
 *    rank-local batch; its logits are addressed relative to sequence
 *    seq_offset (see orl_logits).
 *  - Argument errors are detected on the host before any launch and return a
 *    status without side effects.  Data errors found on the device (token out
 *    of range, non-finite values, ratio guard) never abort a launch: the
 *    offending token's outputs become NaN and a device counter is
 *    incremented; orl_finalize reports them.
 *  - Not thread-safe per context: one context per device per host thread.
 */
#ifndef ORL_H
#define ORL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORL_VERSION 2 /* 2: per-token decision flags in the actor passes, orl_set_pdl_chain,
                         the optional low part of the advantages (adv_lo) */
#define ORL_UNIQUE_ID_BYTES 128 /* == sizeof(ncclUniqueId) */
#define ORL_STATS_N 16          /* length of the device stats vector */
#define ORL_PARTIALS_N 24       /* length of a rank's loss/stat partial (hooks) */
#define ORL_MAX_SEQ_PER_CALL 8192

typedef enum {
    ORL_OK = 0,
    ORL_E_INVALID_ARG = 1,   /* NULL required pointer, bad enum, bad scalar    */
    ORL_E_SHAPE = 2,         /* non-positive/oversized dims, stride < V        */
    ORL_E_ALIGN = 3,         /* per-token array not 4-byte aligned             */
    ORL_E_DTYPE = 4,         /* unknown logits dtype                           */
    ORL_E_TOKEN_RANGE = 5,   /* some valid token outside [0, V)       */
    ORL_E_MASK = 6,          /* lengths[b] < 0 or > T (counted once per        */
                             /* iteration by orl_advantages; the streaming     */
                             /* passes clamp), non-prefix attention mask       */
    ORL_E_NONFINITE = 7,     /* non-finite logits / loss terms    (Z26)        */
    ORL_E_NUMERIC_GUARD = 8, /* |logp_new - logp_old| > guard     (Z22) */
    ORL_E_EMPTY_BATCH = 9,   /* no valid token on any rank                     */
    ORL_E_GROUP_SPLIT = 10,  /* GRPO batch not a whole number of groups        */
    ORL_E_CUDA = 11,         /* CUDA runtime error (see orl_last_error)        */
    ORL_E_NCCL = 12,         /* NCCL error (see orl_last_error)                */
    ORL_E_STATE = 13         /* calls out of order (e.g. loss before whitening)*/
} orl_status;

typedef enum { ORL_BF16 = 0, ORL_F32 = 1 } orl_dtype;

/* KL estimators with d = logp - logp_ref (Z6):
 * k1 = d, k2 = d^2/2, k3 = exp(-d) - 1 + d. */
typedef enum { ORL_KL_K1 = 1, ORL_KL_K2 = 2, ORL_KL_K3 = 3 } orl_kl;

/* Advantage estimators.
 *  GAE          P:195  delta_t = r'_t + gamma V_{t+1} - V_t,
 *                      A_t = sum_l (gamma lambda)^l delta_{t+l}, R_t = A_t + V_t
 *  GRPO         P:102 (name): A_b = (R_b - mu_g)/(sigma_g + 1e-8)
 *  RPP          REINFORCE++ (north star, Z23): A_t = sum_{s>=t} gamma^{s-t} r'_s
 *  RPP_BASELINE RPP after R_b <- R_b - mu_g (group mean)                     */
typedef enum {
    ORL_ADV_GAE = 0,
    ORL_ADV_GRPO = 1,
    ORL_ADV_RPP = 2,
    ORL_ADV_RPP_BASELINE = 3
} orl_adv;

typedef struct orl_ctx orl_ctx; /* opaque */

/* A [B,T,V] logits view.  Row (b,t) of the micro-batch starts at element
 * b*stride_b + t*stride_t of `ptr` (b relative to the micro-batch), with
 * unit stride along V.  Response-aligned (Z1): row (b,t) is the distribution
 * token tokens[b,t] was sampled from; pass a view offset by prompt_len-1 to
 * use a model's full-sequence logits.  Requires stride_t >= V and
 * stride_b >= 0 (ORL_E_SHAPE).  When the base address and both byte pitches
 * are 16-byte aligned and V*elt is a multiple of 16, rows are streamed by the
 * TMA bulk-copy kernel; otherwise a generic (non-TMA) kernel runs. */
typedef struct {
    const void *ptr;
    int32_t dtype; /* orl_dtype */
    int32_t pad_;
    int64_t V;        /* vocabulary size; V * element size < 2^31 bytes (else ORL_E_SHAPE) */
    int64_t stride_b; /* elements */
    int64_t stride_t; /* elements */
} orl_logits;

/* The response rows of one micro-batch. */
typedef struct {
    int64_t B;              /* sequences in this call, 1..ORL_MAX_SEQ_PER_CALL */
    int64_t T;              /* max response length; pitch of per-token arrays */
    int64_t seq_offset;     /* first sequence of the call in the rank batch   */
    const int32_t *tokens;  /* [B_total, T] sampled token ids y_{b,t}         */
    const int32_t *lengths; /* [B_total] response lengths L_b, 0 <= L_b <= T  */
    /* Optional (NULL = padded logits).  Packed varlen logits (NEXT-2):
     * [B_total + 1] token offsets with cu_seqlens[b+1] - cu_seqlens[b] >= L_b;
     * logits row (b,t) of the call is element
     * (cu_seqlens[seq_offset+b] - cu_seqlens[seq_offset] + t) * stride_t of the
     * logits pointer (stride_b unused), and likewise for orl_logits_grad's
     * output.  Per-token arrays stay [B_total, T]. */
    const int32_t *cu_seqlens;
} orl_rows;

/* PPO loss configuration. */
typedef struct {
    double eps_low;     /* clip(rho, 1-eps_low, 1+eps_high); DAPO decoupled */
    double eps_high;    /*   clip when eps_low != eps_high (Z15)      */
    double eps_value;   /* value clip half-width; <= 0: plain (V-R)^2 (Z13) */
    double c1;          /* value-loss coefficient                           */
    double c2;          /* entropy-bonus coefficient                        */
    double beta_loss;   /* KL-in-loss coefficient ("k2 as the loss")   */
    int32_t kl_loss_est;/* orl_kl used for the loss term and the kl stat    */
    int32_t kl_in_loss; /* 1: total += beta_loss * mean k(new, ref)  (Z5)   */
    double ratio_guard; /* |logp_new - logp_old| > guard counts (Z22); 30   */
    int32_t loss_agg;   /* 0 = token mean over all ranks' tokens (Z11);     */
                        /* 1 = mean over sequences of per-sequence token    */
                        /*     means (NEXT-2, Z31; S:243 names the default) */
    int32_t pad_;
} orl_ppo_cfg;

/* Host-side statistics.  Means are over the N valid tokens of
 * ALL ranks (Z11).  total_loss = policy_loss + c1 value_loss - c2 entropy
 * + [kl_in_loss] beta_loss kl (Z12). */
typedef struct {
    double n_tokens;
    double policy_loss;     /* -mean min(rho A', clip(rho) A')                 */
    double value_loss;      /* mean of the (clipped) squared error, no 1/2     */
    double entropy;         /* mean full-vocabulary entropy (nats)             */
    double kl;              /* mean k(logp_new - logp_ref), loss estimator     */
    double approx_kl_old;   /* mean k3(logp_old - logp_new) (Z27)              */
    double clip_frac;       /* share of tokens whose clipped branch is active  */
    double value_clip_frac; /* share whose clipped value branch strictly wins  */
    double ratio_mean;      /* mean rho                                        */
    double total_loss;
    double adv_mean;        /* global whitening moments (0 when not whitened)  */
    double adv_std;
    int64_t n_guard;
    int64_t n_nonfinite;
    int64_t n_token_range;
    int32_t whiten_warn;    /* whitening requested with < 2 tokens     */
    int32_t pad_;
} orl_stats;
/* The device stats vector (double[ORL_STATS_N]) holds, in order: n_tokens,
 * policy_loss, value_loss, entropy, kl, approx_kl_old, clip_frac,
 * value_clip_frac, ratio_mean, total_loss, adv_mean, adv_std, n_guard,
 * n_nonfinite, n_token_range, whiten_warn. */

/* ---- context ----------------------------------------------------------- */

/* Library version (ORL_VERSION). */
int orl_version(void);

/* Host.  Rank 0 creates an NCCL unique id (ORL_UNIQUE_ID_BYTES bytes into
 * `id_out`) and broadcasts it to the other ranks (e.g. torch.distributed). */
orl_status orl_get_unique_id(unsigned char *id_out);

/* Create a context on CUDA `device` for rank `rank` of `world` ranks.
 * world == 1: `id` may be NULL (no communicator; the collectives reduce to
 * local merges) or a unique id (a 1-rank NCCL communicator).  world > 1: `id`
 * (host, ORL_UNIQUE_ID_BYTES) from orl_get_unique_id creates an NCCL
 * communicator (collective: all ranks must call); with id == NULL the context
 * has no communicator and orl_peer_open must be called before the first
 * orl_whiten_stats (ORL_E_STATE otherwise).  The context owns the NCCL
 * communicator, the peer exchange buffer, fp64 partial buffers, device error
 * counters and a pinned host stats slot. */
orl_status orl_create(int device, int world, int rank, const unsigned char *id, orl_ctx **out);

/* Destroy a context (synchronises its device first).  NULL is a no-op. */
orl_status orl_destroy(orl_ctx *ctx);

/* Human-readable text of the last error on `ctx` (or of the calling thread
 * when ctx is NULL).  Valid until the next call on the same ctx/thread. */
const char *orl_last_error(const orl_ctx *ctx);

/* Number of kernels the context has launched so far (for bench accounting). */
uint64_t orl_launch_count(const orl_ctx *ctx);

/* Programmatic dependent launch (PDL) between consecutive streaming passes.
 * Every K1/K5 launch allows the NEXT kernel on its stream to start while its own
 * CTAs retire.  By default (enable = 0) every warp of a K1/K5 launch waits for
 * its preceding kernel to complete (griddepcontrol.wait) before its first read,
 * so inputs written by ANY predecessor -- including one that triggers its
 * dependents early, such as a PDL-aware GEMM writing the logits -- are complete
 * and visible.  enable = 1 lets the K1 producer stream the logits, tokens and
 * lengths without that wait (only the epilogue warps, which read what earlier
 * passes of the path wrote, wait): the next micro-batch's stream then overlaps
 * the tail of the previous launch.  Precondition for enable = 1: on every stream
 * passed to this context, the kernel that immediately precedes an orl_logprobs /
 * orl_ppo_loss / orl_ppo_loss_and_grad call and writes its logits, tokens or
 * lengths either is an orl kernel or triggers no early launch (plain kernels and
 * copies complete before their dependents start).  Host only; takes effect for
 * later calls; returns ORL_E_INVALID_ARG for a NULL ctx. */
orl_status orl_set_pdl_chain(orl_ctx *ctx, int enable);
/* Current setting (0 or 1), -1 for a NULL ctx. */
int orl_get_pdl_chain(const orl_ctx *ctx);

/* Attention-mask input (Z10, "attention masks"): lengths[b] = the number of
 * leading ones of mask[b, 0..T) (device, u8 [B, T] row-major; nonzero = valid).
 * The path's masks are right-padded prefixes: a valid position after the first
 * padded one is counted as a mask error (orl_finalize -> ORL_E_MASK; the row
 * keeps its leading prefix).  Call after orl_begin_iteration (which clears the
 * counters).  Stream-ordered; B = 0 is a no-op; T < 1: ORL_E_SHAPE. */
orl_status orl_lengths_from_mask(orl_ctx *ctx, int64_t B, int64_t T, const uint8_t *mask, int32_t *lengths,
                                 void *stream);

/* NEXT-2, DAPO dynamic sampling: from orl_advantages' group_keep
 * mask (device, uint8 [n_groups]), write the indices of the kept groups in increasing
 * order to kept_groups (device, int32 [n_groups], the first *n_kept entries used) and
 * their count to n_kept (device, int32) -- the list a scheduler keeps while it re-rolls
 * the dropped prompts.  Stream-ordered, deterministic.  n_groups = 0 writes 0. */
orl_status orl_keep_compact(orl_ctx *ctx, int64_t n_groups, const uint8_t *group_keep, int32_t *kept_groups,
                            int32_t *n_kept, void *stream);

/* Pre-size the context's workspaces (host call, synchronises the device):
 * per-sequence whitening partials and the length prefix for up to max_seqs
 * responses per rank-local batch / call, and the NEXT-4 split partials for
 * LM-head calls of up to max_lm_rows hidden rows at vocabulary max_vocab (0:
 * none).  Calls within these sizes then never allocate, which is what CUDA-graph
 * capture of an iteration needs (otherwise the first call of each size
 * allocates; capture after one eager warm-up iteration).  Sizes < 0:
 * ORL_E_SHAPE. */
orl_status orl_reserve(orl_ctx *ctx, int64_t max_seqs, int64_t max_lm_rows, int64_t max_vocab);

/* Start an iteration: zero the loss accumulators, error counters and
 * advantage partials on `stream`. */
orl_status orl_begin_iteration(orl_ctx *ctx, void *stream);

/* ---- S1 (+S2+S3): log-softmax, gather, entropy ------------------------- */

/* For each valid (b,t) of the micro-batch, with x = inv_temp * logits[b,t,:]
 * (Z2):  lse = log sum_v exp(x_v)
 *        logp = x_y - lse,  y = tokens[b,t]
 *        entropy = -sum_v p_v log p_v  (nats, Z3)
 *        gathered = logits[b,t,y] as float (bit-exact)
 * If partner_logp != NULL (the reference pass, partner = logp_old, Z4):
 *        d = partner_logp - logp;  kl = k(d) with estimator kl_est   S2
 *        shaped_reward = [t == L_b-1] seq_reward[b] - beta_reward * kl
 *                                                        S3, Z7
 * logp is required; entropy, lse, gathered, kl, shaped_reward may be NULL.
 * seq_reward is [B_total] (indexed by rank-local sequence) and is required
 * when shaped_reward != NULL.  inv_temp > 0.  All per-token arrays are
 * [B_total, T] and only the micro-batch's rows are written. */
orl_status orl_logprobs(orl_ctx *ctx, const orl_rows *rows, const orl_logits *logits,
                        float inv_temp, float *logp, float *entropy, float *lse,
                        float *gathered, const float *partner_logp, int kl_est,
                        double beta_reward, const float *seq_reward, float *kl,
                        float *shaped_reward, void *stream);

/* ---- S4 / S4' / S5: advantages over the whole rank-local batch --------- */

/* kind = GAE:  needs shaped_reward, values (V_old, Z9); writes adv, ret.
 *        RPP:  needs shaped_reward; writes adv (= return G_t) and, if
 *              given, ret (= adv).
 *        RPP_BASELINE: as RPP but first subtracts the group mean of
 *              seq_reward (group_size consecutive sequences) from the
 *              reward at t = L_b-1 (equivalent to shaping R_b - mu_g, Z23).
 *        GRPO: needs seq_reward, group_size; writes adv[b,t] = A_b on valid
 *              tokens; ret unused; constant groups give exactly 0.
 * group_keep (optional, [B/group_size] uint8, GRPO and RPP_BASELINE) is the
 * DAPO dynamic-sampling flag max_g - min_g >= 1e-12.
 * adv_lo (optional, [B, T] fp32) receives A - (float)A for every valid token, so
 * adv + adv_lo carries the fp64 scan value to ~2^-48 relative; passed to the actor
 * pass it makes the whitening (A - mu)/(sigma + 1e-8) exact to fp64 even when the
 * advantages are nearly constant (|mu|/sigma up to ~1e9; Z33).  With adv_lo the
 * whitening moments are taken from adv + adv_lo, else from adv.
 * gamma, lambda in [0,1].  The whitening partials (count, mean, M2 over valid
 * tokens, fp64) are staged in ctx for orl_whiten_stats.
 * ORL_E_GROUP_SPLIT if B is not a multiple of group_size (GRPO/RPP_BASELINE). */
orl_status orl_advantages(orl_ctx *ctx, int64_t B, int64_t T, const int32_t *lengths,
                          int kind, double gamma, double lambda, int group_size,
                          const float *shaped_reward, const float *values,
                          const float *seq_reward, float *adv, float *adv_lo, float *ret,
                          uint8_t *group_keep, void *stream);

/* ---- S6 + C1: global whitening moments -------------------------------- */

/* Combines every rank's (count, mean, M2) in rank order (all-gather over
 * NCCL when world > 1, then a fixed-order Chan merge on the device, so every
 * rank gets bit-identical results).  whiten = 1: orl_ppo_loss will use
 * A' = (A - mu)/(sigma + 1e-8) with the population sigma (Z18, Z19);
 * with fewer than 2 tokens this is a no-op and whiten_warn is set.
 * whiten = 0: only the global token count N is formed (needed for the
 * token-mean loss, Z11).  Must follow orl_advantages. */
orl_status orl_whiten_stats(orl_ctx *ctx, int whiten, void *stream);

/* ---- S1 + S7..S9: actor pass with the loss epilogue -------------------- */

/* Recomputes logp_new and entropy from the actor logits (as orl_logprobs)
 * and, per valid token, in fp64:
 *   rho = exp(logp_new - logp_old); A' = whitened adv (if whitening on)
 *   obj = min(rho A', clip(rho, 1-eps_low, 1+eps_high) A')
 *   vl  = max((Vn-R)^2, (Vo + clip(Vn-Vo, +-eps_v) - R)^2)       P:197, Z13
 *   k(new, ref) with cfg->kl_loss_est when logp_ref != NULL
 * and accumulates fp64 sums into the context (fixed order: deterministic).
 * Optional per-token outputs:
 *   dloss_dlogp = (-[not clipped] rho A' + [kl_in_loss] beta k'(d_ref)) / N
 *   dloss_dv    = c1 dvl/dVn / N   (ties take the unclipped branch, Z17)
 *   flags       = uint8 [B_total, T] per-token decisions, taken in fp64 exactly
 *                 as the sums above take them:
 *                   bit 0  clipped: clip(rho) A' < rho A' strictly  (Z16)
 *                   bit 1  value-clipped branch strictly wins the max  (Z13)
 *                   bit 2  ratio guard |logp_new - logp_old| > guard   (Z22)
 *                   bit 3  a non-finite loss term                       (Z29)
 *                 masked positions 0 (S:216 clip_fraction per token)
 * with N the global token count from orl_whiten_stats.
 * A = adv (+ adv_lo when given: the low part orl_advantages wrote, Z33).
 * logp_old, adv required; logp_ref, adv_lo optional; ret, v_new, v_old together or
 * all NULL (no critic).  logp_new required; entropy, lse, dloss_*, flags optional. */
orl_status orl_ppo_loss(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                        float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                        const float *logp_ref, const float *adv, const float *adv_lo, const float *ret,
                        const float *v_new, const float *v_old, float *logp_new,
                        float *entropy, float *lse, float *dloss_dlogp, float *dloss_dv,
                        uint8_t *flags, void *stream);
/* (lse, optional: the log-partition of the scaled actor logits, saved for
 * orl_logits_grad.) */

/* ---- NEXT-1: gradient w.r.t. the actor logits -------------------------- */

/* One streaming pass over the actor logits of a micro-batch that writes
 *   dL/dx_v = inv_temp * ( w (delta_{v,y} - p_v) + (c2/N) p_v (ln p_v + H) )
 * for every valid row, where L is the minimised total of orl_finalize (Z12),
 * p = softmax(inv_temp x), w = dloss_dlogp, and lse (the log-partition), H
 * (entropy) and w are the per-token outputs the actor pass saved
 * (orl_ppo_loss); N is the global token count of orl_whiten_stats and c2 is
 * cfg->c2.  P:197 "gradient computation"; SURVEY 8(f) NEXT-1.
 * dlogits (device) has the actor's dtype and V, element strides
 * (out_stride_b, out_stride_t) relative to the micro-batch's first sequence,
 * and must not alias any logits still being read.  zero_masked = 1 also
 * writes zeros into the rows with t >= L_b.  Outputs are rounded to the
 * logits dtype (bf16: round-to-nearest-even).  A -inf logit (allowed in the
 * forward passes) has p_v = 0; with cfg->c2 != 0 its gradient element is NaN, as
 * the entropy term's p_v ln p_v = 0 * (-inf) is in the fp64 oracle, with
 * cfg->c2 = 0 (no entropy term) it is exactly 0 (DESIGN Z39); mask vocabulary
 * entries with a large finite negative logit (e.g. -1e30, which keeps
 * x * inv_temp * log2(e) finite in fp32) for an exact zero gradient either way. */
orl_status orl_logits_grad(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                           float inv_temp, const orl_ppo_cfg *cfg, const float *lse,
                           const float *entropy, const float *dloss_dlogp, void *dlogits,
                           int64_t out_stride_b, int64_t out_stride_t, int zero_masked,
                           void *stream);

/* ---- S10 + C2: statistics ---------------------------------------------- */

/* Sums the context's accumulators and error counters over ranks (all-gather
 * + rank-ordered sum, C2), forms the means and total loss with cfg's c1,c2,
 * beta_loss, writes the device vector dev_out (optional, double[16]) and the
 * host struct host_out (optional), synchronises `stream`, and maps the error
 * counters to a status: NCCL (a peer collective timed out) > TOKEN_RANGE >
 * MASK > SHAPE (LM-head rows) > NONFINITE > NUMERIC_GUARD > EMPTY_BATCH > OK
 * (outputs are written in every case). */
orl_status orl_finalize(orl_ctx *ctx, const orl_ppo_cfg *cfg, orl_stats *host_out,
                        double *dev_out, void *stream);

/* orl_finalize without the host synchronisation, for CUDA-graph capture of a whole
 * iteration: launches C2 and the final statistics on `stream` and copies the
 * device stats vector (double[ORL_STATS_N]) followed by the 4 device flags
 * (whiten_warn, invalid lengths + non-prefix mask rows, collective timeouts,
 * LM-head rows beyond the hidden matrix) into dev_out
 * (device, double[ORL_FINAL_N], required).  No host memory is touched; the
 * caller copies dev_out to the host when it needs it and maps it to a status
 * with orl_stats_decode. */
#define ORL_FINAL_N 20
orl_status orl_finalize_async(orl_ctx *ctx, const orl_ppo_cfg *cfg, double *dev_out, void *stream);

/* Host only: fill host_out (optional) from a host copy of orl_finalize_async's
 * vector (double[ORL_FINAL_N]) and return the status orl_finalize would
 * return (same priority; ratio_guard only enters the message). */
orl_status orl_stats_decode(const double *final_vec, double ratio_guard, orl_stats *host_out);

/* orl_ppo_loss and orl_logits_grad in one pass over the actor logits (NEXT-1,
 * fused): every row is streamed from HBM once for the loss epilogue (kept in L2
 * with an evict_last hint) and re-read from L2 while the next row streams (after
 * its first three 32 KB chunks) for the gradient, so the HBM traffic is about
 * V*elt read + V*elt written per token (reads measured ~1.09x: some re-reads miss L2)
 * instead of 2 V*elt read + V*elt written.  Same arguments and outputs as the
 * two calls, bit for bit; entropy, lse and dloss_dlogp are required here.
 * Rows that are not 16-byte aligned stay fused when every dlogits row is
 * misaligned exactly like its logits row (e.g. both contiguous [B, T, 50257]);
 * other layouts fall back to the two passes. */
orl_status orl_ppo_loss_and_grad(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                                 float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                                 const float *logp_ref, const float *adv, const float *adv_lo,
                                 const float *ret,
                                 const float *v_new, const float *v_old, float *logp_new,
                                 float *entropy, float *lse, float *dloss_dlogp, float *dloss_dv,
                                 uint8_t *flags, void *dlogits, int64_t out_stride_b,
                                 int64_t out_stride_t, int zero_masked, void *stream);

/* ---- NEXT-4: LM head fused with S1 (tensor cores) ---------------------- */

/* The policy's LM head applied to its final hidden states (the actor
 * forward that produces the logits).  Logits row (b,t) is
 *     z[b,t,v] = sum_k hidden[r,k] weight[v,k],   k < d,  v < V,
 * with r = cu_seqlens[seq_offset+b] - cu_seqlens[seq_offset] + t when
 * rows->cu_seqlens is set (packed) and r = b*T + t otherwise, relative to
 * `hidden` (the micro-batch's first row).  The product runs on the tcgen05
 * tensor cores (bf16 inputs, fp32 accumulation) and is reduced on chip to the
 * S1 online state, so the [rows, V] logits are never written to memory.
 * hidden and weight are bf16, 16-byte aligned, with 16-byte aligned row
 * pitches ld_hidden, ld_weight (elements, >= d); ORL_E_ALIGN otherwise.
 * Every r a valid (b,t) maps to must be < R; a row that does not gets NaN
 * outputs and is counted (orl_finalize -> ORL_E_SHAPE, a data error).  Rows of `hidden` that no
 * valid (b,t) maps to are multiplied but do not affect any output. */
typedef struct {
    const void *hidden; /* [R, d] bf16 final hidden states of the micro-batch */
    const void *weight; /* [V, d] bf16 unembedding matrix                     */
    int64_t R;          /* rows of hidden                                     */
    int64_t d;          /* hidden size                                        */
    int64_t V;          /* vocabulary size (= rows of weight)                 */
    int64_t ld_hidden;  /* row pitch of hidden, elements                      */
    int64_t ld_weight;  /* row pitch of weight, elements                      */
} orl_lmhead;

/* orl_logprobs with the logits computed from an LM head: same outputs and
 * options (S1, and S2+S3 when partner_logp is set), x = inv_temp * z.
 * `gathered` receives z[b,t,y] as the fp32 accumulator value. */
orl_status orl_lmhead_logprobs(orl_ctx *ctx, const orl_rows *rows, const orl_lmhead *head,
                               float inv_temp, float *logp, float *entropy, float *lse,
                               float *gathered, const float *partner_logp, int kl_est,
                               double beta_reward, const float *seq_reward, float *kl,
                               float *shaped_reward, void *stream);

/* orl_ppo_loss with the actor logits computed from its LM head (as above). */
orl_status orl_lmhead_ppo_loss(orl_ctx *ctx, const orl_rows *rows, const orl_lmhead *head,
                               float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                               const float *logp_ref, const float *adv, const float *adv_lo,
                               const float *ret,
                               const float *v_new, const float *v_old, float *logp_new,
                               float *entropy, float *lse, float *dloss_dlogp, float *dloss_dv,
                               uint8_t *flags, void *stream);

/* ---- C1 / C2 as single kernels over peer memory (NVLink / NVSwitch) ---- */

/* The two exchanges of the path (C1 = every rank's whitening
 * partial before the actor pass; C2 = every rank's loss/stat partial,
 * S:216) can run as ONE kernel each instead of local kernel + NCCL
 * all-gather + merge kernel: the kernel forms the rank's partial, stores it
 * into its slot of every rank's exchange buffer through peer (NVLink)
 * mappings, publishes an epoch flag with a release store, waits until every
 * rank's flag has arrived, and merges the slots in rank order (the same
 * merge code as the NCCL path, so all ranks get bit-identical results, equal
 * to the NCCL path's).  Setup, once per context, collective over the ranks:
 *   orl_peer_handle  -> ORL_PEER_HANDLE_BYTES (host) naming this context's
 *                       exchange buffer (a cudaIpcMemHandle_t); the caller
 *                       all-gathers the handles (e.g. torch.distributed);
 *   orl_peer_open    <- the world handles in rank order (host); maps the
 *                       peers' buffers and switches C1/C2 to this transport.
 * Requires world <= 8 (one NVLink domain; ORL_E_INVALID_ARG otherwise) and
 * peer access between the ranks' devices (ORL_E_CUDA if a mapping fails; the
 * context then keeps its NCCL transport).  A wait that exceeds the spin limit
 * (env ORL_PEER_SPIN_LIMIT polls, default ~40 M) gives NaN statistics and
 * orl_finalize returns ORL_E_NCCL. */
#define ORL_PEER_HANDLE_BYTES 64
orl_status orl_peer_handle(orl_ctx *ctx, unsigned char *handle_out);
orl_status orl_peer_open(orl_ctx *ctx, const unsigned char *handles);
/* Select the C1/C2 transport: 0 = NCCL all-gather (needs a communicator),
 * 1 = peer-memory kernels (needs orl_peer_open).  world == 1 ignores it. */
orl_status orl_set_collective(orl_ctx *ctx, int mode);
/* Current transport (0 or 1), -1 for a NULL ctx. */
int orl_get_collective(const orl_ctx *ctx);

/* ---- NEXT-3: adaptive KL coefficient and early stop (host only) -------- */

/* Host scalar update, no device work ("adaptive KL penalty
 * coefficients" and "early stopping criteria based on KL divergence
 * thresholds"):
 *   beta <- beta * (1 + clip(observed_kl / target - 1, -0.5, 0.5) / horizon)
 *   *early_stop = observed_kl > max_kl
 * observed_kl is a statistic of orl_finalize chosen by the caller (e.g. kl for
 * the reference KL, approx_kl_old for the old-policy KL).  Requires beta >= 0,
 * target > 0, horizon > 0, finite observed_kl (ORL_E_INVALID_ARG otherwise). */
orl_status orl_kl_controller_step(double *beta, double target, double horizon, double observed_kl,
                                  double max_kl, int *early_stop);

/* ---- collective boundary hooks (testing / custom transports) ----------- */

/* which = 0: this rank's whitening partial (double[4]: count, mean, M2,
 *            sequences with L_b > 0), valid after orl_advantages;
 * which = 1: this rank's loss/stat partial (double[ORL_PARTIALS_N]), valid
 *            after the last orl_ppo_loss.
 * Copies it to host memory `host_out` (synchronises `stream`). */
orl_status orl_export_partials(orl_ctx *ctx, int which, double *host_out, void *stream);

/* Supplies the gathered partials of `world` ranks (host, [world][4] or
 * [world][ORL_PARTIALS_N], rank order) in place of the NCCL all-gather for the
 * next orl_whiten_stats (which = 0) or orl_finalize (which = 1) on this
 * context.  Lets one process emulate n ranks on one GPU with the exact
 * device merge the NCCL path runs. */
orl_status orl_import_partials(orl_ctx *ctx, int which, const double *host_all, int world,
                               void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ORL_H */

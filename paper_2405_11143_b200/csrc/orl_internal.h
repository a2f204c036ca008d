// orl_internal.h -- host/device contract between the C-ABI layer (orl_api.cu)
// and the kernels (k1_logprobs.cu, k3_advantages.cu, k6_stats.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace orl {

// K1 modes: S1 (+ the S2/S3 reward epilogue when `partner` is set) or the
// actor pass with the S7-S9 loss epilogue.
enum K1Mode { kModeLogprob = 0, kModeLoss = 1, kModeLossGrad = 2 };

// Loss-partial vector (fp64), one per CTA and per context accumulator:
//  0 n  1 sum obj  2 sum vl  3 sum H  4 sum k(new,ref)  5 n clipped
//  6 n value-clipped  7 sum k3(old-new)  8 sum rho  9 n guard
//  10 n non-finite loss terms
//  11..14 per-sequence-mean sums (NEXT-2): sum obj/L_b, vl/L_b, H/L_b, k/L_b
constexpr int kNumPartials = 15;
// Whitening/count vector on the device: N_global, mu, sigma, apply, N_seq, 0, 0, 0
constexpr int kWhitenSlots = 8;
// Device error counters (uint64): 0 token out of range, 1 non-finite S1 rows,
// 2 invalid lengths (L_b < 0 or > T; counted once per iteration, by K3 over the
// whole rank batch -- K1/K5 clamp silently), 3 non-prefix attention-mask rows
// (orl_lengths_from_mask), 4 LM-head rows a valid (b,t) maps to but the hidden
// matrix does not hold (K6 merge).
constexpr int kNumErr = 5;

struct K1Params {
    const char *base;  // logits of the micro-batch's first sequence
    int64_t V, stride_b, stride_t;  // elements
    int64_t row_bytes;
    int elt;            // 2 (bf16) or 4 (fp32)
    int unaligned;      // TMA kernel, rows not 16-byte aligned / sized: stream each row's aligned
                        // interior, load the < 16-byte head and tail with scalar loads
    float inv_temp;
    float c2;           // inv_temp * log2(e)
    int poly;           // MUFU offload: every poly-th element pair uses the FMA-pipe exp2 (0 = off)
    int B, T;
    int64_t seq_offset;
    const int32_t *tokens, *lengths;
    const int32_t *cu_seqlens;  // packed varlen logits (NEXT-2), else NULL
    float *logp, *entropy, *lse, *gathered;
    // S2+S3 reward epilogue (reference pass)
    const float *partner;
    int kl_est;
    double beta_reward;
    const float *seq_reward;
    float *kl_out, *shaped;
    // S7-S9 loss epilogue (actor pass)
    const float *logp_old, *logp_ref, *adv, *ret, *v_new, *v_old;
    const float *adv_lo;  // optional low part: A = adv + adv_lo (~48-bit advantages, orl_advantages)
    float *dlogp, *dv;
    uint8_t *flags;     // optional per-token decisions: bit 0 clipped (Z16), 1 value-clipped,
                        // 2 ratio guard (Z22), 3 non-finite loss term; masked positions 0
    double eps_low, eps_high, eps_v, c1, beta_loss, ratio_guard;
    int kl_loss_est, kl_in_loss, loss_agg;
    const double *whiten;  // device [kWhitenSlots]: N_global, mu, sigma, apply, N_seq
    // kModeLossGrad (NEXT-1 fused): dL/dlogits written in the same launch
    void *dlogits;
    int64_t out_stride_b, out_stride_t;
    double c2_ent;         // entropy coefficient of the total loss
    int zero_masked_grad;
    const int32_t *cum_global;  // prefix of the micro-batch lengths (large B), else NULL
    int pdl_chain;              // 1: the caller vouches that the preceding kernel on the stream wrote
                                // none of this launch's inputs after an early PDL trigger (orl_set_pdl_chain):
                                // only the epilogue warps wait for it; 0: every warp waits first
    // NEXT-4 merge (k6_merge_kernel): per-split partials of the LM-head GEMM
    const float4 *lm_parts;     // [lm_nsplit][lm_stride] (m, s, u, z_y) per hidden row
    int64_t lm_stride;          // rows per split slab (>= lm_R)
    int64_t lm_R;               // hidden rows
    int lm_nsplit, lm_split_cols;  // splits, vocab columns per split
    // accounting
    double *ws;            // [kNumPartials][ws_stride] per-CTA partials
    int ws_stride;
    unsigned int *ticket;  // last-CTA ticket (self-resetting)
    double *acc;           // [kNumPartials] context accumulator
    unsigned long long *err;  // [kNumErr]
};

// Launch K1.  Returns the CUDA launch error.  `tma` selects the TMA bulk-copy
// kernel (requires 16-byte aligned rows and row_bytes % 16 == 0).
cudaError_t launch_k1(const K1Params &p, bool tma, int mode, int num_sms, cudaStream_t s);
// Micro-batches with more sequences than this keep the length prefix in global
// memory (written by launch_lengths_prefix) instead of shared memory.
constexpr int kSmemPrefixMax = 1024;
cudaError_t launch_lengths_prefix(const int32_t *lengths, int B, int T, int32_t *cum,
                                  unsigned long long *err, cudaStream_t s);
// Shared-memory footprint of the TMA kernel for B sequences.
size_t k1_tma_smem_bytes(int B);

// K5 (NEXT-1): dL/dlogits streaming pass.
struct K5Params {
    const char *base;  // actor logits of the micro-batch's first sequence
    void *out;         // dlogits, same dtype and V
    int64_t V, stride_b, stride_t, out_stride_b, out_stride_t;  // elements
    int elt;
    float inv_temp;
    float c2x;         // inv_temp * log2(e)
    double c2;         // entropy coefficient of the total loss
    int B, T;
    int64_t seq_offset;
    const int32_t *tokens, *lengths;
    const int32_t *cu_seqlens;           // packed varlen logits / dlogits, else NULL
    const float *lse, *entropy, *dlogp;  // saved by the actor pass
    const double *whiten;                // device [kWhitenSlots]: N_global first, N_seq at 4
    const int32_t *cum_global;           // prefix of the micro-batch lengths (large B), else NULL
    int zero_masked;
    int loss_agg;                        // 0 token mean, 1 sequence mean (NEXT-2)
    int unaligned;                       // TMA over each row's 16-byte aligned interior (input and
                                         // output rows equally misaligned), scalar head / tail
};
cudaError_t launch_k5(const K5Params &p, bool tma, int num_sms, cudaStream_t s);
size_t k5_smem_bytes(int B);

// K6 (NEXT-4): LM-head GEMM (tcgen05) + online LSE partials.
constexpr int kLmTileN = 256;  // vocab columns per UMMA tile
struct K6Params {
    int64_t R;          // hidden rows (TMA map height)
    int d, V;           // hidden size, vocabulary
    int m_tiles, n_tiles, tiles_per_split, n_split, grid, two_sm;  // filled by k6_plan
    int m_group;        // M units (pairs / tiles) per schedule group (k6_plan)
    int pol_a, pol_b;   // L2 policies of the h / W loads: 0 normal, 1 evict_last, 2 evict_first
    float c2;           // inv_temp * log2(e)
    int B, T;
    int64_t seq_offset;
    const int32_t *tokens, *lengths, *cu_seqlens;
    float4 *parts;      // [n_split][part_stride]
    int64_t part_stride;
};
void k6_plan(K6Params &p, int num_sms);
// hidden [R, d] and weight [V, d] bf16 with row pitches in elements (16-byte aligned rows).
cudaError_t launch_k6(const K6Params &p, const void *hidden, int64_t ld_hidden, const void *weight,
                      int64_t ld_weight, cudaStream_t s);
// Merge the K6 partials of every valid row and run K1's row epilogue (mode 0 or 1).
cudaError_t launch_k6_merge(const K1Params &p, int mode, int num_sms, cudaStream_t s);

struct K3Params {
    int B, T, kind, G;
    double gamma, lambda;
    const int32_t *lengths;
    const float *shaped, *values, *seq_reward;
    float *adv, *ret;
    float *adv_lo;     // optional: A - (float)A, so adv + adv_lo carries the fp64 scan value
    uint8_t *keep;
    double *seq_part;  // [B][3]: n_b, mean_b, M2_b of the stored advantages (adv + adv_lo)
    unsigned long long *err;
};
cudaError_t launch_k3(const K3Params &p, cudaStream_t s);

// Whitening: merge per-sequence partials [B][3] in order into the rank partial
// (count, mean, M2) -> gather[rank*4 ...].
// ---- C1 / C2 over peer memory (one kernel each: local partial -> NVLink stores
// into every rank's exchange buffer -> flag wait -> rank-ordered merge).
constexpr int kPeerMax = 8;  // one NVLink/NVSwitch domain
// exchange buffer (64-bit words), double-buffered by epoch parity:
constexpr int kXW = 0;                                   // [2][kPeerMax][4]      whitening partials
constexpr int kXS = kXW + 2 * kPeerMax * 4;              // [2][kPeerMax][24]     stats partials
constexpr int kXFW = kXS + 2 * kPeerMax * 24;            // [2][kPeerMax]         C1 flags (= epoch)
constexpr int kXFS = kXFW + 2 * kPeerMax;                // [2][kPeerMax]         C2 flags
constexpr int kXWords = kXFS + 2 * kPeerMax;
struct PeerArgs {
    unsigned long long *x[kPeerMax];  // every rank's exchange buffer, mapped in this process
    int world, rank;
    unsigned long long *epoch;        // device counter of this collective (C1: [0], C2: [1]); the
                                      // kernel uses *epoch + 1 and stores it back (graph-replay safe)
    long long spin_limit;             // polls before a wait gives up (flags[2] += 1)
};
cudaError_t launch_whiten_peer(const double *seq_part, int B, const PeerArgs &pa, int want, double *whiten,
                               double *flags, cudaStream_t s);
cudaError_t launch_stats_peer(const double *acc, const unsigned long long *err, const PeerArgs &pa,
                              const double *whiten, double *flags, double c1, double c2, double beta_loss,
                              int kl_in_loss, int loss_agg, double *stats_out, cudaStream_t s);
cudaError_t launch_keep_compact(const uint8_t *keep, int64_t n, int32_t *idx, int32_t *count, cudaStream_t s);
cudaError_t launch_mask_lengths(const uint8_t *mask, int64_t B, int64_t T, int32_t *lengths,
                                unsigned long long *err, cudaStream_t s);
cudaError_t launch_whiten_local(const double *seq_part, int B, double *gather_slot, cudaStream_t s);
// Merge gathered [world][4] rank partials in rank order -> whiten[4] =
// {N, mu, sigma, apply}; warn flag into flags[0].
cudaError_t launch_whiten_merge(const double *gather, int world, int want_whiten, double *whiten,
                                double *flags, cudaStream_t s);

// Fold the error counters into the loss accumulator copy for the collective:
// out[kStatsSlots] = acc[0..14], err[0..kNumErr) -> slots 16.. (ORL_PARTIALS_N in orl.h).
constexpr int kStatsSlots = 24;
static_assert(16 + kNumErr <= kStatsSlots, "error counters fit the stats partial");
constexpr int kStatsOut = 16;  // final stats vector (ORL_STATS_N)
cudaError_t launch_stats_pack(const double *acc, const unsigned long long *err, double *out,
                              cudaStream_t s);
// Sum gathered [world][16] in rank order and form the stats vector.
cudaError_t launch_stats_final(const double *gather, int world, const double *whiten,
                               const double *flags, double c1, double c2, double beta_loss,
                               int kl_in_loss, int loss_agg, double *stats_out, cudaStream_t s);

}  // namespace orl

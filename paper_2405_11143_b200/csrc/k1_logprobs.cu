// k1_logprobs.cu -- K1: streaming full-vocabulary log-softmax + target gather +
// entropy over [B,T,V] logits, with the S2/S3 reward epilogue (reference pass)
// or the S7-S9 PPO-loss epilogue (actor pass).
//
//   lse = ln sum_v exp(x_v), logp = x_y - lse, H = -sum_v p_v ln p_v
//
//
// B200 design: the path is HBM-bound (every logit is read
// exactly once, ~0.013% of the bytes are anything else), so K1 is a
// persistent, warp-specialised streaming kernel:
//   * 1 CTA per SM: 16 consumer warps + 1 producer warp + 2 epilogue warps
//     (608 threads, ~217 KB shared memory).
//   * The producer's elected lane streams each row in 32 KB chunks with 1-D
//     TMA bulk copies (cp.async.bulk ... complete_tx, L2 evict_first) into a
//     6-stage shared-memory ring guarded by full/empty mbarriers: ~192 KB in
//     flight per SM (Little's law needs ~45 KB at ~7 TB/s).
//   * Consumers copy their 4 x 16 B of a chunk to registers with conflict-free
//     128-bit ld.shared, hand the stage back at once (every thread arrives on
//     the stage's empty barrier), and keep a per-thread online (max, sum,
//     first-moment) state in log2 units with packed f32x2 FMA/ADD
//     (FFMA2/FADD2), one MUFU.EX2 per element; m is seeded from the thread's
//     first vector, a chunk is summed into fresh partials that join the row
//     state only if the fast pass held, else the chunk is redone exactly.
//   * Fused actor pass (loss + dL/dlogits): the backward of row i-1 re-reads
//     the row from L2 after 3 forward chunks of row i; the epilogue publishes
//     the row's gradient constants early (ratio chain beside the lse chain,
//     per-row terms computed before the row arrives).
//   * Row end: every consumer thread's state goes into a 4-slot row ring
//     (mbarrier protected); the two epilogue warps take alternate rows, merge
//     the 512 states in a fixed order and run the fp64 epilogue while the
//     consumers already stream the next row.  Side inputs of the epilogue are
//     loaded before the row's merge so their latency hides under the row.
//   * Valid rows are enumerated compactly (prefix sum of lengths in smem) and
//     dealt round-robin to CTAs: equal work per CTA, masked rows never read.
//   * Loss partials: fp64 per epilogue warp in smem, per CTA in a workspace,
//     reduced in fixed order by the last CTA (ticket) -> deterministic, no
//     extra launch.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "orl_device.cuh"
#include "orl_internal.h"

namespace orl {

// mbarrier wait with an explicit suspend-time hint (ns): a waiting warp is parked until
// the phase completes or the hint expires instead of re-polling (fewer issue slots and
// less energy under the power cap).  NS = 0: the default polling wait.
#ifndef ORL_K1_EPI_WAIT_NS
#define ORL_K1_EPI_WAIT_NS 0
#endif
#ifndef ORL_K1_CONS_WAIT_NS
#define ORL_K1_CONS_WAIT_NS 0
#endif
template <int NS>
__device__ __forceinline__ void mbar_wait_hint(uint64_t *bar, uint32_t parity) {
    if (NS == 0) {
        mbar_wait(bar, parity);
        return;
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(NS)
        : "memory");
}

// Launch shape (tunable at build time; defaults are the measured best, DESIGN 5.1).
#ifndef ORL_K1_CONSUMER_WARPS
#define ORL_K1_CONSUMER_WARPS 16
#endif
#ifndef ORL_K1_CHUNK
#define ORL_K1_CHUNK 32768
#endif
#ifndef ORL_K1_STAGES
#define ORL_K1_STAGES 6
#endif
#ifndef ORL_K1_MINBLOCKS
#define ORL_K1_MINBLOCKS 1
#endif
#ifndef ORL_K1_EPI_WARPS
#define ORL_K1_EPI_WARPS 2
#endif
constexpr int kConsumerWarps = ORL_K1_CONSUMER_WARPS;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kProducerWarp = kConsumerWarps;      // TMA issue
constexpr int kEpilogueWarp = kConsumerWarps + 1;  // first of the merge + fp64 epilogue warps
constexpr int kEpiWarps = ORL_K1_EPI_WARPS;         // rows alternate between them
// Fused actor pass: dlogits of full backward chunks written back into the chunk's stage and
// stored by a TMA bulk copy from a dedicated store warp (n > 0: every n-th chunk of a row,
// the others by STG.128), or STG.128 from the consumer threads only (0).
#ifndef ORL_K1_BWD_TMA_STORE
#define ORL_K1_BWD_TMA_STORE 0
#endif
constexpr bool kTmaStore = ORL_K1_BWD_TMA_STORE != 0;
constexpr int kTmaStoreEvery = ORL_K1_BWD_TMA_STORE > 0 ? ORL_K1_BWD_TMA_STORE : 1;
#ifndef ORL_K1_STORE_WAIT_NS
#define ORL_K1_STORE_WAIT_NS 20000  // the store warp parks while the consumers compute a chunk
#endif
constexpr int kStoreWarp = kConsumerWarps + 1 + ORL_K1_EPI_WARPS;
constexpr int kThreads = kConsumers + 32 + 32 * kEpiWarps + (kTmaStore ? 32 : 0);
constexpr int kChunk = ORL_K1_CHUNK;  // bytes per TMA stage
constexpr int kStages = ORL_K1_STAGES;
// Row-partial ring (consumers -> epilogue warps).  Row rl uses slot rl % kSlots
// and epilogue warp rl % kEpiWarps; kSlots is a multiple of kEpiWarps so every
// slot is always drained by the same warp, in order (parity waits stay exact).
constexpr int kSlots = kEpiWarps * (kEpiWarps == 1 ? 3 : 2);
constexpr int kRowInfo = 16;   // row-info ring (producer -> consumers), >= kStages + 1
constexpr int kVecPerThread = kChunk / 16 / kConsumers;  // 16-byte vectors per thread per chunk
constexpr int kW = 4 * kVecPerThread;                    // 32-bit words per thread per chunk
static_assert(kVecPerThread >= 1 && kChunk % (16 * kConsumers) == 0, "chunk must split evenly");
static_assert((kW & (kW - 1)) == 0, "words per thread must be a power of two");
static_assert(kRowInfo >= kStages + 1, "row-info ring must outrun the stage ring");

// Every consumer thread's online state for one row, plus the target logit.
struct RowSlot {
    float m[kConsumers], s[kConsumers], u[kConsumers];
    float target;
    float pad[31];
};

// Backward row constants (kModeLossGrad): published by the epilogue warp of the
// row, read by the consumers when they stream the row a second time (from L2).
struct GradRow {
    int64_t out_off;  // element offset of the dlogits row
    int32_t y;
    float l2;         // lse * log2(e)
    float A1;         // inv_temp * a * ln2,   a = c2/N or c2/(N_seq L_b)
    float A0;         // inv_temp * (a H - w)
    float wt;         // inv_temp * w   (delta term at v = y)
    int32_t pad;
};
constexpr int kGradRows = 4;  // ring; each slot always written by the same epilogue warp
// Fused actor pass: the backward of row i starts after the first kFusedSplit
// chunks of row i+1's forward (0 = right after row i: the re-read is an L2 hit
// but the consumers wait for row i's epilogue; the full row = a one-row lag,
// which re-reads from HBM because ~76 MB of traffic separates the two touches).
#ifndef ORL_K1_FUSED_SPLIT
#define ORL_K1_FUSED_SPLIT 3
#endif
constexpr int kFusedSplit = ORL_K1_FUSED_SPLIT;
// Stage release: every consumer thread arrives on the stage's empty barrier after its
// shared-memory loads (1), or lane 0 of each warp after a __syncwarp (0).
#ifndef ORL_K1_THREAD_ARRIVE
#define ORL_K1_THREAD_ARRIVE 1
#endif
constexpr int kEmptyArrivals = ORL_K1_THREAD_ARRIVE ? kConsumers : kConsumerWarps;
__device__ __forceinline__ void release_stage(uint64_t *empty, int lane) {
#if ORL_K1_THREAD_ARRIVE
    (void)lane;
    mbar_arrive(empty);  // release: this thread's loads of the stage happen before
#else
    __syncwarp();
    if (lane == 0) mbar_arrive(empty);
#endif
}
#ifdef ORL_K1_PROF  // latency probes of the fused pass (tools only; not in the product build)
__device__ unsigned long long g_k1prof[8];
#define K1PROF(i, v) atomicAdd(&g_k1prof[i], (unsigned long long)(v))
#else
#define K1PROF(i, v) ((void)0)
#endif

struct __align__(128) K1Smem {
    uint8_t stage[kStages][kChunk];
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t row_full[kSlots];
    uint64_t row_empty[kSlots];
    int32_t row_y[kRowInfo];
    int32_t row_h[kRowInfo];        // unaligned rows: head bytes before the 16-byte aligned interior
    float row_x[kRowInfo][16];      // unaligned rows: raw head elements, then tail elements
    uint64_t grad_full[kGradRows];
    GradRow grad[kGradRows];
    uint64_t written[kStages];      // kTmaStore: consumers -> store warp, chunk results in the stage
    uint64_t st_dst[kStages];       // kTmaStore: global destination of the staged chunk
    RowSlot slot[kSlots];
    double wacc[kEpiWarps][kNumPartials];
};

size_t k1_tma_smem_bytes(int B) {
    return sizeof(K1Smem) + sizeof(int32_t) * (size_t)((B > kSmemPrefixMax ? 0 : B) + 32);
}

// Large micro-batches: the inclusive prefix of the clamped lengths is built once
// in global memory by one CTA (the same block scan) and read by every CTA.
__global__ void __launch_bounds__(1024) lengths_prefix_kernel(const int32_t *lengths, int B, int T, int32_t *cum,
                                                              unsigned long long *err) {
    __shared__ int32_t warp_tot[32];
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int per = (B + nthr - 1) / nthr;
    const int beg = min(B, tid * per), end = min(B, beg + per);
    int local = 0, bad = 0;
    for (int b = beg; b < end; ++b) {
        int L = lengths[b];
        if (L < 0 || L > T) ++bad;
        L = L < 0 ? 0 : (L > T ? T : L);
        local += L;
        cum[b] = local;
    }
    if (bad && err) atomicAdd(&err[2], (unsigned long long)bad);
    const int lane = tid & 31, warp = tid >> 5;
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int w = 0; w < nthr / 32; ++w) {
            int v = warp_tot[w];
            warp_tot[w] = run;
            run += v;
        }
    }
    __syncthreads();
    const int excl = warp_tot[warp] + incl - local;
    for (int b = beg; b < end; ++b) cum[b] += excl;
}

cudaError_t launch_lengths_prefix(const int32_t *lengths, int B, int T, int32_t *cum, unsigned long long *err,
                                  cudaStream_t s) {
    lengths_prefix_kernel<<<1, 1024, 0, s>>>(lengths, B, T, cum, err);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- prologue
// Inclusive prefix of the clamped lengths of the micro-batch into cum[0..B).
// Invalid lengths (< 0 or > T) are clamped here and counted once per iteration by K3.
__device__ void build_prefix(const K1Params &p, int32_t *cum, int32_t *warp_tot) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int per = (p.B + nthr - 1) / nthr;
    const int beg = min(p.B, tid * per), end = min(p.B, beg + per);
    int local = 0;
    for (int b = beg; b < end; ++b) {
        int L = p.lengths[p.seq_offset + b];
        L = L < 0 ? 0 : (L > p.T ? p.T : L);
        local += L;
        cum[b] = local;
    }
    // exclusive scan of the per-thread totals across the block
    const int lane = tid & 31, warp = tid >> 5;
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (tid == 0) {
        int run = 0;
        for (int w = 0; w < (nthr + 31) / 32; ++w) {
            int v = warp_tot[w];
            warp_tot[w] = run;
            run += v;
        }
    }
    __syncthreads();
    const int excl = warp_tot[warp] + incl - local;
    for (int b = beg; b < end; ++b) cum[b] += excl;
    __syncthreads();
}

// Write exact zeros to every output at the masked positions of the call.
// (blk, nblk): this block's index among the blocks sharing the work (default: the grid).
__device__ void zero_masked(const K1Params &p, const int32_t *cum, int lt, int nthr, int mode, int64_t blk = -1,
                            int64_t nblk = -1) {
    if (blk < 0) {
        blk = blockIdx.x;
        nblk = gridDim.x;
    }
    const int64_t total = (int64_t)p.B * p.T;
    for (int64_t q = blk * nthr + lt; q < total; q += nblk * nthr) {
        const int b = (int)(q / p.T), t = (int)(q % p.T);
        const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
        if (t < L) continue;
        const int64_t i = (p.seq_offset + b) * (int64_t)p.T + t;
        if (p.logp) p.logp[i] = 0.f;
        if (p.entropy) p.entropy[i] = 0.f;
        if (p.lse) p.lse[i] = 0.f;
        if (p.gathered) p.gathered[i] = 0.f;
        if (mode == kModeLogprob) {
            if (p.kl_out) p.kl_out[i] = 0.f;
            if (p.shaped) p.shaped[i] = 0.f;
        } else {
            if (p.dlogp) p.dlogp[i] = 0.f;
            if (p.dv) p.dv[i] = 0.f;
            if (p.flags) p.flags[i] = 0;
        }
    }
}

// ---------------------------------------------------------------- epilogue
// Side inputs of one row (loaded ahead of time): loss mode {logp_old,
// logp_ref, adv, ret, v_new, v_old, adv_lo}; logprob mode {partner, seq_reward}.
constexpr int kSide = 7;
__device__ __forceinline__ float load_side(const K1Params &p, int mode, int k, int64_t i, int b) {
    const float *ptr = nullptr;
    int64_t idx = i;
    if (mode != kModeLogprob) {
        ptr = k == 0 ? p.logp_old : k == 1 ? p.logp_ref : k == 2 ? p.adv : k == 3 ? p.ret
            : k == 4 ? p.v_new : k == 5 ? p.v_old : k == 6 ? p.adv_lo : nullptr;
    } else {
        if (k == 0) ptr = p.partner;
        if (k == 1) { ptr = p.seq_reward; idx = p.seq_offset + b; }
    }
    return ptr ? __ldg(ptr + idx) : 0.f;
}

// fp64 per-row epilogue (runs on one thread).  `tot` is the merged online
// state of the row, `target` the raw logit x[b,t,y] (as float, exact).
// Quantities the fused backward needs from the forward epilogue of a row.
struct EpiOut {
    float lse, H, w;
};

// publish(eo) runs as soon as (lse, H, w) are known, before the rest of the loss
// terms: the fused backward waits for exactly these.
struct NoPublish {
    __device__ void operator()(const EpiOut &) const {}
};
// Per-row quantities of the actor epilogue that do not depend on the logits row
// (whitened advantage, 1/N, the entropy coefficient a of the backward): the TMA
// kernel computes them before it waits for the row, off the backward's critical path.
struct RowPre {
    double A, invN;
    float a;
};
__device__ __forceinline__ RowPre row_pre(const K1Params &p, int L, const float *side, const double *wh) {
    RowPre r;
    // derivatives are per token of the token mean (1/N) or, NEXT-2 sequence mean (Z31),
    // of the mean of per-sequence means (1/(N_seq L_b))
    const double N = p.loss_agg == 1 ? wh[4] * (double)L : wh[0];
    r.invN = 1.0 / N;
    double A = (double)side[2] + (double)side[6];  // adv (+ its low part, 0 when not given)
    if (wh[3] != 0.0) A = (A - wh[1]) / (wh[2] + 1e-8);
    r.A = A;
    // same fp32 constant as K5 (orl_logits_grad) computes from the saved arrays
    r.a = (float)(p.loss_agg == 1 ? p.c2_ent / (wh[4] * (double)L) : p.c2_ent / wh[0]);
    return r;
}

template <int MODE, typename Publish = NoPublish>
__device__ void row_epilogue(const K1Params &p, int b, int t, int L, int y, Online tot,
                             float target, const float *side, const double *wh, double *wacc,
                             EpiOut *eo = nullptr, const Publish &publish = Publish(),
                             const RowPre *pre = nullptr) {
    const int64_t i = (p.seq_offset + b) * (int64_t)p.T + t;
    const bool oob = (y < 0) || (y >= p.V);
    const double log2s = log2((double)tot.s);
    double lse = kLn2 * ((double)tot.m + log2s);
    double H = kLn2 * (log2s - (double)tot.u / (double)tot.s);
    double logp = (double)target * (double)p.inv_temp - lse;
    const bool dead = tot.m / p.c2 < 0.5f * kNegClampF32;  // every logit -inf
    if (oob) {
        atomicAdd(&p.err[0], 1ull);
        lse = H = logp = __longlong_as_double(0x7ff8000000000000ll);
    } else if (dead || !(isfinite(lse) && isfinite(logp) && isfinite(H))) {
        atomicAdd(&p.err[1], 1ull);
        if (dead) lse = H = logp = __longlong_as_double(0x7ff8000000000000ll);
    }
    const float logp_f = (float)logp, H_f = (float)H;
    auto store_row = [&]() {
        p.logp[i] = logp_f;
        if (p.entropy) p.entropy[i] = H_f;
        if (p.lse) p.lse[i] = (float)lse;
        if (p.gathered) p.gathered[i] = oob ? __int_as_float(0x7fc00000) : target;
    };

    if (MODE == kModeLogprob) {
        store_row();
        if (p.partner) {
            // S2 + S3 (Z4, Z7): d = logp_old - logp_ref,
            // r'_t = [t = L_b - 1] R_b - beta k(d)
            const double d = (double)side[0] - (double)logp_f;
            const double k = kl_est(d, p.kl_est);
            if (p.kl_out) p.kl_out[i] = (float)k;
            if (p.shaped) {
                const double r = (t == L - 1) ? (double)side[1] : 0.0;
                p.shaped[i] = (float)(r - p.beta_reward * k);
            }
        }
        return;
    } else {
        // S7-S9 (Z11-Z17, Z22, Z38), all in fp64.
        const RowPre pr = pre ? *pre : row_pre(p, L, side, wh);
        const double A = pr.A;
        const double lpo = side[0];
        // The loss terms use the stored fp32 log-prob lpn (Z38), as every consumer of the
        // per-token outputs does.  The ratio rho = exp(lpn - logp_old) is evaluated as
        //   exp(x_y / T - logp_old - ln2 m) / s  *  exp(lpn - logp),
        // the first factor (= exp(logp - logp_old)) on a chain that does not wait for log2(s),
        // side by side with the lse chain, the second from |lpn - logp| <= 2^-24 |logp| as
        // 1 + d + d^2 / 2 (error < d^3 ~ 1e-21): the fused backward (which needs lse, H and w)
        // starts sooner, and rho matches exp(lpn - logp_old) to fp64 rounding.
        const double lpn = (double)logp_f;
        const double rho_x = exp((double)target * (double)p.inv_temp - lpo - kLn2 * (double)tot.m) / (double)tot.s;
        double rho;
        if (oob || dead || !isfinite(logp)) {
            rho = exp(lpn - lpo);
        } else {
            const double d = lpn - logp;
            rho = rho_x * fma(d, fma(d, 0.5, 1.0), 1.0);
        }
        const double rc = fmin(fmax(rho, 1.0 - p.eps_low), 1.0 + p.eps_high);
        const double unc = rho * A, clt = rc * A;
        const bool clipped = clt < unc;
        const double obj = clipped ? clt : unc;
        double dr = 0.0, dkref = 0.0;
        if (p.logp_ref) {
            dr = lpn - (double)side[1];
            dkref = kl_grad(dr, p.kl_loss_est);
        }
        const float wf = (float)(((clipped ? 0.0 : -rho * A) + (p.kl_in_loss ? p.beta_loss * dkref : 0.0)) * pr.invN);
        if (eo) {
            eo->lse = (float)lse;
            eo->H = H_f;
            eo->w = wf;
            publish(*eo);
        }
        store_row();
        double vl = 0.0, dvl = 0.0;
        bool vclipped = false;
        if (p.v_new) {
            const double vn = side[4], vo = side[5], R = side[3];
            const double e1 = vn - R;
            if (p.eps_v > 0.0) {
                const double dvv = vn - vo;
                const double dvc = fmin(fmax(dvv, -p.eps_v), p.eps_v);
                const double e2 = vo + dvc - R;
                vclipped = (e2 * e2) > (e1 * e1);
                vl = vclipped ? e2 * e2 : e1 * e1;
                dvl = vclipped ? (fabs(dvv) < p.eps_v ? 2.0 * e2 : 0.0) : 2.0 * e1;
            } else {
                vl = e1 * e1;
                dvl = 2.0 * e1;
            }
        }
        const double kref = p.logp_ref ? kl_est(dr, p.kl_loss_est) : 0.0;
        const double k3old = kl_est(lpo - lpn, 3);
        const double Hd = (double)H_f;
        const double dold = lpn - lpo;
        wacc[0] += 1.0;
        wacc[1] += obj;
        wacc[2] += vl;
        wacc[3] += Hd;
        wacc[4] += kref;
        wacc[5] += clipped ? 1.0 : 0.0;
        wacc[6] += vclipped ? 1.0 : 0.0;
        wacc[7] += k3old;
        wacc[8] += rho;
        const bool guard = fabs(dold) > p.ratio_guard;
        const bool nonfin = !(isfinite(obj) && isfinite(vl) && isfinite(Hd) && isfinite(kref));
        if (guard) wacc[9] += 1.0;
        if (nonfin) wacc[10] += 1.0;
        if (p.flags)
            p.flags[i] = (uint8_t)((clipped ? 1u : 0u) | (vclipped ? 2u : 0u) | (guard ? 4u : 0u) | (nonfin ? 8u : 0u));
        const double invL = 1.0 / (double)L;
        wacc[11] += obj * invL;
        wacc[12] += vl * invL;
        wacc[13] += Hd * invL;
        wacc[14] += kref * invL;
        if (p.dlogp) p.dlogp[i] = wf;
        if (p.dv) p.dv[i] = (float)(p.c1 * dvl * pr.invN);
    }
}

// ---------------------------------------------------------------- CTA partials
// Deterministic reduction of the loss partials: per-warp smem accumulators
// summed in warp order, per-CTA partials summed in CTA order by the last CTA.
__device__ void finish_partials(const K1Params &p, double (*wacc)[kNumPartials], int nwarps,
                                int lt, int nthr, int bar_id) {
    __shared__ double scratch[8][kNumPartials];
    if (bar_id >= 0) named_bar_sync(bar_id, nthr);
    else __syncthreads();
    if (lt < kNumPartials) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) s += wacc[w][lt];
        p.ws[(size_t)lt * p.ws_stride + blockIdx.x] = s;
    }
    __threadfence();
    if (bar_id >= 0) named_bar_sync(bar_id, nthr);
    else __syncthreads();
    __shared__ unsigned int s_last;
    if (lt == 0) s_last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    if (bar_id >= 0) named_bar_sync(bar_id, nthr);
    else __syncthreads();
    if (!s_last) return;
    __threadfence();
    // fixed-shape reduction over CTAs: thread lt sums CTAs lt, lt+nthr, ...
    // per column, then a fixed warp tree and a fixed in-order warp sum.
    const int lane = lt & 31, w = lt >> 5;
    for (int c = 0; c < kNumPartials; ++c) {
        double s = 0.0;
        for (int q = lt; q < (int)gridDim.x; q += nthr)
            s += __ldcg(&p.ws[(size_t)c * p.ws_stride + q]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) scratch[w][c] = s;
    }
    if (bar_id >= 0) named_bar_sync(bar_id, nthr);
    else __syncthreads();
    if (lt < kNumPartials) {
        double s = 0.0;
        for (int q = 0; q < nthr / 32; ++q) s += scratch[q][lt];
        p.acc[lt] += s;
    }
    if (lt == 0) *p.ticket = 0u;
}

// ---------------------------------------------------------------- chunk math
// Per-thread streaming state: running reference m (log2 units) and packed
// (even, odd) accumulators s = sum 2^t, u = sum 2^t t with t = x c - m.
struct ThreadAcc {
    float m;
    uint64_t sA, sB, uA, uB;
};

__device__ __forceinline__ uint64_t bf16x2_to_f32x2(uint32_t w) {
    uint64_t r;
#ifdef ORL_K1_PRMT_UNPACK
    // byte permutes on the ALU pipe (no IMAD on the FMA pipe for the shift)
    asm("{\n\t.reg .b32 lo, hi;\n\tprmt.b32 lo, %1, 0, 0x1044;\n\tprmt.b32 hi, %1, 0, 0x3244;\n\t"
        "mov.b64 %0, {lo, hi};\n\t}" : "=l"(r) : "r"(w));
#else
    asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\t"
        "mov.b64 %0, {lo, hi};\n\t}" : "=l"(r) : "r"(w));
#endif
    return r;
}

// Number of element pairs held in NW raw 32-bit words.
template <typename Tin, int NW> struct Words { static constexpr int kPairs = sizeof(Tin) == 2 ? NW : NW / 2; };

template <typename Tin, int NW>
__device__ __forceinline__ uint64_t pair_at(const uint32_t (&w)[NW], int q) {
    if (sizeof(Tin) == 2) return bf16x2_to_f32x2(w[q]);
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(w[2 * q]), "r"(w[2 * q + 1]));
    return r;
}

// Accumulate every pair of the chunk against the current m (no max, no clamp).
// POLY = k > 0: every k-th pair takes the FMA-pipe polynomial instead of MUFU.
template <typename Tin, bool ENT, int POLY, int NW = kW>
__device__ __forceinline__ void acc_words(ThreadAcc &a, const uint32_t (&w)[NW], uint64_t c2p) {
    const uint64_t nm = pack2(-a.m, -a.m);
#pragma unroll
    for (int q = 0; q < Words<Tin, NW>::kPairs; ++q) {
        const uint64_t tt = ffma2(pair_at<Tin, NW>(w, q), c2p, nm);
        uint64_t e;
        if (POLY > 0 && (q % POLY) == POLY - 1) {
            e = poly_ex2x2(tt);
        } else {
            float t0, t1;
            unpack2(tt, t0, t1);
            e = pack2(ex2(t0), ex2(t1));
        }
        if (q & 1) {
            a.sB = fadd2(a.sB, e);
            if (ENT) a.uB = ffma2(e, tt, a.uB);
        } else {
            a.sA = fadd2(a.sA, e);
            if (ENT) a.uA = ffma2(e, tt, a.uA);
        }
    }
}

// Exact path: clamp -inf (NaN kept), chunk max, rescale, accumulate.  Used for
// the first chunk of every row and to redo a chunk whose fast pass overflowed
// (an element more than 64 log2-units above m), produced a non-finite moment
// (-inf logits in the entropy moment) or saw NaN.
template <typename Tin, bool ENT, int NW = kW>
__device__ __forceinline__ void exact_words(ThreadAcc &a, uint32_t (&w)[NW], float c2, uint64_t c2p) {
    static_assert((NW & (NW - 1)) == 0, "words per thread must be a power of two");
    float cm;
    if (sizeof(Tin) == 2) {
#pragma unroll
        for (int q = 0; q < NW; ++q) w[q] = hmax2_nan(w[q], kNegClampBf16x2);
        uint32_t mx[NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) mx[q] = w[q];
#pragma unroll
        for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int q = 0; q < h; ++q) mx[q] = hmax2_nan(mx[q], mx[q + h]);
        cm = fmax_nan(bf16lo(mx[0]), bf16hi(mx[0]));
    } else {
        cm = kNegClampF32;
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const float f = fmax_nan(__uint_as_float(w[q]), kNegClampF32);
            w[q] = __float_as_uint(f);
            cm = fmax_nan(cm, f);
        }
    }
    const float mn = fmax_nan(a.m, cm * c2);
    const float d = a.m - mn;
    const float r = ex2(d);
    const uint64_t d2 = pack2(d, d), r2 = pack2(r, r);
    if (ENT) {
        a.uA = fmul2(r2, ffma2(d2, a.sA, a.uA));
        a.uB = fmul2(r2, ffma2(d2, a.sB, a.uB));
    }
    a.sA = fmul2(r2, a.sA);
    a.sB = fmul2(r2, a.sB);
    a.m = mn;
    acc_words<Tin, ENT, 0, NW>(a, w, c2p);
}

// True if the fast pass must be redone exactly.
template <bool ENT>
__device__ __forceinline__ bool needs_redo(const ThreadAcc &a) {
    float s0, s1, s2, s3;
    unpack2(fadd2(a.sA, a.sB), s0, s1);
    s2 = s0 + s1;
    bool bad = !(s2 < 1.8446744e19f);  // 2^64; also NaN / inf
    if (ENT) {
        unpack2(fadd2(a.uA, a.uB), s0, s1);
        s3 = s0 + s1;
        bad |= !(fabsf(s3) < 3.0e38f);
    }
    return bad;
}

// Load this thread's 4 x 16 B of the chunk (ragged tail padded with a finite
// very negative logit, so padding gives 2^t = 0 and 2^t t = 0).
template <typename Tin, bool FULL, int NW = kW>
__device__ __forceinline__ void load_words(uint32_t (&w)[NW], const uint8_t *sb, int ct, int nvec) {
    const uint32_t pad = sizeof(Tin) == 2 ? kNegClampBf16x2 : __float_as_uint(kNegClampF32);
#pragma unroll
    for (int k = 0; k < NW / 4; ++k) {
        const int vi = ct + k * kConsumers;
        uint4 v;
        if (FULL || vi < nvec) v = lds128(sb + vi * 16);
        else v = make_uint4(pad, pad, pad, pad);
        w[4 * k + 0] = v.x; w[4 * k + 1] = v.y; w[4 * k + 2] = v.z; w[4 * k + 3] = v.w;
    }
}

template <typename Tin, bool ENT, int POLY, int NW = kW>
__device__ __forceinline__ void process_words(ThreadAcc &a, uint32_t (&w)[NW], bool first, float c2,
                                              uint64_t c2p) {
    if (first) {
        // Row start: seed m with the max of this thread's first 16-byte vector
        // (cheap); the fast pass below redoes the chunk exactly if anything in
        // it lies more than 64 log2-units above that seed.
        float cm;
        if (sizeof(Tin) == 2) {
            const uint32_t m01 = hmax2_nan(hmax2_nan(w[0], kNegClampBf16x2), w[1]);
            const uint32_t m23 = hmax2_nan(w[2], w[3]);
            const uint32_t mx = hmax2_nan(m01, m23);
            cm = fmax_nan(bf16lo(mx), bf16hi(mx));
        } else {
            cm = fmax_nan(fmax_nan(__uint_as_float(w[0]), __uint_as_float(w[1])),
                          fmax_nan(__uint_as_float(w[2]), __uint_as_float(w[3])));
            cm = fmax_nan(cm, kNegClampF32);
        }
        a.m = fmax_nan(cm * c2, kMInit);
    }
#ifndef ORL_K1_CHUNK_PARTIAL
#define ORL_K1_CHUNK_PARTIAL 1
#endif
#if ORL_K1_CHUNK_PARTIAL
    // the chunk is summed into fresh partials and added to the row state only if the
    // fast pass held (no saved copy of the state to restore: fewer moves per chunk)
    ThreadAcc c{a.m, 0ull, 0ull, 0ull, 0ull};
    acc_words<Tin, ENT, POLY, NW>(c, w, c2p);
#if ORL_K1_ABL & 16  // timing ablation: no overflow check (fast pass always accepted)
    if (false) {
#else
    if (needs_redo<ENT>(c)) {
#endif
        exact_words<Tin, ENT, NW>(a, w, c2, c2p);
    } else {
        a.sA = fadd2(a.sA, c.sA);
        a.sB = fadd2(a.sB, c.sB);
        if (ENT) {
            a.uA = fadd2(a.uA, c.uA);
            a.uB = fadd2(a.uB, c.uB);
        }
    }
#else
    const ThreadAcc saved = a;
    acc_words<Tin, ENT, POLY, NW>(a, w, c2p);
    if (needs_redo<ENT>(a)) {
        a = saved;
        exact_words<Tin, ENT, NW>(a, w, c2, c2p);
    }
#endif
}

// One scalar logit (an unaligned row's head or tail element) folded exactly into the
// thread's state: clamp -inf as the exact path does, rescale to a new max if needed,
// accumulate into the even lane of the packed sums.
template <bool ENT>
__device__ __forceinline__ void acc_scalar(ThreadAcc &a, float x, float c2) {
    x = fmax_nan(x, kNegClampF32);
    const float mn = fmax_nan(a.m, x * c2);
    const float d = a.m - mn, r = ex2(d);
    const uint64_t d2 = pack2(d, d), r2 = pack2(r, r);
    if (ENT) {
        a.uA = fmul2(r2, ffma2(d2, a.sA, a.uA));
        a.uB = fmul2(r2, ffma2(d2, a.sB, a.uB));
    }
    a.sA = fmul2(r2, a.sA);
    a.sB = fmul2(r2, a.sB);
    a.m = mn;
    const float t = fmaf(x, c2, -a.m), e = ex2(t);
    a.sA = fadd2(a.sA, pack2(e, 0.f));
    if (ENT) a.uA = ffma2(pack2(e, 0.f), pack2(t, 0.f), a.uA);
}

// Warp-level variant for the TMA kernel (epilogue warp 0 owns the partials).
// The last CTA loads every CTA's partials at once (all loads in flight), then
// sums each column in a fixed order: lane-strided CTA order, then a fixed
// xor-shuffle tree.
__device__ void finish_partials_warp(const K1Params &p, const double (&wacc)[kNumPartials], int lane) {
#pragma unroll
    for (int c = 0; c < kNumPartials; ++c)
        if (lane == c) p.ws[(size_t)c * p.ws_stride + blockIdx.x] = wacc[c];
    __threadfence();
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) last = (atomicAdd(p.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    __threadfence();
    double v[kNumPartials];
#pragma unroll
    for (int c = 0; c < kNumPartials; ++c) v[c] = 0.0;
    for (int q = lane; q < (int)gridDim.x; q += 32) {
        double x[kNumPartials];
#pragma unroll
        for (int c = 0; c < kNumPartials; ++c) x[c] = __ldcg(&p.ws[(size_t)c * p.ws_stride + q]);
#pragma unroll
        for (int c = 0; c < kNumPartials; ++c) v[c] += x[c];
    }
#pragma unroll
    for (int c = 0; c < kNumPartials; ++c) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], off);
    }
    if (lane == 0) {
#pragma unroll
        for (int c = 0; c < kNumPartials; ++c) p.acc[c] += v[c];
        *p.ticket = 0u;
    }
}

// ---------------------------------------------------------------- TMA kernel
// GENT (fused actor pass only): the loss has an entropy term (c2 != 0), so the backward's
// factor is A1 t + A0; with c2 = 0 it is the row constant A0 (one FFMA2 per pair less, and
// a -inf logit gets the exact zero gradient -w p = 0 instead of 0 * (-inf); DESIGN Z39).
template <typename Tin, int MODE, int POLY, bool UNAL = false, bool GENT = true>
__global__ void __launch_bounds__(kThreads, ORL_K1_MINBLOCKS) k1_tma_kernel(const K1Params p) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    K1Smem &S = *reinterpret_cast<K1Smem *>(smem_raw);
    int32_t *cum_s = reinterpret_cast<int32_t *>(smem_raw + sizeof(K1Smem));
    int32_t *warp_tot = cum_s + (p.cum_global ? 0 : p.B);  // 32 ints after the prefix
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifndef ORL_K1_PREMERGE
#define ORL_K1_PREMERGE 1
#endif
#ifndef ORL_K1_ABL
#define ORL_K1_ABL 0  // timing ablations (tools only): 1 fwd math, 2 bwd math, 4 bwd stores, 8 const wait, 16 no overflow check, 32 no fp64 row epilogue
#endif
    // 1: actor passes only; 2: every pass (A/B knob)
    constexpr bool kPremerge = ORL_K1_PREMERGE == 2 || (ORL_K1_PREMERGE == 1 && MODE != kModeLogprob);

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kEmptyArrivals);
        }
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&S.row_full[s], kConsumerWarps);
            mbar_init(&S.row_empty[s], 1);
        }
        for (int s = 0; s < kGradRows; ++s) mbar_init(&S.grad_full[s], 1);
        if (kTmaStore)
            for (int s = 0; s < kStages; ++s) mbar_init(&S.written[s], kConsumers);
        fence_mbar_init();
    }
    if (tid < kEpiWarps * kNumPartials) (&S.wacc[0][0])[tid] = 0.0;
    // Programmatic dependent launch: let the next kernel in the stream start
    // as our CTAs retire (it fills the SMs of this launch's tail).  By default
    // every warp waits for the preceding grid (griddepcontrol.wait) before its
    // first global read, so a predecessor that triggers early (e.g. a GEMM
    // writing the logits) is always complete and visible.  With p.pdl_chain
    // (orl_set_pdl_chain: the caller vouches that the predecessor wrote no
    // input of this launch after an early trigger -- e.g. the previous K1 of the
    // same iteration) only the epilogue warps, which read or write memory other
    // kernels of the path touch, wait; the producer streams the logits at once.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int32_t *cum = p.cum_global ? p.cum_global : cum_s;
    if (!p.pdl_chain || p.cum_global) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.cum_global) __syncthreads();  // prefix written by the prefix kernel just before us
    else build_prefix(p, cum_s, warp_tot);  // contains __syncthreads
    const int64_t N = cum[p.B - 1];
    const int64_t row_bytes = p.row_bytes;

    if (warp == kProducerWarp) {
        // ===================== producer: one lane issues the TMA bulk copies ======
        // kModeLossGrad streams every row twice: forward chunks F(i) (kept in L2
        // with evict_last) and, one row later, the same row again for the backward
        // B(i) (an L2 hit, evict_first): F0, F1, B0, F2, B1, ..., B(n-1).
        if (lane == 0) {
            const uint64_t pol_first = l2_evict_first_policy();
#ifndef ORL_K1_FUSED_FWD_POL
#define ORL_K1_FUSED_FWD_POL 1
#endif

#ifndef ORL_K1_FUSED_BWD_POL
#define ORL_K1_FUSED_BWD_POL 0
#endif
            const uint64_t pol_fwd = MODE != kModeLossGrad ? pol_first
                                     : ORL_K1_FUSED_FWD_POL == 1 ? l2_evict_last_policy()
                                     : ORL_K1_FUSED_FWD_POL == 2 ? l2_evict_normal_policy() : pol_first;
            const uint64_t pol_bwd = ORL_K1_FUSED_BWD_POL == 0 ? pol_first
                                     : ORL_K1_FUSED_BWD_POL == 2 ? l2_evict_normal_policy()
                                     : l2_evict_unchanged_policy();
            int stage = 0;
            uint32_t phase = 0;
            const int64_t n_rows = N > (int64_t)blockIdx.x ? (N - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
            const int64_t nch = (row_bytes + kChunk - 1) / kChunk;
            const int64_t ksplit = MODE == kModeLossGrad ? min((int64_t)kFusedSplit, nch) : nch;
            int b = 0, t = 0, y = 0;
            if (n_rows > 0) {
                locate_row(cum, p.B, blockIdx.x, b, t);
                y = __ldg(p.tokens + (p.seq_offset + b) * (int64_t)p.T + t);
            }
            // unaligned rows: TMA streams the 16-byte aligned interior [h, h + ib) of the row;
            // this lane loads the < 16-byte head and tail (<= 7 + 7 bf16 / 3 + 3 fp32 elements)
            // before it waits for the row's first stage and publishes them with the row info
            int h = 0;
            int64_t ib = row_bytes;
            float hx[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) hx[k] = 0.f;
            auto issue = [&](const char *src, int64_t rbytes, int64_t c0, int64_t c1, uint64_t pol,
                             int64_t publish_rl) {
                for (int64_t c = c0; c < c1; ++c) {
                    const int64_t off = c * kChunk;
                    const uint32_t bytes = (uint32_t)min((int64_t)kChunk, rbytes - off);
                    mbar_wait(&S.empty[stage], phase ^ 1u);
                    if (c == 0 && publish_rl >= 0) {  // released by the arrive below
                        S.row_y[publish_rl % kRowInfo] = y;
                        S.row_h[publish_rl % kRowInfo] = h;
                        if (UNAL && MODE == kModeLossGrad) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) S.row_x[publish_rl % kRowInfo][k] = hx[k];
                        }
                    }
                    mbar_arrive_expect_tx(&S.full[stage], bytes);
                    tma_load_1d(S.stage[stage], src + off, bytes, &S.full[stage], pol);
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
            };
            const char *prev_src = nullptr;
            int64_t prev_ib = row_bytes;
            // kModeLossGrad schedule per CTA: F(i)[0, k), B(i-1), F(i)[k, nch), ... , B(n-1)
            for (int64_t rl = 0; rl <= n_rows; ++rl) {
                const char *src = nullptr;
                int bn = 0, tn = 0, yn = 0;
                if (rl < n_rows) {
                    const int64_t jn = blockIdx.x + (rl + 1) * (int64_t)gridDim.x;  // prefetch next row's token
                    if (jn < N) {
                        locate_row(cum, p.B, jn, bn, tn);
                        yn = __ldg(p.tokens + (p.seq_offset + bn) * (int64_t)p.T + tn);
                    }
                    src = p.base + logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.stride_b, p.stride_t) * p.elt;
                    if (UNAL) {
                        h = (int)((16u - (uint32_t)(reinterpret_cast<uintptr_t>(src) & 15u)) & 15u);
                        ib = (row_bytes - h) & ~(int64_t)15;
                        const int head_e = h / (int)sizeof(Tin);
                        const int tail_e = (int)((row_bytes - h - ib) / (int64_t)sizeof(Tin));
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            const int idx = k < head_e ? k : (k - head_e < tail_e ? (int)p.V - tail_e + (k - head_e) : -1);
                            if (MODE == kModeLossGrad && idx >= 0)  // the fused backward's head / tail
                                hx[k] = sizeof(Tin) == 2
                                    ? __uint_as_float(((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(src) + idx)) << 16)
                                    : __ldg(reinterpret_cast<const float *>(src) + idx);
                        }
                        src += h;
                    }
                    issue(src, ib, 0, min(ksplit, (ib + kChunk - 1) / kChunk), pol_fwd, rl);
                }
                if (MODE == kModeLossGrad && rl > 0) issue(prev_src, prev_ib, 0, (prev_ib + kChunk - 1) / kChunk, pol_bwd, -1);
                if (rl < n_rows) {
                    const int64_t nch_r = (ib + kChunk - 1) / kChunk;
                    issue(src, ib, min(ksplit, nch_r), nch_r, pol_fwd, -1);
                    b = bn; t = tn; y = yn;
                }
                prev_src = src;
                prev_ib = ib;
            }
        }
        return;
    }

    if (kTmaStore && warp == kStoreWarp) {
        // ===================== store warp (kTmaStore): one lane bulk-stores each full
        // backward chunk the consumers wrote back into its stage, then frees the stage.
        // It replays the producer's chunk schedule (all rows have nch chunks: aligned rows)
        // and touches only the staged chunks.
        if (MODE == kModeLossGrad && !UNAL && lane == 0) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            const uint64_t pol = l2_evict_first_policy();
            const int64_t n_rows = N > (int64_t)blockIdx.x ? (N - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
            const int nch = (int)((row_bytes + kChunk - 1) / kChunk);
            const int ksplit = min(kFusedSplit, nch);
            int stage = 0;
            uint32_t wph = 0;  // bit s: parity of written[s]
            for (int64_t rl = 0; rl <= n_rows; ++rl) {
                if (rl < n_rows) stage = (stage + ksplit) % kStages;
                if (rl > 0) {
                    // two bulk stores in flight: stage j is freed once store j+1 has been issued and
                    // store j has read its shared memory; the row's last staged stage is freed
                    // before the store warp waits on the next row (the ring needs it for the forward)
                    int pend = -1;
                    for (int c = 0; c < nch; ++c) {
                        const int bytes = min(kChunk, (int)row_bytes - c * kChunk);
                        if (bytes == kChunk && (c % kTmaStoreEvery) == 0) {
                            mbar_wait_hint<ORL_K1_STORE_WAIT_NS>(&S.written[stage], (wph >> stage) & 1u);
                            wph ^= 1u << stage;
                            tma_store_1d(reinterpret_cast<void *>(S.st_dst[stage]), S.stage[stage], kChunk, pol);
                            if (pend >= 0) {
                                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                                mbar_arrive_cnt(&S.empty[pend], kEmptyArrivals);
                            }
                            pend = stage;
                        }
                        stage = (stage + 1) % kStages;
                    }
                    if (pend >= 0) {
                        tma_store_wait_read0();
                        mbar_arrive_cnt(&S.empty[pend], kEmptyArrivals);
                    }
                }
                if (rl < n_rows) stage = (stage + nch - ksplit) % kStages;
            }
            tma_store_wait_all();
        }
        return;
    }
    if (warp >= kEpilogueWarp) {
        // ===================== epilogue: merge the partials, fp64 per-row math ===
        const int ew = warp - kEpilogueWarp;  // rows rl with rl % kEpiWarps == ew
        asm volatile("griddepcontrol.wait;" ::: "memory");
        zero_masked(p, cum, lane + 32 * ew, 32 * kEpiWarps, MODE);
        double wh[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        if (MODE != kModeLogprob) {
            wh[0] = p.whiten[0]; wh[1] = p.whiten[1]; wh[2] = p.whiten[2]; wh[3] = p.whiten[3];
            wh[4] = p.whiten[4];
        }
        const int nside = MODE != kModeLogprob ? kSide : 2;
        for (int64_t j = blockIdx.x + (int64_t)ew * gridDim.x, rl = ew; j < N;
             j += (int64_t)kEpiWarps * gridDim.x, rl += kEpiWarps) {
            int b, t;
            locate_row(cum, p.B, j, b, t);
            const int64_t gi = (p.seq_offset + b) * (int64_t)p.T + t;
            const int y = __ldg(p.tokens + gi);
            float side = 0.f;
            if (lane < nside) side = load_side(p, MODE, lane, gi, b);
            // unaligned rows: the < 16-byte head and tail of the row (<= 7 + 7 bf16 elements) are
            // not in the TMA interior the consumers streamed; lane k loads edge element k here,
            // ahead of the row wait, and the warp folds them into the merged state below
            float ex = 0.f;
            int eidx = -1;
            if (UNAL) {
                const char *rsrc =
                    p.base + logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.stride_b, p.stride_t) * p.elt;
                const int hh = (int)((16u - (uint32_t)(reinterpret_cast<uintptr_t>(rsrc) & 15u)) & 15u);
                const int64_t ibb = (row_bytes - hh) & ~(int64_t)15;
                const int head_e = hh / (int)sizeof(Tin);
                const int tail_e = (int)((row_bytes - hh - ibb) / (int64_t)sizeof(Tin));
                if (lane < head_e) eidx = lane;
                else if (lane < head_e + tail_e) eidx = (int)p.V - tail_e + (lane - head_e);
                if (eidx >= 0)
                    ex = sizeof(Tin) == 2
                             ? __uint_as_float(((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(rsrc) + eidx)) << 16)
                             : __ldg(reinterpret_cast<const float *>(rsrc) + eidx);
            }
            // everything that does not depend on the row's logits is ready before the wait
            float sv[kSide];
#pragma unroll
            for (int k = 0; k < kSide; ++k) sv[k] = __shfl_sync(0xffffffffu, side, k);
            const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
            RowPre pre{0.0, 0.0, 0.f};
            if (MODE != kModeLogprob && lane == 0) pre = row_pre(p, L, sv, wh);
            const int slot = (int)(rl % kSlots);
            mbar_wait_hint<ORL_K1_EPI_WAIT_NS>(&S.row_full[slot], (uint32_t)(rl / kSlots) & 1u);
#ifdef ORL_K1_PROF
            const long long t_full = clock64();
#endif
            const RowSlot &R = S.slot[slot];
            Online st{R.m[lane], R.s[lane], R.u[lane]};
#pragma unroll
            for (int w = 1; w < (kPremerge ? kConsumerWarps / 4 : kConsumerWarps); ++w)
                st = online_merge(st, Online{R.m[lane + 32 * w], R.s[lane + 32 * w], R.u[lane + 32 * w]});
            st = warp_merge(st);
            float target = R.target;
            if (UNAL) {
                Online e{kMInit, 0.f, 0.f};
                if (eidx >= 0) e = Online{fmax_nan(fmax_nan(ex, kNegClampF32) * p.c2, kMInit), 1.f, 0.f};
                st = online_merge(st, warp_merge(e));
                const unsigned hit = __ballot_sync(0xffffffffu, eidx >= 0 && eidx == y);
                const float xt = __shfl_sync(0xffffffffu, ex, hit ? __ffs(hit) - 1 : 0);
                if (hit) target = xt;
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&S.row_empty[slot]);
                EpiOut eo{0.f, 0.f, 0.f};
                // the backward's row constants are published as soon as (lse, H, w) exist
#ifdef ORL_K1_PROF
                if (MODE == kModeLossGrad) K1PROF(1, clock64() - t_full);
#endif
                auto publish = [&](const EpiOut &e) {
                    if (MODE == kModeLossGrad) {
#ifdef ORL_K1_PROF
                        K1PROF(0, clock64() - t_full);
                        K1PROF(2, 1);
#endif
                        // same fp32 constants as K5 (orl_logits_grad) computes from the saved arrays
                        const float a = pre.a;
                        GradRow &g = S.grad[rl % kGradRows];
                        g.out_off = logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.out_stride_b, p.out_stride_t);
                        g.y = y;
                        g.l2 = e.lse * kLog2e;
                        g.A1 = p.inv_temp * a * (float)kLn2;
                        g.A0 = p.inv_temp * (a * e.H - e.w);
                        g.wt = p.inv_temp * e.w;
                        mbar_arrive(&S.grad_full[rl % kGradRows]);
                    }
                };
#if ORL_K1_ABL & 32  // timing ablation: no fp64 row epilogue (the backward's constants still published)
                if (MODE == kModeLossGrad) publish(EpiOut{st.m, st.s, st.u});
                else if (st.m == 1234.5f) p.logp[0] = st.s;
#else
                row_epilogue<MODE>(p, b, t, L, y, st, target, sv, wh, S.wacc[ew], &eo, publish, &pre);
#endif
            }
            __syncwarp();
        }
        if (MODE != kModeLogprob) {
            if (kEpiWarps > 1) named_bar_sync(1, 32 * kEpiWarps);
            if (ew == 0) {
                double tot[kNumPartials];
#pragma unroll
                for (int c = 0; c < kNumPartials; ++c) {
                    double v = 0.0;
                    for (int e = 0; e < kEpiWarps; ++e) v += S.wacc[e][c];   // fixed order
                    tot[c] = v;
                }
                finish_partials_warp(p, tot, lane);
            }
        }
        return;
    }

    // ========================= consumers (warps 0..7) ============================
    const int ct = tid;  // 0..kConsumers-1
#ifdef ORL_K1_ALWAYS_ENT
    const bool ent = true;
#else
    const bool ent = MODE != kModeLogprob || p.entropy != nullptr;
#endif
    const uint64_t c2p = pack2(p.c2, p.c2);
    int stage = 0;
    uint32_t phase = 0;
    const int64_t n_rows = N > (int64_t)blockIdx.x ? (N - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    // chunk bookkeeping in 32 bits (a row is < 2^31 bytes: V <= 2^28, checked on the host)
    const int nch = (int)((row_bytes + kChunk - 1) / kChunk);
    const int ksplit = MODE == kModeLossGrad ? min(kFusedSplit, nch) : nch;
    // forward state of the row in progress (survives an interleaved backward row)
    ThreadAcc acc{kMInit, 0ull, 0ull, 0ull, 0ull};
    float tgt = 0.f;
    bool have_tgt = false;
    int tchunk = -1;
    int tin = 0;
    bool towner = false;
    // unaligned rows (p.unaligned, not in the fused mode): the chunks cover the aligned
    // interior [h, h + ib) of the row; its < 16-byte head and tail are folded in by
    // scalar loads after the first chunk
    constexpr bool unal = UNAL;
    int ib = (int)row_bytes, row_nch = nch;
    int row_h = 0, row_yv = -1;
    auto fwd_chunks = [&](int64_t rl, int c0, int c1) {
        for (int ci = c0; ci < (unal ? (ci == 0 ? 1 : min(c1, row_nch)) : c1); ++ci) {
            mbar_wait_hint<ORL_K1_CONS_WAIT_NS>(&S.full[stage], phase);
            if (ci == 0) {  // row start: which chunk / thread holds the target logit
                acc = ThreadAcc{kMInit, 0ull, 0ull, 0ull, 0ull};
                have_tgt = false;
                const int y = S.row_y[rl % kRowInfo];
                row_yv = y;
                if (unal) {
                    row_h = S.row_h[rl % kRowInfo];
                    ib = ((int)row_bytes - row_h) & ~15;
                    row_nch = (ib + kChunk - 1) / kChunk;
                }
                const bool y_ok = (y >= 0) && ((int64_t)y < p.V);
                const int ybyte = y * (int)sizeof(Tin) - row_h;  // offset in the interior
                tchunk = (y_ok && ybyte >= 0 && ybyte < ib) ? ybyte / kChunk : -1;
                tin = ybyte % kChunk;
                towner = ((tin >> 4) % kConsumers) == ct;
            }
            const int off = ci * kChunk;
            const int bytes = min(kChunk, ib - off);
            const uint8_t *sb = S.stage[stage];
            if (ci == tchunk && towner) {  // raw target value, before any clamping
                tgt = sizeof(Tin) == 2
                          ? __uint_as_float(((uint32_t)*reinterpret_cast<const uint16_t *>(sb + tin)) << 16)
                          : *reinterpret_cast<const float *>(sb + tin);
                have_tgt = true;
            }
            // copy this thread's bytes to registers and hand the stage back to the
            // producer before computing, so the ring keeps ~all stages in flight
            uint32_t w[kW];
            if (bytes == kChunk) load_words<Tin, true>(w, sb, ct, kChunk >> 4);
            else load_words<Tin, false>(w, sb, ct, bytes >> 4);
            release_stage(&S.empty[stage], lane);
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
#if ORL_K1_ABL & 1  // timing ablation: no forward math (loads kept)
            acc.sA ^= (uint64_t)w[0] ^ ((uint64_t)w[kW - 1] << 32);
#else
            if (ent) process_words<Tin, true, POLY>(acc, w, ci == 0, p.c2, c2p);
            else process_words<Tin, false, POLY>(acc, w, ci == 0, p.c2, c2p);
#endif
        }
    };
    auto fwd_publish = [&](int64_t rl) {  // row end: this thread's state into the row slot
#ifdef ORL_K1_PROF
        const long long t_p0 = clock64();
#endif
        float s0, s1, s2, s3;
        unpack2(fadd2(acc.sA, acc.sB), s0, s1);
        unpack2(fadd2(acc.uA, acc.uB), s2, s3);
        Online st{acc.m, s0 + s1, s2 + s3};
        if (kPremerge) {
            // actor passes: a 2-round xor pre-merge (lanes 4k..4k+3, lane 4k keeps it) shortens the
            // epilogue's merge from 16 to 4 states per lane -- the fused backward waits for it
#pragma unroll
            for (int off = 1; off <= 2; off <<= 1) {
                Online o;
                o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
                o.s = __shfl_xor_sync(0xffffffffu, st.s, off);
                o.u = __shfl_xor_sync(0xffffffffu, st.u, off);
                st = online_merge(st, o);
            }
        }
        const int slot = (int)(rl % kSlots);
        mbar_wait(&S.row_empty[slot], ((uint32_t)(rl / kSlots) & 1u) ^ 1u);
        RowSlot &R = S.slot[slot];
        if (!kPremerge || (lane & 3) == 0) {
            const int k = kPremerge ? warp * 8 + (lane >> 2) : ct;
            R.m[k] = st.m;
            R.s[k] = st.s;
            R.u[k] = st.u;
        }
        if (have_tgt) R.target = tgt;
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.row_full[slot]);
#ifdef ORL_K1_PROF
        if (MODE == kModeLossGrad && ct == 0) { K1PROF(5, clock64() - t_p0); K1PROF(6, 1); }
#endif
    };
    auto bwd_row = [&](int64_t rb) {
        // backward pass over row rb (NEXT-1, re-read from L2):
        // dL/dx_v = p_v (A1 t_v + A0) + [v = y] wt,  t_v = x_v c - lse log2 e
#if ORL_K1_ABL & 8  // timing ablation: wait for the row constants of the first rows only (then stale ones)
        if (rb < kGradRows)
#endif
#ifdef ORL_K1_PROF
        const long long t_w0 = clock64();
#endif
        mbar_wait(&S.grad_full[rb % kGradRows], (uint32_t)(rb / kGradRows) & 1u);
#ifdef ORL_K1_PROF
        if (ct == 0) { K1PROF(3, clock64() - t_w0); K1PROF(4, 1); }
#endif
        const GradRow g = S.grad[rb % kGradRows];
        Tin *orow = reinterpret_cast<Tin *>(p.dlogits) + g.out_off;
        const uint64_t nl2 = pack2(-g.l2, -g.l2), A1p = pack2(g.A1, g.A1), A0p = pack2(g.A0, g.A0);
        // unaligned rows: the chunks are the row's aligned interior [bh, bh + bib) (dlogits rows are
        // misaligned like the logits rows, checked on the host); head / tail written singly here
        const int bh = UNAL ? S.row_h[rb % kRowInfo] : 0;
        const int rbytes = (int)row_bytes;
        const int bib = UNAL ? ((rbytes - bh) & ~15) : rbytes;
        if (UNAL && warp == 0) {  // head / tail (<= 14 elements): warp 0
            const int head_e = bh / (int)sizeof(Tin);
            const int tail_e = (rbytes - bh - bib) / (int)sizeof(Tin);
            int idx = -1;
            if (ct < head_e) idx = ct;
            else if (ct < head_e + tail_e) idx = (int)p.V - tail_e + (ct - head_e);
            if (idx >= 0) {
                const float t2 = fmaf(S.row_x[rb % kRowInfo][ct], p.c2, -g.l2);
                float gv = __fmul_rn(ex2(t2), GENT ? fmaf(g.A1, t2, g.A0) : g.A0);  // no contraction: same bits on every path
                if (idx == g.y) gv = __fadd_rn(gv, g.wt);
                if (sizeof(Tin) == 2) {
                    const uint32_t hb = f32x2_to_bf16x2_rn(gv, 0.f) & 0xffffu;
                    asm volatile("st.global.u16 [%0], %1;" ::"l"(orow + idx), "h"((unsigned short)hb) : "memory");
                } else {
                    reinterpret_cast<float *>(orow)[idx] = gv;
                }
            }
        }
        const bool y_ok = g.y >= 0 && (int64_t)g.y < p.V;
        const int ybyte = g.y * (int)sizeof(Tin) - bh;  // offset in the interior
#ifndef ORL_K1_FUSED_STORE
#define ORL_K1_FUSED_STORE 0  // dlogits stores: 0 evict_first hint, 1 .cs, 2 plain, 3 evict_normal hint, 4 evict_unchanged hint
#endif
        const uint64_t st_pol = ORL_K1_FUSED_STORE == 3 ? l2_evict_normal_policy()
                                : ORL_K1_FUSED_STORE == 4 ? l2_evict_unchanged_policy() : l2_evict_first_policy();
        for (int off = 0; off < bib; off += kChunk) {
            const int bytes = min(kChunk, bib - off);
            const int nvec = bytes >> 4;
            mbar_wait(&S.full[stage], phase);
            const int cst = stage;  // this chunk's stage
            const uint8_t *sb = S.stage[stage];
            const bool own_y = y_ok && ybyte >= off && ybyte < off + bytes && (((ybyte - off) >> 4) % kConsumers) == ct;
            // kTmaStore: a full chunk's results go back into its stage; the store warp bulk-stores
            // the stage and frees it (same rule as the store warp's schedule: aligned rows, full chunk)
            const bool staged = kTmaStore && !UNAL && bytes == kChunk && ((off / kChunk) % kTmaStoreEvery) == 0;
            float xy = 0.f;
            if (own_y) {
                const uint8_t *q = sb + (ybyte - off);
                xy = sizeof(Tin) == 2 ? __uint_as_float(((uint32_t)*reinterpret_cast<const uint16_t *>(q)) << 16)
                                      : *reinterpret_cast<const float *>(q);
            }
            uint4 v[kVecPerThread];
#pragma unroll
            for (int k = 0; k < kVecPerThread; ++k) {
                const int vi = ct + k * kConsumers;
                if (vi < nvec) v[k] = lds128(sb + vi * 16);
            }
            if (!staged) release_stage(&S.empty[stage], lane);
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
            char *obase = reinterpret_cast<char *>(orow) + bh + off;
            // dL/dx of one 16-byte vector: the same per-element operations on every path (and as K5)
            auto grad_vec = [&](const uint4 &vv, uint32_t (&o)[4]) {
                const uint32_t w4[4] = {vv.x, vv.y, vv.z, vv.w};
#if ORL_K1_ABL & 2  // timing ablation: no backward math (stores kept)
                if (true) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) o[q] = w4[q] ^ 0x55u;
                } else
#endif
                if (sizeof(Tin) == 2) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t t2 = ffma2(bf16x2_to_f32x2(w4[q]), c2p, nl2);
                        float t0, t1;
                        unpack2(t2, t0, t1);
                        const uint64_t gr = fmul2(pack2(ex2(t0), ex2(t1)), GENT ? ffma2(A1p, t2, A0p) : A0p);
                        float g0, g1;
                        unpack2(gr, g0, g1);
                        o[q] = f32x2_to_bf16x2_rn(g0, g1);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        uint64_t x;
                        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(w4[2 * q]), "r"(w4[2 * q + 1]));
                        const uint64_t t2 = ffma2(x, c2p, nl2);
                        float t0, t1;
                        unpack2(t2, t0, t1);
                        const uint64_t gr = fmul2(pack2(ex2(t0), ex2(t1)), GENT ? ffma2(A1p, t2, A0p) : A0p);
                        float g0, g1;
                        unpack2(gr, g0, g1);
                        o[2 * q] = __float_as_uint(g0);
                        o[2 * q + 1] = __float_as_uint(g1);
                    }
                }
            };
            auto store_vec = [&](char *dst, const uint32_t (&o)[4]) {
#if ORL_K1_ABL & 4  // timing ablation: no backward stores (math kept)
                if (o[0] == 0x7fc17fc1u && o[3] == 0x7fc17fc1u)
                stg128_hint(dst, make_uint4(o[0], o[1], o[2], o[3]), st_pol);
#elif ORL_K1_FUSED_STORE == 1
                stg128_cs(dst, make_uint4(o[0], o[1], o[2], o[3]));
#elif ORL_K1_FUSED_STORE == 2
                asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "r"(o[0]), "r"(o[1]),
                             "r"(o[2]), "r"(o[3]) : "memory");
#else
                stg128_hint(dst, make_uint4(o[0], o[1], o[2], o[3]), st_pol);
#endif
            };
            if (staged) {
                uint32_t o[kVecPerThread][4];
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) grad_vec(v[k], o[k]);
                uint8_t *wb = const_cast<uint8_t *>(sb);
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    uint4 *q = reinterpret_cast<uint4 *>(wb + (ct + k * kConsumers) * 16);
                    *q = make_uint4(o[k][0], o[k][1], o[k][2], o[k][3]);
                }
                if (own_y) {  // the target element with the delta term, after its vector (program order)
                    const float t2 = fmaf(xy, p.c2, -g.l2);
                    const float gy = __fadd_rn(__fmul_rn(ex2(t2), GENT ? fmaf(g.A1, t2, g.A0) : g.A0), g.wt);
                    if (sizeof(Tin) == 2)
                        *reinterpret_cast<uint16_t *>(wb + (ybyte - off)) = (uint16_t)(f32x2_to_bf16x2_rn(gy, 0.f) & 0xffffu);
                    else
                        *reinterpret_cast<float *>(wb + (ybyte - off)) = gy;
                }
                fence_proxy_async();  // generic-proxy smem writes -> the bulk copy engine
                if (ct == 0) S.st_dst[cst] = reinterpret_cast<uint64_t>(obase);
                mbar_arrive(&S.written[cst]);
                continue;
            }
            if (nvec == kVecPerThread * kConsumers) {
                // full chunk: every thread owns kVecPerThread vectors -- one straight-line block
                // (no per-vector branches), so the vectors' MUFU / FMA chains interleave
                char *tb = obase + ct * 16;
                uint32_t o[kVecPerThread][4];
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) grad_vec(v[k], o[k]);
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) store_vec(tb + k * (kConsumers * 16), o[k]);
            } else {
#pragma unroll
                for (int k = 0; k < kVecPerThread; ++k) {
                    const int vi = ct + k * kConsumers;
                    if (vi >= nvec) continue;
                    uint32_t o[4];
                    grad_vec(v[k], o);
                    store_vec(obase + vi * 16, o);
                }
            }
            if (own_y) {  // program-ordered rewrite of the target element with the delta term
                const float t2 = fmaf(xy, p.c2, -g.l2);
                const float gy = __fadd_rn(__fmul_rn(ex2(t2), GENT ? fmaf(g.A1, t2, g.A0) : g.A0), g.wt);  // p (A1 t + A0) + wt, not contracted
                if (sizeof(Tin) == 2) {
                    const uint32_t hb = f32x2_to_bf16x2_rn(gy, 0.f) & 0xffffu;
                    asm volatile("st.global.u16 [%0], %1;" ::"l"(orow + g.y), "h"((unsigned short)hb) : "memory");
                } else {
                    reinterpret_cast<float *>(orow)[g.y] = gy;
                }
            }
        }
    };
    // schedule (mirrors the producer): F(i)[0, k), B(i-1), F(i)[k, nch), publish F(i)
    for (int64_t rl = 0; rl <= n_rows; ++rl) {
        if (rl < n_rows) fwd_chunks(rl, 0, ksplit);
        if (MODE == kModeLossGrad && rl > 0) bwd_row(rl - 1);
        if (rl < n_rows) {
            fwd_chunks(rl, ksplit, nch);
            fwd_publish(rl);
        }
    }
    if (MODE == kModeLossGrad && p.zero_masked_grad && !p.cu_seqlens) {
        // zero the dlogits rows of the masked positions (padded layout)
        const int64_t total = (int64_t)p.B * p.T;
        for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
            const int b = (int)(q / p.T), t = (int)(q % p.T);
            const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
            if (t < L) continue;
            char *orow = reinterpret_cast<char *>(p.dlogits) +
                         ((int64_t)b * p.out_stride_b + (int64_t)t * p.out_stride_t) * (int64_t)sizeof(Tin);
            const int zh = UNAL ? (int)((16u - (uint32_t)(reinterpret_cast<uintptr_t>(orow) & 15u)) & 15u) : 0;
            const int64_t zib = UNAL ? ((row_bytes - zh) & ~(int64_t)15) : row_bytes;
            for (int64_t o = (int64_t)ct * 16; o < zib; o += (int64_t)kConsumers * 16)
                stg128_cs(orow + zh + o, make_uint4(0u, 0u, 0u, 0u));
            if (UNAL) {  // head and tail elements
                const int64_t nh = zh / (int64_t)sizeof(Tin), t0 = (zh + zib) / (int64_t)sizeof(Tin);
                if (ct < nh) reinterpret_cast<Tin *>(orow)[ct] = Tin(0);
                else if (t0 + (ct - nh) < p.V) reinterpret_cast<Tin *>(orow)[t0 + (ct - nh)] = Tin(0);
            }
        }
    }
}

// ---------------------------------------------------------------- generic kernel
// Unaligned rows (e.g. V = 50257 bf16): 256 threads per row, element-strided
// global loads, the same online state and epilogue.  Correctness path.
template <typename Tin, int MODE>
__global__ void __launch_bounds__(256) k1_generic_kernel(const K1Params p) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ double wacc[1][kNumPartials];
    __shared__ float sm_m[8], sm_s[8], sm_u[8];
    __shared__ float sm_tgt;
    int32_t *cum_s = reinterpret_cast<int32_t *>(smem_raw);
    int32_t *warp_tot = cum_s + (p.cum_global ? 0 : p.B);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < kNumPartials) wacc[0][tid] = 0.0;
    const int32_t *cum = p.cum_global ? p.cum_global : cum_s;
    if (p.cum_global) {  // written by the prefix kernel just before us (PDL: wait for it)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        __syncthreads();
    }
    else build_prefix(p, cum_s, warp_tot);
    const int64_t N = cum[p.B - 1];
    zero_masked(p, cum, tid, 256, MODE);
    double wh[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (MODE != kModeLogprob) {
        wh[0] = p.whiten[0]; wh[1] = p.whiten[1]; wh[2] = p.whiten[2]; wh[3] = p.whiten[3];
        wh[4] = p.whiten[4];
    }
    for (int64_t j = blockIdx.x; j < N; j += gridDim.x) {
        int b, t;
        locate_row(cum, p.B, j, b, t);
        const int64_t gi = (p.seq_offset + b) * (int64_t)p.T + t;
        const int y = __ldg(p.tokens + gi);
        const Tin *row = reinterpret_cast<const Tin *>(p.base) +
                         logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.stride_b, p.stride_t);
        Online st{kMInit, 0.f, 0.f};
        for (int64_t v0 = 0; v0 < p.V; v0 += 256 * 8) {
            float x[8];
            float cmx = kNegClampF32;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t v = v0 + tid + k * 256;
                float xv = kNegClampF32;
                if (v < p.V) {
                    if (sizeof(Tin) == 2)
                        xv = __uint_as_float(((uint32_t)reinterpret_cast<const uint16_t *>(row)[v]) << 16);
                    else
                        xv = reinterpret_cast<const float *>(row)[v];
                    if (v == y) sm_tgt = xv;
                }
                x[k] = fmax_nan(xv, kNegClampF32);
                cmx = fmax_nan(cmx, x[k]);
            }
            const float mn = fmax_nan(st.m, cmx * p.c2);
            const float d = st.m - mn, r = ex2(d);
            st.u = r * fmaf(d, st.s, st.u);
            st.s = r * st.s;
            st.m = mn;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float tt = fmaf(x[k], p.c2, -st.m);
                const float e = ex2(tt);
                st.s += e;
                st.u = fmaf(e, tt, st.u);
            }
        }
        st = warp_merge(st);
        if (lane == 0) { sm_m[warp] = st.m; sm_s[warp] = st.s; sm_u[warp] = st.u; }
        __syncthreads();
        float side[kSide] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (tid == 0) {
            Online tot{sm_m[0], sm_s[0], sm_u[0]};
            for (int w = 1; w < 8; ++w) tot = online_merge(tot, Online{sm_m[w], sm_s[w], sm_u[w]});
            const int nside = MODE != kModeLogprob ? kSide : 2;
            for (int k = 0; k < nside; ++k) side[k] = load_side(p, MODE, k, gi, b);
            const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
            row_epilogue<MODE>(p, b, t, L, y, tot, sm_tgt, side, wh, wacc[0]);
        }
        __syncthreads();
    }
    if (MODE != kModeLogprob) finish_partials(p, wacc, 1, tid, 256, -1);
}

// ---------------------------------------------------------------- NEXT-4 merge
// One thread per valid row: merge the row's K6 split partials (m, s, u) in
// split order (online_merge), take z_y from the split holding column y, and
// run the same row epilogue as the streaming kernels.  Loss partials: per
// thread, xor-tree per warp, warp order per CTA, CTA order by the last CTA.
template <int MODE>
__global__ void __launch_bounds__(256) k6_merge_kernel(const K1Params p) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    __shared__ double wacc[8][kNumPartials];
    int32_t *cum_s = reinterpret_cast<int32_t *>(smem_raw);
    int32_t *warp_tot = cum_s + (p.cum_global ? 0 : p.B);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t *cum = p.cum_global ? p.cum_global : cum_s;
    // launched programmatically after K6: its partials are visible after this wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.cum_global) __syncthreads();
    else build_prefix(p, cum_s, warp_tot);
    const int64_t N = cum[p.B - 1];
    zero_masked(p, cum, tid, 256, MODE);
    double wh[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (MODE != kModeLogprob) {
        wh[0] = p.whiten[0]; wh[1] = p.whiten[1]; wh[2] = p.whiten[2]; wh[3] = p.whiten[3];
        wh[4] = p.whiten[4];
    }
    double acc[kNumPartials];
#pragma unroll
    for (int c = 0; c < kNumPartials; ++c) acc[c] = 0.0;
    for (int64_t j = (int64_t)blockIdx.x * 256 + tid; j < N; j += (int64_t)gridDim.x * 256) {
        int b, t;
        locate_row(cum, p.B, j, b, t);
        const int64_t gi = (p.seq_offset + b) * (int64_t)p.T + t;
        const int y = __ldg(p.tokens + gi);
        const int64_t r = p.cu_seqlens
                              ? (int64_t)(__ldg(p.cu_seqlens + p.seq_offset + b) - __ldg(p.cu_seqlens + p.seq_offset)) + t
                              : (int64_t)b * p.T + t;
        if (r >= p.lm_R) {  // the hidden matrix does not hold this row: layout/lengths mismatch
            atomicAdd(&p.err[4], 1ull);
            const float nan = __int_as_float(0x7fc00000);
            p.logp[gi] = nan;
            if (p.entropy) p.entropy[gi] = nan;
            if (p.lse) p.lse[gi] = nan;
            continue;
        }
        Online tot{kMInit, 0.f, 0.f};
        for (int sp = 0; sp < p.lm_nsplit; ++sp) {
            const float4 q = p.lm_parts[(int64_t)sp * p.lm_stride + r];
            tot = online_merge(tot, Online{q.x, q.y, q.z});
        }
        float target = 0.f;
        if (y >= 0 && y < p.V) target = p.lm_parts[(int64_t)(y / p.lm_split_cols) * p.lm_stride + r].w;
        float side[kSide] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int nside = MODE != kModeLogprob ? kSide : 2;
        for (int k = 0; k < nside; ++k) side[k] = load_side(p, MODE, k, gi, b);
        const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
        row_epilogue<MODE>(p, b, t, L, y, tot, target, side, wh, acc);
    }
    if (MODE != kModeLogprob) {
#pragma unroll
        for (int c = 0; c < kNumPartials; ++c) {
            double v = acc[c];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0) wacc[warp][c] = v;
        }
        finish_partials(p, wacc, 8, tid, 256, -1);
    }
}

cudaError_t launch_k6_merge(const K1Params &p, int mode, int num_sms, cudaStream_t s) {
    const size_t smem = sizeof(int32_t) * (size_t)((p.cum_global ? 0 : p.B) + 32);
    auto kern = mode == kModeLoss ? k6_merge_kernel<kModeLoss> : k6_merge_kernel<kModeLogprob>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = ((int64_t)p.B * p.T + 255) / 256;
    if (grid > (int64_t)num_sms * 4) grid = (int64_t)num_sms * 4;
    if (grid > p.ws_stride) grid = p.ws_stride;
    if (grid < 1) grid = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

// ---------------------------------------------------------------- launcher
template <typename Tin, int MODE, int POLY>
static cudaError_t launch_tma(const K1Params &p, int num_sms, cudaStream_t s) {
    const int64_t N_upper = (int64_t)p.B * p.T;  // rows are counted on device; size by the bound
    const size_t smem = k1_tma_smem_bytes(p.B);
    // unaligned rows: a separate instantiation, so the aligned path carries none of it; the fused
    // pass without an entropy term (c2 = 0) likewise
    const bool gent = MODE != kModeLossGrad || p.c2_ent != 0.0;
    auto kern = (POLY == 0 && p.unaligned) ? (gent ? k1_tma_kernel<Tin, MODE, 0, true, true>
                                                   : k1_tma_kernel<Tin, MODE, 0, true, MODE != kModeLossGrad>)
                                           : (gent ? k1_tma_kernel<Tin, MODE, POLY, false, true>
                                                   : k1_tma_kernel<Tin, MODE, POLY, false, MODE != kModeLossGrad>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)num_sms * per_sm;
    if (grid > N_upper) grid = N_upper;
    if (grid > p.ws_stride) grid = p.ws_stride;
    if (grid < 1) grid = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename Tin, int MODE>
static cudaError_t launch_typed(const K1Params &p, bool tma, int num_sms, cudaStream_t s) {
    const int64_t N_upper = (int64_t)p.B * p.T;
    if (tma) {
        if (p.poly == 8 && !p.unaligned) return launch_tma<Tin, MODE, 8>(p, num_sms, s);
        if (p.poly == 16 && !p.unaligned) return launch_tma<Tin, MODE, 16>(p, num_sms, s);
        return launch_tma<Tin, MODE, 0>(p, num_sms, s);
    }
    const size_t smem = sizeof(int32_t) * (size_t)((p.cum_global ? 0 : p.B) + 32);
    cudaError_t e = cudaFuncSetAttribute(k1_generic_kernel<Tin, MODE>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)num_sms * 4;
    if (grid > N_upper) grid = N_upper;
    if (grid > p.ws_stride) grid = p.ws_stride;
    if (grid < 1) grid = 1;
    k1_generic_kernel<Tin, MODE><<<(unsigned)grid, 256, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_k1(const K1Params &p, bool tma, int mode, int num_sms, cudaStream_t s) {
    if (mode == kModeLossGrad) {  // fused actor forward + backward: TMA kernel only
        if (!tma) return cudaErrorInvalidValue;
        return p.elt == 2 ? launch_tma<uint16_t, kModeLossGrad, 0>(p, num_sms, s)
                          : launch_tma<float, kModeLossGrad, 0>(p, num_sms, s);
    }
    if (p.elt == 2)
        return mode == kModeLoss ? launch_typed<uint16_t, kModeLoss>(p, tma, num_sms, s)
                                 : launch_typed<uint16_t, kModeLogprob>(p, tma, num_sms, s);
    return mode == kModeLoss ? launch_typed<float, kModeLoss>(p, tma, num_sms, s)
                             : launch_typed<float, kModeLogprob>(p, tma, num_sms, s);
}

}  // namespace orl

#ifdef ORL_K1_PROF
extern "C" int orl_debug_k1_prof(unsigned long long *out8) {
    if (cudaMemcpyFromSymbol(out8, orl::g_k1prof, sizeof(unsigned long long) * 8) != cudaSuccess) return -1;
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    return cudaMemcpyToSymbol(orl::g_k1prof, z, sizeof(z)) == cudaSuccess ? 0 : -1;
}
#endif

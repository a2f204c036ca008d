// orl_api.cu -- the C ABI of liborl.so (include/orl.h): host-side validation,
// context (NCCL communicator, fp64 accumulators, device error counters,
// pinned stats slot), launch configuration and the two collectives:
//   C1 = all-gather of the rank whitening partials (count, mean, M2) + a
//        fixed-order Chan merge on the device (orl_whiten_stats),
//   C2 = all-gather of the rank loss/stat partials + a rank-ordered sum
//        (orl_finalize).
// An all-gather of a few doubles followed by an ordered merge gives every
// rank bit-identical results (a ring all-reduce would not fix the order);
// messages are <= 128 B per rank, so the cost is NCCL launch latency.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/orl.h"
#include "orl_internal.h"

using namespace orl;

static_assert(sizeof(ncclUniqueId) == ORL_UNIQUE_ID_BYTES, "unique id size");
static_assert(kStatsSlots == ORL_PARTIALS_N && kStatsOut == ORL_STATS_N, "stats vector sizes");

namespace {
constexpr int kMaxWorld = 256;
#ifndef ORL_K1_POLY
#define ORL_K1_POLY 0
#endif
constexpr int kDefaultPoly = ORL_K1_POLY;  // rejected (DESIGN 5.1); the library's numerics do not depend on the environment
thread_local std::string g_thread_err;
}  // namespace

struct orl_ctx {
    int device = 0, world = 1, rank = 0, num_sms = 148;
    ncclComm_t comm = nullptr;
    double *d_acc = nullptr;           // [16] loss accumulators
    unsigned long long *d_err = nullptr;  // [kNumErr]
    double *d_ws = nullptr;            // [kNumPartials][ws_stride]
    int ws_stride = 0;
    unsigned int *d_ticket = nullptr;
    double *d_seq_part = nullptr;      // [cap][3]
    int64_t seq_cap = 0;
    int64_t adv_B = 0;
    double *d_gather_w = nullptr;      // [kMaxWorld][4]
    double *d_whiten = nullptr;        // [4] N, mu, sigma, apply
    double *d_flags = nullptr;         // [4] whiten_warn, mask errors
    double *d_gather_s = nullptr;      // [kMaxWorld][16]
    double *d_stats = nullptr;         // [16]
    double *h_stats = nullptr;         // pinned [16 + 4]
    int32_t *d_cum = nullptr;          // length prefix of large micro-batches
    int64_t cum_cap = 0;
    float4 *d_lm_parts = nullptr;      // NEXT-4 split partials
    int64_t lm_cap = 0;
    unsigned long long *d_x = nullptr;  // C1/C2 peer exchange buffer [kXWords] (IPC-shared)
    PeerArgs peer{};                    // every rank's exchange buffer, mapped here
    bool peer_open = false;
    int coll = 0;                       // 0 NCCL all-gather, 1 peer-memory kernels
    unsigned long long *d_epoch = nullptr;  // [2] C1 / C2 peer epochs (device: graph-replay safe)
    bool have_adv = false, have_whiten = false;
    int pdl_chain = 0;                  // orl_set_pdl_chain
    int imported_w = 0, imported_s = 0;
    uint64_t launches = 0;
    std::string err;
};

// ------------------------------------------------------------------ helpers
static orl_status fail(orl_ctx *ctx, orl_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    g_thread_err = buf;
    return st;
}

#define CUDA_TRY(ctx, expr)                                                                     \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail((ctx), ORL_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),      \
                        __FILE__, __LINE__);                                                    \
    } while (0)

#define NCCL_TRY(ctx, expr)                                                                     \
    do {                                                                                        \
        ncclResult_t r_ = (expr);                                                               \
        if (r_ != ncclSuccess)                                                                  \
            return fail((ctx), ORL_E_NCCL, "%s: %s", #expr, ncclGetErrorString(r_));           \
    } while (0)

static bool aligned4(const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 3u) == 0; }
static cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static orl_status set_device(orl_ctx *ctx) {
    CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    return ORL_OK;
}

static orl_status validate_rows(orl_ctx *ctx, const orl_rows *rows, float inv_temp) {
    if (!rows) return fail(ctx, ORL_E_INVALID_ARG, "rows is NULL");
    if (!rows->tokens || !rows->lengths)
        return fail(ctx, ORL_E_INVALID_ARG, "tokens and lengths are required");
    if (rows->B < 1 || rows->B > ORL_MAX_SEQ_PER_CALL)
        return fail(ctx, ORL_E_SHAPE, "B=%lld outside [1, %d]", (long long)rows->B, ORL_MAX_SEQ_PER_CALL);
    if (rows->T < 1 || rows->seq_offset < 0)
        return fail(ctx, ORL_E_SHAPE, "T=%lld / seq_offset=%lld invalid", (long long)rows->T,
                    (long long)rows->seq_offset);
    if (rows->B * rows->T >= (int64_t)1 << 31 || (rows->seq_offset + rows->B) * rows->T >= (int64_t)1 << 40)
        return fail(ctx, ORL_E_SHAPE, "B*T too large");
    if (!(inv_temp > 0.f) || !(inv_temp <= 1.0e4f))
        return fail(ctx, ORL_E_INVALID_ARG, "inv_temp=%g must be in (0, 1e4]", (double)inv_temp);
    if (!aligned4(rows->tokens) || !aligned4(rows->lengths) || !aligned4(rows->cu_seqlens))
        return fail(ctx, ORL_E_ALIGN, "tokens/lengths/cu_seqlens must be 4-byte aligned");
    return ORL_OK;
}

static orl_status validate_rows_logits(orl_ctx *ctx, const orl_rows *rows, const orl_logits *lg,
                                       float inv_temp) {
    if (!lg) return fail(ctx, ORL_E_INVALID_ARG, "logits is NULL");
    if (!lg->ptr) return fail(ctx, ORL_E_INVALID_ARG, "logits.ptr is required");
    if (lg->dtype != ORL_BF16 && lg->dtype != ORL_F32)
        return fail(ctx, ORL_E_DTYPE, "unknown logits dtype %d", lg->dtype);
    orl_status st = validate_rows(ctx, rows, inv_temp);
    if (st) return st;
    // a row (V elements) must stay below 2^31 bytes: the kernels keep row offsets in 32 bits
    if (lg->V < 1 || lg->V * (lg->dtype == ORL_BF16 ? 2 : 4) >= ((int64_t)1 << 31))
        return fail(ctx, ORL_E_SHAPE, "V=%lld invalid (a row must be < 2 GiB)", (long long)lg->V);
    if (lg->stride_t < lg->V || lg->stride_b < 0)
        return fail(ctx, ORL_E_SHAPE, "strides (%lld, %lld) invalid for V=%lld", (long long)lg->stride_b,
                    (long long)lg->stride_t, (long long)lg->V);
    return ORL_OK;
}

// NEXT-4: the LM-head source (hidden states + unembedding matrix, bf16).
static orl_status validate_rows_lmhead(orl_ctx *ctx, const orl_rows *rows, const orl_lmhead *h,
                                       float inv_temp) {
    if (!h) return fail(ctx, ORL_E_INVALID_ARG, "lmhead is NULL");
    if (!h->hidden || !h->weight) return fail(ctx, ORL_E_INVALID_ARG, "lmhead.hidden and lmhead.weight are required");
    orl_status st = validate_rows(ctx, rows, inv_temp);
    if (st) return st;
    if (h->V < 1 || h->V >= ((int64_t)1 << 31)) return fail(ctx, ORL_E_SHAPE, "V=%lld invalid", (long long)h->V);
    if (h->d < 1 || h->d >= ((int64_t)1 << 31)) return fail(ctx, ORL_E_SHAPE, "d=%lld invalid", (long long)h->d);
    if (h->R < 1 || h->R >= ((int64_t)1 << 31)) return fail(ctx, ORL_E_SHAPE, "R=%lld invalid", (long long)h->R);
    if (h->ld_hidden < h->d || h->ld_weight < h->d)
        return fail(ctx, ORL_E_SHAPE, "row pitches (%lld, %lld) < d=%lld", (long long)h->ld_hidden,
                    (long long)h->ld_weight, (long long)h->d);
    if ((reinterpret_cast<uintptr_t>(h->hidden) | reinterpret_cast<uintptr_t>(h->weight)) % 16 != 0 ||
        (h->ld_hidden * 2) % 16 != 0 || (h->ld_weight * 2) % 16 != 0)
        return fail(ctx, ORL_E_ALIGN, "lmhead rows must be 16-byte aligned (base and pitch)");
    return ORL_OK;
}

static bool tma_eligible(const orl_logits *lg) {
    if (getenv("ORL_FORCE_GENERIC")) return false;
    const int64_t elt = lg->dtype == ORL_BF16 ? 2 : 4;
    const uintptr_t base = reinterpret_cast<uintptr_t>(lg->ptr);
    return (base % 16 == 0) && ((lg->V * elt) % 16 == 0) && ((lg->stride_t * elt) % 16 == 0) &&
           ((lg->stride_b * elt) % 16 == 0);
}

// K1 streaming layout: 1 = TMA, aligned rows; 2 = TMA over each row's 16-byte aligned
// interior with scalar head/tail loads (rows naturally aligned, >= 64 bytes, e.g.
// V = 50257 bf16 or padded pitches); 0 = the generic kernel.
static int k1_layout(const orl_logits *lg) {
    if (tma_eligible(lg)) return 1;
    if (getenv("ORL_FORCE_GENERIC") || getenv("ORL_K1_NO_UNALIGNED_TMA")) return 0;
    const int64_t elt = lg->dtype == ORL_BF16 ? 2 : 4;
    const uintptr_t base = reinterpret_cast<uintptr_t>(lg->ptr);
    return (base % elt == 0) && lg->V * elt >= 64 ? 2 : 0;
}

static void fill_common(orl_ctx *ctx, K1Params &p, const orl_rows *rows, const orl_logits *lg,
                        float inv_temp) {
    std::memset(&p, 0, sizeof p);
    if (lg) {
        p.base = static_cast<const char *>(lg->ptr);
        p.V = lg->V;
        p.stride_b = lg->stride_b;
        p.stride_t = lg->stride_t;
        p.elt = lg->dtype == ORL_BF16 ? 2 : 4;
        p.row_bytes = lg->V * p.elt;
    }
    p.inv_temp = inv_temp;
    p.c2 = inv_temp * 1.4426950408889634f;
    p.poly = kDefaultPoly;  // FMA-pipe exp2 offload: a build-time experiment (-DORL_K1_POLY=8|16), off
    p.B = (int)rows->B;
    p.T = (int)rows->T;
    p.seq_offset = rows->seq_offset;
    p.tokens = rows->tokens;
    p.lengths = rows->lengths;
    p.cu_seqlens = rows->cu_seqlens;
    p.ws = ctx->d_ws;
    p.ws_stride = ctx->ws_stride;
    p.ticket = ctx->d_ticket;
    p.acc = ctx->d_acc;
    p.err = ctx->d_err;
    p.whiten = ctx->d_whiten;
    p.pdl_chain = ctx->pdl_chain;
}

// Large micro-batches (B > kSmemPrefixMax): build the length prefix in global memory.
static orl_status prepare_prefix(orl_ctx *ctx, const orl_rows *rows, bool count_err, cudaStream_t s,
                                 const int32_t **out) {
    *out = nullptr;
    if (rows->B <= kSmemPrefixMax) return ORL_OK;
    if (rows->B > ctx->cum_cap) {
        cudaFree(ctx->d_cum);
        ctx->d_cum = nullptr;
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_cum, (size_t)rows->B * sizeof(int32_t)));
        ctx->cum_cap = rows->B;
    }
    (void)count_err;  // invalid lengths are counted once per iteration, by K3 (orl_advantages)
    CUDA_TRY(ctx, launch_lengths_prefix(rows->lengths + rows->seq_offset, (int)rows->B, (int)rows->T, ctx->d_cum,
                                        nullptr, s));
    ctx->launches += 1;
    *out = ctx->d_cum;
    return ORL_OK;
}

// ------------------------------------------------------------------ context
extern "C" int orl_version(void) { return ORL_VERSION; }

extern "C" orl_status orl_get_unique_id(unsigned char *id_out) {
    if (!id_out) return fail(nullptr, ORL_E_INVALID_ARG, "id_out is NULL");
    ncclUniqueId id;
    NCCL_TRY(nullptr, ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof id);
    return ORL_OK;
}

extern "C" orl_status orl_create(int device, int world, int rank, const unsigned char *id, orl_ctx **out) {
    if (!out) return fail(nullptr, ORL_E_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return fail(nullptr, ORL_E_INVALID_ARG, "world=%d rank=%d invalid", world, rank);
    int ndev = 0;
    CUDA_TRY(nullptr, cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(nullptr, ORL_E_INVALID_ARG, "device %d of %d", device, ndev);
    orl_ctx *ctx = new orl_ctx();
    ctx->device = device;
    ctx->world = world;
    ctx->rank = rank;
    auto cleanup_fail = [&](orl_status st) {
        orl_destroy(ctx);
        return st;
    };
    if (cudaSetDevice(device) != cudaSuccess) return cleanup_fail(fail(nullptr, ORL_E_CUDA, "cudaSetDevice"));
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
        return cleanup_fail(fail(nullptr, ORL_E_CUDA, "cudaGetDeviceProperties"));
    if (prop.major != 10)
        return cleanup_fail(fail(nullptr, ORL_E_CUDA, "liborl is built for sm_100a; device is sm_%d%d",
                                 prop.major, prop.minor));
    ctx->num_sms = prop.multiProcessorCount;
    ctx->ws_stride = ctx->num_sms * 8;
    bool ok = cudaMalloc(&ctx->d_acc, 16 * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_err, kNumErr * sizeof(unsigned long long)) == cudaSuccess &&
              cudaMalloc(&ctx->d_ws, (size_t)kNumPartials * ctx->ws_stride * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_ticket, sizeof(unsigned int)) == cudaSuccess &&
              cudaMalloc(&ctx->d_gather_w, (size_t)kMaxWorld * 4 * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_whiten, kWhitenSlots * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_flags, 4 * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_gather_s, (size_t)kMaxWorld * kStatsSlots * sizeof(double)) == cudaSuccess &&
              cudaMalloc(&ctx->d_stats, kStatsOut * sizeof(double)) == cudaSuccess &&
              cudaMallocHost(&ctx->h_stats, (kStatsOut + 4) * sizeof(double)) == cudaSuccess;
    if (!ok) return cleanup_fail(fail(nullptr, ORL_E_CUDA, "device allocation failed"));
    ok = cudaMemset(ctx->d_acc, 0, 16 * sizeof(double)) == cudaSuccess &&
         cudaMemset(ctx->d_err, 0, kNumErr * sizeof(unsigned long long)) == cudaSuccess &&
         cudaMemset(ctx->d_ticket, 0, sizeof(unsigned int)) == cudaSuccess &&
         cudaMemset(ctx->d_whiten, 0, kWhitenSlots * sizeof(double)) == cudaSuccess &&
         cudaMemset(ctx->d_flags, 0, 4 * sizeof(double)) == cudaSuccess &&
         cudaDeviceSynchronize() == cudaSuccess;
    if (!ok) return cleanup_fail(fail(nullptr, ORL_E_CUDA, "device init failed"));
    if (id) {  // world == 1 with an id: a 1-rank communicator (exercises the NCCL path); no id: peer transport
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        ncclResult_t r = ncclCommInitRank(&ctx->comm, world, uid, rank);
        if (r != ncclSuccess)
            return cleanup_fail(fail(nullptr, ORL_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
    }
    *out = ctx;
    return ORL_OK;
}

extern "C" orl_status orl_destroy(orl_ctx *ctx) {
    if (!ctx) return ORL_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->peer_open)
        for (int r = 0; r < ctx->world; ++r)
            if (r != ctx->rank && ctx->peer.x[r]) cudaIpcCloseMemHandle(ctx->peer.x[r]);
    cudaFree(ctx->d_x);
    cudaFree(ctx->d_epoch);
    cudaFree(ctx->d_acc);
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_ws);
    cudaFree(ctx->d_ticket);
    cudaFree(ctx->d_seq_part);
    cudaFree(ctx->d_gather_w);
    cudaFree(ctx->d_whiten);
    cudaFree(ctx->d_flags);
    cudaFree(ctx->d_gather_s);
    cudaFree(ctx->d_stats);
    cudaFree(ctx->d_cum);
    cudaFree(ctx->d_lm_parts);
    if (ctx->h_stats) cudaFreeHost(ctx->h_stats);
    delete ctx;
    return ORL_OK;
}

extern "C" const char *orl_last_error(const orl_ctx *ctx) {
    return ctx ? ctx->err.c_str() : g_thread_err.c_str();
}

extern "C" uint64_t orl_launch_count(const orl_ctx *ctx) { return ctx ? ctx->launches : 0; }

extern "C" orl_status orl_set_pdl_chain(orl_ctx *ctx, int enable) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    ctx->pdl_chain = enable ? 1 : 0;
    return ORL_OK;
}

extern "C" int orl_get_pdl_chain(const orl_ctx *ctx) { return ctx ? ctx->pdl_chain : -1; }

extern "C" orl_status orl_begin_iteration(orl_ctx *ctx, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_acc, 0, 16 * sizeof(double), s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_err, 0, kNumErr * sizeof(unsigned long long), s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_whiten, 0, kWhitenSlots * sizeof(double), s));
    CUDA_TRY(ctx, cudaMemsetAsync(ctx->d_flags, 0, 4 * sizeof(double), s));
    ctx->have_adv = ctx->have_whiten = false;
    ctx->imported_w = ctx->imported_s = 0;
    return ORL_OK;
}

// ------------------------------------------------------------------ S1 (+S2/S3)
// NEXT-4: K6 (tcgen05 LM-head GEMM -> per-split online partials) then the
// merge kernel with K1's row epilogue in `mode`.
static orl_status run_lmhead(orl_ctx *ctx, K1Params &p, const orl_lmhead *h, int mode, cudaStream_t s) {
    K6Params q;
    std::memset(&q, 0, sizeof q);
    q.R = h->R;
    q.d = (int)h->d;
    q.V = (int)h->V;
    q.c2 = p.c2;
    q.B = p.B;
    q.T = p.T;
    q.seq_offset = p.seq_offset;
    q.tokens = p.tokens;
    q.lengths = p.lengths;
    q.cu_seqlens = p.cu_seqlens;
    k6_plan(q, ctx->num_sms);
    const int64_t need = (int64_t)q.n_split * q.R;
    if (need > ctx->lm_cap) {
        CUDA_TRY(ctx, cudaStreamSynchronize(s));
        cudaFree(ctx->d_lm_parts);
        ctx->d_lm_parts = nullptr;
        ctx->lm_cap = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_lm_parts, (size_t)need * sizeof(float4)));
        ctx->lm_cap = need;
    }
    q.parts = ctx->d_lm_parts;
    q.part_stride = q.R;
    CUDA_TRY(ctx, launch_k6(q, h->hidden, h->ld_hidden, h->weight, h->ld_weight, s));
    p.V = h->V;
    p.lm_parts = ctx->d_lm_parts;
    p.lm_stride = q.R;
    p.lm_R = q.R;
    p.lm_nsplit = q.n_split;
    p.lm_split_cols = q.tiles_per_split * kLmTileN;
    CUDA_TRY(ctx, launch_k6_merge(p, mode, ctx->num_sms, s));
    ctx->launches += 2;
    return ORL_OK;
}

static orl_status logprobs_impl(orl_ctx *ctx, const orl_rows *rows, const orl_logits *logits,
                                const orl_lmhead *head, float inv_temp, float *logp, float *entropy,
                                float *lse, float *gathered, const float *partner_logp, int kl_est,
                                double beta_reward, const float *seq_reward, float *kl,
                                float *shaped_reward, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    orl_status st = head ? validate_rows_lmhead(ctx, rows, head, inv_temp)
                         : validate_rows_logits(ctx, rows, logits, inv_temp);
    if (st) return st;
    if (!logp) return fail(ctx, ORL_E_INVALID_ARG, "logp is required");
    if (!aligned4(logp) || !aligned4(entropy) || !aligned4(lse) || !aligned4(gathered) ||
        !aligned4(partner_logp) || !aligned4(seq_reward) || !aligned4(kl) || !aligned4(shaped_reward))
        return fail(ctx, ORL_E_ALIGN, "per-token arrays must be 4-byte aligned");
    if ((kl || shaped_reward) && !partner_logp)
        return fail(ctx, ORL_E_INVALID_ARG, "kl/shaped_reward need partner_logp");
    if (partner_logp && (kl_est < 1 || kl_est > 3))
        return fail(ctx, ORL_E_INVALID_ARG, "kl_est=%d not in {1,2,3}", kl_est);
    if (shaped_reward && !seq_reward) return fail(ctx, ORL_E_INVALID_ARG, "shaped_reward needs seq_reward");
    if (!std::isfinite(beta_reward)) return fail(ctx, ORL_E_INVALID_ARG, "beta_reward not finite");
    if ((st = set_device(ctx))) return st;
    K1Params p;
    fill_common(ctx, p, rows, logits, inv_temp);
    p.logp = logp;
    p.entropy = entropy;
    p.lse = lse;
    p.gathered = gathered;
    p.partner = partner_logp;
    p.kl_est = kl_est;
    p.beta_reward = beta_reward;
    p.seq_reward = seq_reward;
    p.kl_out = kl;
    p.shaped = shaped_reward;
    if ((st = prepare_prefix(ctx, rows, true, as_stream(stream), &p.cum_global))) return st;
    if (head) return run_lmhead(ctx, p, head, kModeLogprob, as_stream(stream));
    const int lay = k1_layout(logits);
    p.unaligned = lay == 2;
    CUDA_TRY(ctx, launch_k1(p, lay != 0, kModeLogprob, ctx->num_sms, as_stream(stream)));
    ctx->launches += 1;
    return ORL_OK;
}

extern "C" orl_status orl_logprobs(orl_ctx *ctx, const orl_rows *rows, const orl_logits *logits,
                                   float inv_temp, float *logp, float *entropy, float *lse,
                                   float *gathered, const float *partner_logp, int kl_est,
                                   double beta_reward, const float *seq_reward, float *kl,
                                   float *shaped_reward, void *stream) {
    return logprobs_impl(ctx, rows, logits, nullptr, inv_temp, logp, entropy, lse, gathered, partner_logp,
                         kl_est, beta_reward, seq_reward, kl, shaped_reward, stream);
}

extern "C" orl_status orl_lmhead_logprobs(orl_ctx *ctx, const orl_rows *rows, const orl_lmhead *head,
                                          float inv_temp, float *logp, float *entropy, float *lse,
                                          float *gathered, const float *partner_logp, int kl_est,
                                          double beta_reward, const float *seq_reward, float *kl,
                                          float *shaped_reward, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!head) return fail(ctx, ORL_E_INVALID_ARG, "lmhead is NULL");
    return logprobs_impl(ctx, rows, nullptr, head, inv_temp, logp, entropy, lse, gathered, partner_logp,
                         kl_est, beta_reward, seq_reward, kl, shaped_reward, stream);
}

// ------------------------------------------------------------------ S4/S4'/S5
extern "C" orl_status orl_advantages(orl_ctx *ctx, int64_t B, int64_t T, const int32_t *lengths,
                                     int kind, double gamma, double lambda, int group_size,
                                     const float *shaped_reward, const float *values,
                                     const float *seq_reward, float *adv, float *adv_lo, float *ret,
                                     uint8_t *group_keep, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (B < 1 || B > (1 << 24) || T < 1 || T > INT32_MAX || B * T >= ((int64_t)1 << 40))
        return fail(ctx, ORL_E_SHAPE, "B=%lld T=%lld invalid (1 <= B <= 2^24, 1 <= T <= 2^31-1, B*T < 2^40)",
                    (long long)B, (long long)T);
    if (kind < ORL_ADV_GAE || kind > ORL_ADV_RPP_BASELINE)
        return fail(ctx, ORL_E_INVALID_ARG, "unknown advantage kind %d", kind);
    if (!lengths || !adv) return fail(ctx, ORL_E_INVALID_ARG, "lengths and adv are required");
    if (!(gamma >= 0.0 && gamma <= 1.0) || !(lambda >= 0.0 && lambda <= 1.0))
        return fail(ctx, ORL_E_INVALID_ARG, "gamma=%g lambda=%g must be in [0,1]", gamma, lambda);
    const bool grouped = kind == ORL_ADV_GRPO || kind == ORL_ADV_RPP_BASELINE;
    if (kind == ORL_ADV_GAE && (!shaped_reward || !values))
        return fail(ctx, ORL_E_INVALID_ARG, "GAE needs shaped_reward and values");
    if ((kind == ORL_ADV_RPP || kind == ORL_ADV_RPP_BASELINE) && !shaped_reward)
        return fail(ctx, ORL_E_INVALID_ARG, "REINFORCE++ needs shaped_reward");
    if (grouped && !seq_reward) return fail(ctx, ORL_E_INVALID_ARG, "group advantages need seq_reward");
    if (grouped && (group_size < 1 || B % group_size != 0))
        return fail(ctx, ORL_E_GROUP_SPLIT, "B=%lld is not a multiple of group_size=%d", (long long)B, group_size);
    if (!aligned4(lengths) || !aligned4(shaped_reward) || !aligned4(values) || !aligned4(seq_reward) ||
        !aligned4(adv) || !aligned4(adv_lo) || !aligned4(ret))
        return fail(ctx, ORL_E_ALIGN, "per-token arrays must be 4-byte aligned");
    orl_status st = set_device(ctx);
    if (st) return st;
    if (B > ctx->seq_cap) {
        cudaFree(ctx->d_seq_part);
        ctx->d_seq_part = nullptr;
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_seq_part, (size_t)B * 3 * sizeof(double)));
        ctx->seq_cap = B;
    }
    K3Params p;
    std::memset(&p, 0, sizeof p);
    p.B = (int)B;
    p.T = (int)T;
    p.kind = kind;
    p.G = grouped ? group_size : 1;
    p.gamma = gamma;
    p.lambda = lambda;
    p.lengths = lengths;
    p.shaped = shaped_reward;
    p.values = values;
    p.seq_reward = seq_reward;
    p.adv = adv;
    p.adv_lo = adv_lo;
    p.ret = ret;
    p.keep = grouped ? group_keep : nullptr;
    p.seq_part = ctx->d_seq_part;
    p.err = ctx->d_err;
    CUDA_TRY(ctx, launch_k3(p, as_stream(stream)));
    ctx->launches += 1;
    ctx->adv_B = B;
    ctx->have_adv = true;
    ctx->have_whiten = false;
    return ORL_OK;
}

// ------------------------------------------------------------------ S6 + C1
extern "C" orl_status orl_whiten_stats(orl_ctx *ctx, int whiten, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!ctx->have_adv && !ctx->imported_w)
        return fail(ctx, ORL_E_STATE, "orl_whiten_stats before orl_advantages");
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    int world = ctx->world;
    if (!ctx->imported_w && ctx->world > 1 && ctx->coll == 1) {  // C1 as one peer-memory kernel
        PeerArgs pa = ctx->peer;
        pa.epoch = ctx->d_epoch;
        CUDA_TRY(ctx, launch_whiten_peer(ctx->d_seq_part, (int)ctx->adv_B, pa, whiten ? 1 : 0, ctx->d_whiten,
                                         ctx->d_flags, s));
        ctx->launches += 1;
        ctx->have_whiten = true;
        return ORL_OK;
    }
    if (!ctx->imported_w && ctx->world > 1 && !ctx->comm)
        return fail(ctx, ORL_E_STATE, "world > 1 without a transport: create with a unique id or call orl_peer_open");
    if (ctx->imported_w) {
        world = ctx->imported_w;
    } else {
        CUDA_TRY(ctx, launch_whiten_local(ctx->d_seq_part, (int)ctx->adv_B, ctx->d_gather_w + 4 * ctx->rank, s));
        ctx->launches += 1;
        if (ctx->comm) {
            NCCL_TRY(ctx, ncclAllGather(ctx->d_gather_w + 4 * ctx->rank, ctx->d_gather_w, 4, ncclDouble,
                                        ctx->comm, s));
        }
    }
    CUDA_TRY(ctx, launch_whiten_merge(ctx->d_gather_w, world, whiten ? 1 : 0, ctx->d_whiten, ctx->d_flags, s));
    ctx->launches += 1;
    ctx->imported_w = 0;
    ctx->have_whiten = true;
    return ORL_OK;
}

// ------------------------------------------------------------------ S1 + S7..S9
struct GradOut {  // optional fused backward (orl_ppo_loss_and_grad)
    void *dlogits;
    int64_t stride_b, stride_t;
    int zero_masked;
};

static orl_status ppo_loss_impl(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor, float inv_temp,
                                const orl_ppo_cfg *cfg, const float *logp_old, const float *logp_ref,
                                const float *adv, const float *adv_lo, const float *ret, const float *v_new,
                                const float *v_old, float *logp_new, float *entropy, float *lse, float *dloss_dlogp,
                                float *dloss_dv, uint8_t *flags, const GradOut *grad, void *stream,
                                const orl_lmhead *head = nullptr) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    orl_status st = head ? validate_rows_lmhead(ctx, rows, head, inv_temp)
                         : validate_rows_logits(ctx, rows, actor, inv_temp);
    if (st) return st;
    if (!cfg || !logp_old || !adv || !logp_new)
        return fail(ctx, ORL_E_INVALID_ARG, "cfg, logp_old, adv and logp_new are required");
    const int critic = (ret != nullptr) + (v_new != nullptr) + (v_old != nullptr);
    if (critic != 0 && critic != 3) return fail(ctx, ORL_E_INVALID_ARG, "ret, v_new, v_old go together");
    if (dloss_dv && critic == 0) return fail(ctx, ORL_E_INVALID_ARG, "dloss_dv needs the critic arrays");
    if (!aligned4(logp_old) || !aligned4(logp_ref) || !aligned4(adv) || !aligned4(adv_lo) || !aligned4(ret) ||
        !aligned4(v_new) ||
        !aligned4(v_old) || !aligned4(logp_new) || !aligned4(entropy) || !aligned4(dloss_dlogp) ||
        !aligned4(dloss_dv) || !aligned4(lse))
        return fail(ctx, ORL_E_ALIGN, "per-token arrays must be 4-byte aligned");
    if (!(cfg->eps_low >= 0.0 && cfg->eps_low < 1.0) || !(cfg->eps_high >= 0.0) ||
        !std::isfinite(cfg->eps_high) || !std::isfinite(cfg->eps_value) || !std::isfinite(cfg->c1) ||
        !std::isfinite(cfg->c2) || !std::isfinite(cfg->beta_loss) || !(cfg->ratio_guard > 0.0))
        return fail(ctx, ORL_E_INVALID_ARG, "invalid orl_ppo_cfg values");
    if (cfg->kl_loss_est < 1 || cfg->kl_loss_est > 3)
        return fail(ctx, ORL_E_INVALID_ARG, "kl_loss_est=%d not in {1,2,3}", cfg->kl_loss_est);
    if (cfg->loss_agg != 0 && cfg->loss_agg != 1)
        return fail(ctx, ORL_E_INVALID_ARG, "loss_agg=%d not in {0,1}", cfg->loss_agg);
    if (cfg->kl_in_loss && !logp_ref) return fail(ctx, ORL_E_INVALID_ARG, "kl_in_loss needs logp_ref");
    if (!ctx->have_whiten) return fail(ctx, ORL_E_STATE, "orl_ppo_loss before orl_whiten_stats");
    if ((st = set_device(ctx))) return st;
    K1Params p;
    fill_common(ctx, p, rows, actor, inv_temp);
    p.logp = logp_new;
    p.entropy = entropy;
    p.lse = lse;
    p.logp_old = logp_old;
    p.logp_ref = logp_ref;
    p.adv = adv;
    p.adv_lo = adv_lo;
    p.ret = ret;
    p.v_new = v_new;
    p.v_old = v_old;
    p.dlogp = dloss_dlogp;
    p.dv = dloss_dv;
    p.flags = flags;
    p.eps_low = cfg->eps_low;
    p.eps_high = cfg->eps_high;
    p.eps_v = cfg->eps_value;
    p.c1 = cfg->c1;
    p.beta_loss = cfg->beta_loss;
    p.ratio_guard = cfg->ratio_guard;
    p.kl_loss_est = cfg->kl_loss_est;
    p.kl_in_loss = cfg->kl_in_loss;
    p.loss_agg = cfg->loss_agg;
    if ((st = prepare_prefix(ctx, rows, true, as_stream(stream), &p.cum_global))) return st;
    if (head) return run_lmhead(ctx, p, head, kModeLoss, as_stream(stream));
    const int lay = k1_layout(actor);
    const bool tma = lay == 1;
    p.unaligned = lay == 2;
    if (!grad) {
        CUDA_TRY(ctx, launch_k1(p, lay != 0, kModeLoss, ctx->num_sms, as_stream(stream)));
        ctx->launches += 1;
        return ORL_OK;
    }
    // fused actor forward + backward (NEXT-1): one TMA launch when both the logits
    // and dlogits layouts allow it, else the loss pass followed by the K5 pass.
    const int64_t elt = p.elt;
    const bool out_ok = (reinterpret_cast<uintptr_t>(grad->dlogits) % 16 == 0) &&
                        ((grad->stride_t * elt) % 16 == 0) && ((grad->stride_b * elt) % 16 == 0);
    // unaligned rows: fused too when every dlogits row is misaligned like its logits row
    const intptr_t dgap = reinterpret_cast<intptr_t>(grad->dlogits) - reinterpret_cast<intptr_t>(actor->ptr);
    const bool out_same = lay == 2 && dgap % 16 == 0 && ((grad->stride_t - actor->stride_t) * elt) % 16 == 0 &&
                          ((grad->stride_b - actor->stride_b) * elt) % 16 == 0 &&
                          reinterpret_cast<uintptr_t>(grad->dlogits) % elt == 0;
    if ((tma && out_ok) || out_same) {
        p.unaligned = out_same ? 1 : 0;
        p.dlogits = grad->dlogits;
        p.out_stride_b = grad->stride_b;
        p.out_stride_t = grad->stride_t;
        p.c2_ent = cfg->c2;
        p.zero_masked_grad = grad->zero_masked;
        CUDA_TRY(ctx, launch_k1(p, true, kModeLossGrad, ctx->num_sms, as_stream(stream)));
        ctx->launches += 1;
        return ORL_OK;
    }
    CUDA_TRY(ctx, launch_k1(p, lay != 0, kModeLoss, ctx->num_sms, as_stream(stream)));
    ctx->launches += 1;
    return orl_logits_grad(ctx, rows, actor, inv_temp, cfg, lse, entropy, dloss_dlogp, grad->dlogits,
                           grad->stride_b, grad->stride_t, grad->zero_masked, stream);
}

extern "C" orl_status orl_ppo_loss(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                                   float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                                   const float *logp_ref, const float *adv, const float *adv_lo,
                                   const float *ret, const float *v_new, const float *v_old, float *logp_new,
                                   float *entropy, float *lse, float *dloss_dlogp, float *dloss_dv,
                                   uint8_t *flags, void *stream) {
    return ppo_loss_impl(ctx, rows, actor, inv_temp, cfg, logp_old, logp_ref, adv, adv_lo, ret, v_new, v_old,
                         logp_new, entropy, lse, dloss_dlogp, dloss_dv, flags, nullptr, stream);
}

extern "C" orl_status orl_lmhead_ppo_loss(orl_ctx *ctx, const orl_rows *rows, const orl_lmhead *head,
                                          float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                                          const float *logp_ref, const float *adv, const float *adv_lo,
                                          const float *ret, const float *v_new, const float *v_old,
                                          float *logp_new, float *entropy, float *lse, float *dloss_dlogp,
                                          float *dloss_dv, uint8_t *flags, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!head) return fail(ctx, ORL_E_INVALID_ARG, "lmhead is NULL");
    return ppo_loss_impl(ctx, rows, nullptr, inv_temp, cfg, logp_old, logp_ref, adv, adv_lo, ret, v_new, v_old,
                         logp_new, entropy, lse, dloss_dlogp, dloss_dv, flags, nullptr, stream, head);
}

extern "C" orl_status orl_ppo_loss_and_grad(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                                            float inv_temp, const orl_ppo_cfg *cfg, const float *logp_old,
                                            const float *logp_ref, const float *adv, const float *adv_lo,
                                            const float *ret, const float *v_new, const float *v_old,
                                            float *logp_new,
                                            float *entropy, float *lse, float *dloss_dlogp, float *dloss_dv,
                                            uint8_t *flags, void *dlogits, int64_t out_stride_b,
                                            int64_t out_stride_t, int zero_masked, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!actor || !dlogits || !entropy || !lse || !dloss_dlogp)
        return fail(ctx, ORL_E_INVALID_ARG, "dlogits, entropy, lse and dloss_dlogp are required");
    if (out_stride_t < actor->V || out_stride_b < 0)
        return fail(ctx, ORL_E_SHAPE, "dlogits strides (%lld, %lld) invalid", (long long)out_stride_b,
                    (long long)out_stride_t);
    const GradOut g{dlogits, out_stride_b, out_stride_t, zero_masked ? 1 : 0};
    return ppo_loss_impl(ctx, rows, actor, inv_temp, cfg, logp_old, logp_ref, adv, adv_lo, ret, v_new, v_old,
                         logp_new, entropy, lse, dloss_dlogp, dloss_dv, flags, &g, stream);
}

// ------------------------------------------------------------------ NEXT-1
extern "C" orl_status orl_logits_grad(orl_ctx *ctx, const orl_rows *rows, const orl_logits *actor,
                                      float inv_temp, const orl_ppo_cfg *cfg, const float *lse,
                                      const float *entropy, const float *dloss_dlogp, void *dlogits,
                                      int64_t out_stride_b, int64_t out_stride_t, int zero_masked,
                                      void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    orl_status st = validate_rows_logits(ctx, rows, actor, inv_temp);
    if (st) return st;
    if (!cfg || !lse || !entropy || !dloss_dlogp || !dlogits)
        return fail(ctx, ORL_E_INVALID_ARG, "cfg, lse, entropy, dloss_dlogp and dlogits are required");
    if (!aligned4(lse) || !aligned4(entropy) || !aligned4(dloss_dlogp))
        return fail(ctx, ORL_E_ALIGN, "per-token arrays must be 4-byte aligned");
    if (out_stride_t < actor->V || out_stride_b < 0)
        return fail(ctx, ORL_E_SHAPE, "dlogits strides (%lld, %lld) invalid", (long long)out_stride_b,
                    (long long)out_stride_t);
    if (!std::isfinite(cfg->c2)) return fail(ctx, ORL_E_INVALID_ARG, "cfg->c2 not finite");
    if (!ctx->have_whiten) return fail(ctx, ORL_E_STATE, "orl_logits_grad before orl_whiten_stats");
    if ((st = set_device(ctx))) return st;
    K5Params p;
    std::memset(&p, 0, sizeof p);
    p.base = static_cast<const char *>(actor->ptr);
    p.out = dlogits;
    p.V = actor->V;
    p.stride_b = actor->stride_b;
    p.stride_t = actor->stride_t;
    p.out_stride_b = out_stride_b;
    p.out_stride_t = out_stride_t;
    p.elt = actor->dtype == ORL_BF16 ? 2 : 4;
    p.inv_temp = inv_temp;
    p.c2x = inv_temp * 1.4426950408889634f;
    p.c2 = cfg->c2;
    p.B = (int)rows->B;
    p.T = (int)rows->T;
    p.seq_offset = rows->seq_offset;
    p.tokens = rows->tokens;
    p.lengths = rows->lengths;
    p.cu_seqlens = rows->cu_seqlens;
    p.lse = lse;
    p.entropy = entropy;
    p.dlogp = dloss_dlogp;
    p.whiten = ctx->d_whiten;
    p.zero_masked = zero_masked ? 1 : 0;
    p.loss_agg = cfg->loss_agg;
    const int64_t elt = p.elt;
    bool tma = tma_eligible(actor) && (reinterpret_cast<uintptr_t>(dlogits) % 16 == 0) &&
               ((out_stride_t * elt) % 16 == 0) && ((out_stride_b * elt) % 16 == 0);
    if (!tma && k1_layout(actor) == 2) {
        // unaligned rows: TMA over the aligned interiors when every output row is misaligned
        // exactly like its input row (same offset mod 16), scalar heads and tails
        const intptr_t dbase = reinterpret_cast<intptr_t>(dlogits) - reinterpret_cast<intptr_t>(actor->ptr);
        p.unaligned = (dbase % 16 == 0) && (((out_stride_t - actor->stride_t) * elt) % 16 == 0) &&
                      (((out_stride_b - actor->stride_b) * elt) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(dlogits) % elt == 0);
        tma = p.unaligned != 0;
    }
    if ((st = prepare_prefix(ctx, rows, false, as_stream(stream), &p.cum_global))) return st;
    CUDA_TRY(ctx, launch_k5(p, tma, ctx->num_sms, as_stream(stream)));
    ctx->launches += 1;
    return ORL_OK;
}

// ------------------------------------------------------------------ S10 + C2
// C2 and the final statistics on `s` (no copies, no host synchronisation).
static orl_status finalize_launch(orl_ctx *ctx, const orl_ppo_cfg *cfg, cudaStream_t s) {
    int world = ctx->world;
    if (!ctx->imported_s && ctx->world > 1 && ctx->coll == 0 && !ctx->comm)
        return fail(ctx, ORL_E_STATE, "world > 1 without a transport: create with a unique id or call orl_peer_open");
    if (!ctx->imported_s && ctx->world > 1 && ctx->coll == 1) {  // C2 as one peer-memory kernel
        PeerArgs pa = ctx->peer;
        pa.epoch = ctx->d_epoch + 1;
        CUDA_TRY(ctx, launch_stats_peer(ctx->d_acc, ctx->d_err, pa, ctx->d_whiten, ctx->d_flags, cfg->c1, cfg->c2,
                                        cfg->beta_loss, cfg->kl_in_loss, cfg->loss_agg, ctx->d_stats, s));
        ctx->launches += 1;
        ctx->imported_s = 0;
        return ORL_OK;
    }
    if (ctx->imported_s) {
        world = ctx->imported_s;
    } else {
        CUDA_TRY(ctx, launch_stats_pack(ctx->d_acc, ctx->d_err, ctx->d_gather_s + kStatsSlots * ctx->rank, s));
        ctx->launches += 1;
        if (ctx->comm)
            NCCL_TRY(ctx, ncclAllGather(ctx->d_gather_s + kStatsSlots * ctx->rank, ctx->d_gather_s,
                                        kStatsSlots, ncclDouble, ctx->comm, s));
    }
    CUDA_TRY(ctx, launch_stats_final(ctx->d_gather_s, world, ctx->d_whiten, ctx->d_flags, cfg->c1, cfg->c2,
                                     cfg->beta_loss, cfg->kl_in_loss, cfg->loss_agg, ctx->d_stats, s));
    ctx->launches += 1;
    ctx->imported_s = 0;
    return ORL_OK;
}

extern "C" orl_status orl_stats_decode(const double *h, double ratio_guard, orl_stats *host_out) {
    if (!h) return fail(nullptr, ORL_E_INVALID_ARG, "stats vector is NULL");
    if (host_out) {
        host_out->n_tokens = h[0];
        host_out->policy_loss = h[1];
        host_out->value_loss = h[2];
        host_out->entropy = h[3];
        host_out->kl = h[4];
        host_out->approx_kl_old = h[5];
        host_out->clip_frac = h[6];
        host_out->value_clip_frac = h[7];
        host_out->ratio_mean = h[8];
        host_out->total_loss = h[9];
        host_out->adv_mean = h[10];
        host_out->adv_std = h[11];
        host_out->n_guard = (int64_t)h[12];
        host_out->n_nonfinite = (int64_t)h[13];
        host_out->n_token_range = (int64_t)h[14];
        host_out->whiten_warn = h[15] != 0.0;
        host_out->pad_ = 0;
    }
    const double mask_err = h[kStatsOut + 1];
    if (h[kStatsOut + 2] > 0)
        return fail(nullptr, ORL_E_NCCL, "peer-memory collective: %lld wait(s) timed out (a rank did not arrive)",
                    (long long)h[kStatsOut + 2]);
    if (h[14] > 0) return fail(nullptr, ORL_E_TOKEN_RANGE, "%lld token(s) outside [0, V)", (long long)h[14]);
    if (mask_err > 0)
        return fail(nullptr, ORL_E_MASK, "%lld invalid length(s) / non-prefix attention-mask row(s)",
                    (long long)mask_err);
    if (h[kStatsOut + 3] > 0)
        return fail(nullptr, ORL_E_SHAPE, "%lld valid token(s) map to LM-head rows beyond the hidden matrix",
                    (long long)h[kStatsOut + 3]);
    if (h[13] > 0) return fail(nullptr, ORL_E_NONFINITE, "%lld non-finite value(s)", (long long)h[13]);
    if (h[12] > 0)
        return fail(nullptr, ORL_E_NUMERIC_GUARD, "%lld token(s) with |logp_new - logp_old| > %g", (long long)h[12],
                    ratio_guard);
    if (!(h[0] > 0)) return fail(nullptr, ORL_E_EMPTY_BATCH, "no valid tokens");
    return ORL_OK;
}

extern "C" orl_status orl_finalize_async(orl_ctx *ctx, const orl_ppo_cfg *cfg, double *dev_out, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!cfg || !dev_out) return fail(ctx, ORL_E_INVALID_ARG, "cfg/dev_out is NULL");
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    if ((st = finalize_launch(ctx, cfg, s))) return st;
    CUDA_TRY(ctx, cudaMemcpyAsync(dev_out, ctx->d_stats, kStatsOut * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(dev_out + kStatsOut, ctx->d_flags, 4 * sizeof(double), cudaMemcpyDeviceToDevice,
                                  s));
    return ORL_OK;
}

extern "C" orl_status orl_finalize(orl_ctx *ctx, const orl_ppo_cfg *cfg, orl_stats *host_out,
                                   double *dev_out, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (!cfg) return fail(ctx, ORL_E_INVALID_ARG, "cfg is NULL");
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    if ((st = finalize_launch(ctx, cfg, s))) return st;
    if (dev_out)
        CUDA_TRY(ctx, cudaMemcpyAsync(dev_out, ctx->d_stats, kStatsOut * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, kStatsOut * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaMemcpyAsync(ctx->h_stats + kStatsOut, ctx->d_flags, 4 * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    st = orl_stats_decode(ctx->h_stats, cfg->ratio_guard, host_out);
    if (st) ctx->err = g_thread_err;
    return st;
}

// ------------------------------------------------------------------ NEXT-3
extern "C" orl_status orl_kl_controller_step(double *beta, double target, double horizon, double observed_kl,
                                             double max_kl, int *early_stop) {
    if (!beta || !early_stop) return fail(nullptr, ORL_E_INVALID_ARG, "beta/early_stop is NULL");
    if (!(*beta >= 0.0) || !(target > 0.0) || !(horizon > 0.0) || !std::isfinite(observed_kl))
        return fail(nullptr, ORL_E_INVALID_ARG, "kl controller: beta=%g target=%g horizon=%g observed=%g", *beta,
                    target, horizon, observed_kl);
    double e = observed_kl / target - 1.0;
    e = e < -0.5 ? -0.5 : (e > 0.5 ? 0.5 : e);
    *beta = *beta * (1.0 + e / horizon);
    *early_stop = observed_kl > max_kl ? 1 : 0;
    return ORL_OK;
}

// ------------------------------------------------------------------ masks
extern "C" orl_status orl_lengths_from_mask(orl_ctx *ctx, int64_t B, int64_t T, const uint8_t *mask,
                                            int32_t *lengths, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (B < 0 || T < 1 || T > INT32_MAX) return fail(ctx, ORL_E_SHAPE, "B=%lld T=%lld", (long long)B, (long long)T);
    if (B > 0 && (!mask || !lengths)) return fail(ctx, ORL_E_INVALID_ARG, "mask/lengths is NULL");
    if (!aligned4(lengths)) return fail(ctx, ORL_E_ALIGN, "lengths must be 4-byte aligned");
    orl_status st = set_device(ctx);
    if (st) return st;
    CUDA_TRY(ctx, launch_mask_lengths(mask, B, T, lengths, ctx->d_err, as_stream(stream)));
    ctx->launches += B > 0 ? 1 : 0;
    return ORL_OK;
}

// ------------------------------------------------------------------ DAPO re-roll list
extern "C" orl_status orl_keep_compact(orl_ctx *ctx, int64_t n_groups, const uint8_t *group_keep,
                                       int32_t *kept_groups, int32_t *n_kept, void *stream) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (n_groups < 0 || n_groups > INT32_MAX) return fail(ctx, ORL_E_SHAPE, "n_groups=%lld", (long long)n_groups);
    if (!n_kept || (n_groups > 0 && (!group_keep || !kept_groups)))
        return fail(ctx, ORL_E_INVALID_ARG, "group_keep/kept_groups/n_kept is NULL");
    if (!aligned4(kept_groups) || !aligned4(n_kept)) return fail(ctx, ORL_E_ALIGN, "outputs must be 4-byte aligned");
    orl_status st = set_device(ctx);
    if (st) return st;
    CUDA_TRY(ctx, launch_keep_compact(group_keep, n_groups, kept_groups, n_kept, as_stream(stream)));
    ctx->launches += 1;
    return ORL_OK;
}

// ------------------------------------------------------------------ workspace
extern "C" orl_status orl_reserve(orl_ctx *ctx, int64_t max_seqs, int64_t max_lm_rows, int64_t max_vocab) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (max_seqs < 0 || max_lm_rows < 0 || max_vocab < 0)
        return fail(ctx, ORL_E_SHAPE, "orl_reserve: negative size");
    orl_status st = set_device(ctx);
    if (st) return st;
    if (max_seqs > ctx->seq_cap) {
        cudaFree(ctx->d_seq_part);
        ctx->d_seq_part = nullptr;
        ctx->seq_cap = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_seq_part, (size_t)max_seqs * 3 * sizeof(double)));
        ctx->seq_cap = max_seqs;
    }
    if (max_seqs > kSmemPrefixMax && max_seqs > ctx->cum_cap) {
        cudaFree(ctx->d_cum);
        ctx->d_cum = nullptr;
        ctx->cum_cap = 0;
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_cum, (size_t)max_seqs * sizeof(int32_t)));
        ctx->cum_cap = max_seqs;
    }
    if (max_lm_rows > 0 && max_vocab > 0) {
        K6Params q;
        std::memset(&q, 0, sizeof q);
        q.R = max_lm_rows;
        q.V = (int)max_vocab;
        q.d = 64;
        k6_plan(q, ctx->num_sms);
        const int64_t need = (int64_t)q.n_split * q.R;
        if (need > ctx->lm_cap) {
            cudaFree(ctx->d_lm_parts);
            ctx->d_lm_parts = nullptr;
            ctx->lm_cap = 0;
            CUDA_TRY(ctx, cudaMalloc(&ctx->d_lm_parts, (size_t)need * sizeof(float4)));
            ctx->lm_cap = need;
        }
    }
    CUDA_TRY(ctx, cudaDeviceSynchronize());
    return ORL_OK;
}

// ------------------------------------------------------------------ peer-memory collectives
extern "C" orl_status orl_peer_handle(orl_ctx *ctx, unsigned char *handle_out) {
    if (!ctx || !handle_out) return fail(ctx, ORL_E_INVALID_ARG, "ctx/handle_out is NULL");
    orl_status st = set_device(ctx);
    if (st) return st;
    if (!ctx->d_x) {
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_x, kXWords * sizeof(unsigned long long)));
        CUDA_TRY(ctx, cudaMemset(ctx->d_x, 0, kXWords * sizeof(unsigned long long)));
        CUDA_TRY(ctx, cudaMalloc(&ctx->d_epoch, 2 * sizeof(unsigned long long)));
        CUDA_TRY(ctx, cudaMemset(ctx->d_epoch, 0, 2 * sizeof(unsigned long long)));
        CUDA_TRY(ctx, cudaDeviceSynchronize());
    }
    cudaIpcMemHandle_t h;
    CUDA_TRY(ctx, cudaIpcGetMemHandle(&h, ctx->d_x));
    std::memcpy(handle_out, &h, sizeof h);
    return ORL_OK;
}

extern "C" orl_status orl_peer_open(orl_ctx *ctx, const unsigned char *handles) {
    if (!ctx || !handles) return fail(ctx, ORL_E_INVALID_ARG, "ctx/handles is NULL");
    if (ctx->world > kPeerMax)
        return fail(ctx, ORL_E_INVALID_ARG, "peer collectives need world <= %d (one NVLink domain)", kPeerMax);
    if (!ctx->d_x) return fail(ctx, ORL_E_STATE, "orl_peer_open before orl_peer_handle");
    if (ctx->peer_open) return fail(ctx, ORL_E_STATE, "peer buffers already open");
    orl_status st = set_device(ctx);
    if (st) return st;
    PeerArgs pa{};
    pa.world = ctx->world;
    pa.rank = ctx->rank;
    pa.spin_limit = 40ll << 20;
    if (const char *e = getenv("ORL_PEER_SPIN_LIMIT")) pa.spin_limit = atoll(e);
    for (int r = 0; r < ctx->world; ++r) {
        if (r == ctx->rank) {
            pa.x[r] = ctx->d_x;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + (size_t)r * sizeof h, sizeof h);
        void *ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int q = 0; q < r; ++q)
                if (q != ctx->rank && pa.x[q]) cudaIpcCloseMemHandle(pa.x[q]);
            return fail(ctx, ORL_E_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r, cudaGetErrorString(e));
        }
        pa.x[r] = static_cast<unsigned long long *>(ptr);
    }
    ctx->peer = pa;
    ctx->peer_open = true;
    ctx->coll = ctx->world > 1 ? 1 : 0;
    return ORL_OK;
}

extern "C" orl_status orl_set_collective(orl_ctx *ctx, int mode) {
    if (!ctx) return fail(nullptr, ORL_E_INVALID_ARG, "ctx is NULL");
    if (mode == 0) {
        if (ctx->world > 1 && !ctx->comm) return fail(ctx, ORL_E_STATE, "no NCCL communicator (created without an id)");
    } else if (mode == 1) {
        if (ctx->world > 1 && !ctx->peer_open) return fail(ctx, ORL_E_STATE, "peer buffers not open (orl_peer_open)");
    } else {
        return fail(ctx, ORL_E_INVALID_ARG, "collective mode %d not in {0, 1}", mode);
    }
    ctx->coll = mode;
    return ORL_OK;
}

extern "C" int orl_get_collective(const orl_ctx *ctx) { return ctx ? ctx->coll : -1; }

// ------------------------------------------------------------------ hooks
extern "C" orl_status orl_export_partials(orl_ctx *ctx, int which, double *host_out, void *stream) {
    if (!ctx || !host_out) return fail(ctx, ORL_E_INVALID_ARG, "ctx/host_out is NULL");
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    if (which == 0) {
        if (!ctx->have_adv) return fail(ctx, ORL_E_STATE, "export of whitening partial before orl_advantages");
        double *slot = ctx->d_gather_w + 4 * ctx->rank;
        CUDA_TRY(ctx, launch_whiten_local(ctx->d_seq_part, (int)ctx->adv_B, slot, s));
        ctx->launches += 1;
        CUDA_TRY(ctx, cudaMemcpyAsync(host_out, slot, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    } else if (which == 1) {
        double *slot = ctx->d_gather_s + kStatsSlots * ctx->rank;
        CUDA_TRY(ctx, launch_stats_pack(ctx->d_acc, ctx->d_err, slot, s));
        ctx->launches += 1;
        CUDA_TRY(ctx, cudaMemcpyAsync(host_out, slot, kStatsSlots * sizeof(double), cudaMemcpyDeviceToHost, s));
    } else {
        return fail(ctx, ORL_E_INVALID_ARG, "which=%d not in {0,1}", which);
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return ORL_OK;
}

extern "C" orl_status orl_import_partials(orl_ctx *ctx, int which, const double *host_all, int world,
                                          void *stream) {
    if (!ctx || !host_all) return fail(ctx, ORL_E_INVALID_ARG, "ctx/host_all is NULL");
    if (world < 1 || world > kMaxWorld) return fail(ctx, ORL_E_INVALID_ARG, "world=%d invalid", world);
    orl_status st = set_device(ctx);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    if (which == 0) {
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_gather_w, host_all, (size_t)world * 4 * sizeof(double),
                                      cudaMemcpyHostToDevice, s));
        ctx->imported_w = world;
    } else if (which == 1) {
        CUDA_TRY(ctx, cudaMemcpyAsync(ctx->d_gather_s, host_all, (size_t)world * kStatsSlots * sizeof(double),
                                      cudaMemcpyHostToDevice, s));
        ctx->imported_s = world;
    } else {
        return fail(ctx, ORL_E_INVALID_ARG, "which=%d not in {0,1}", which);
    }
    CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return ORL_OK;
}

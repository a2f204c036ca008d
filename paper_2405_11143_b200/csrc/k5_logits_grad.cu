// k5_logits_grad.cu -- K5 (NEXT-1): gradient of the minimised PPO total w.r.t.
// the actor's raw logits, one streaming pass (read logits, write dlogits).
//
//   z = inv_temp x,  p = softmax(z),  H = -sum_v p_v ln p_v,  logp_y = z_y - lse
//   dL/dz_v = w (delta_vy - p_v) + a p_v (ln p_v + H),   a = c2 / N
//   dL/dx_v = inv_temp dL/dz_v
// with w = dL/dlogp_new from the actor pass (orl_ppo_loss's dloss_dlogp) and
// lse, H saved by that pass ("gradient computation"; SURVEY
// 8(f) NEXT-1).
//
// Same streaming skeleton as K1 (persistent CTA per SM, producer warp with a
// 1-D TMA bulk-copy ring), but no row reduction: each consumer thread turns its
// 16-byte vectors into gradient vectors and writes them with st.global.v4;
// the per-row constants (y, lse, H, w) are published by the producer.  The
// target element's delta term is patched by its owner thread afterwards.
#include <cuda_runtime.h>

#include <cstdint>

#include "orl_device.cuh"
#include "orl_internal.h"

namespace orl {

namespace k5 {
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;
constexpr int kChunk = 32768;
constexpr int kStages = 6;
constexpr int kRowInfo = 16;
constexpr int kVPT = kChunk / 16 / kConsumers;  // 4
static_assert(kRowInfo >= kStages + 1, "row-info ring must outrun the stage ring");

struct RowInfo {
    int32_t y;
    float l2;   // lse * log2(e)
    float A1;   // inv_temp * a * ln2
    float A0;   // inv_temp * (a H - w)
    float wt;   // inv_temp * w   (the delta term at v = y)
    int32_t h;  // unaligned rows: head bytes before the 16-byte aligned interior
    int32_t pad[2];
    float hx[16];  // unaligned rows: raw head elements, then tail elements
};

struct __align__(128) Smem {
    uint8_t stage[kStages][kChunk];
    uint64_t full[kStages];
    uint64_t empty[kStages];
    RowInfo info[kRowInfo];
};
}  // namespace k5

size_t k5_smem_bytes(int B) {
    return sizeof(k5::Smem) + sizeof(int32_t) * (size_t)((B > kSmemPrefixMax ? 0 : B) + 32);
}

__device__ void k5_build_prefix(const K5Params &p, int32_t *cum, int32_t *warp_tot) {
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

__device__ __forceinline__ void stg128(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint32_t f32x2_to_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// One gradient element written singly (unaligned heads / tails, the target's delta term).
template <typename Tin>
__device__ __forceinline__ void st_elem(Tin *orow, int64_t v, float g) {
    if (sizeof(Tin) == 2) {
        const uint32_t hb = f32x2_to_bf16x2(g, 0.f) & 0xffffu;
        asm volatile("st.global.u16 [%0], %1;" ::"l"(orow + v), "h"((unsigned short)hb) : "memory");
    } else {
        reinterpret_cast<float *>(orow)[v] = g;
    }
}

// Zero one output row of row_bytes at any element-aligned address: scalar head and tail,
// 16-byte stores for the aligned interior; threads ct of nthr share it.
template <typename Tin>
__device__ void zero_row(char *orow, int64_t row_bytes, int ct, int nthr) {
    const int h = (int)((16u - (uint32_t)(reinterpret_cast<uintptr_t>(orow) & 15u)) & 15u);
    const int hb = (int)min((int64_t)h, row_bytes);
    const int64_t ib = (row_bytes - hb) & ~(int64_t)15;
    for (int64_t e = ct; e < hb / (int64_t)sizeof(Tin); e += nthr) reinterpret_cast<Tin *>(orow)[e] = Tin(0);
    for (int64_t o = (int64_t)ct * 16; o < ib; o += (int64_t)nthr * 16) stg128(orow + hb + o, make_uint4(0u, 0u, 0u, 0u));
    const int64_t tail0 = (hb + ib) / (int64_t)sizeof(Tin), V = row_bytes / (int64_t)sizeof(Tin);
    for (int64_t e = tail0 + ct; e < V; e += nthr) reinterpret_cast<Tin *>(orow)[e] = Tin(0);
}

// Row constants from the saved forward quantities.  a = c2/N (token mean) or
// c2/(N_seq L_b) (NEXT-2 sequence mean).
__device__ __forceinline__ k5::RowInfo row_info(const K5Params &p, int64_t gi, int y, int L) {
    const float a = (float)(p.loss_agg == 1 ? p.c2 / (p.whiten[4] * (double)L) : p.c2 / p.whiten[0]);
    k5::RowInfo r;
    const float lse = __ldg(p.lse + gi), H = __ldg(p.entropy + gi), w = __ldg(p.dlogp + gi);
    r.y = y;
    r.l2 = lse * kLog2e;
    r.A1 = p.inv_temp * a * (float)kLn2;
    r.A0 = p.inv_temp * (a * H - w);
    r.wt = p.inv_temp * w;
    return r;
}

// GENT: the loss has an entropy term (c2 != 0): factor A1 t + A0; with c2 = 0 the row constant
// A0 (one FFMA2 per pair less; a -inf logit gets the exact zero gradient, DESIGN Z39).  The
// fused actor pass (K1, kModeLossGrad) makes the same choice, so both paths give the same bits.
template <typename Tin, bool UNAL = false, bool GENT = true>
__global__ void __launch_bounds__(k5::kThreads, 1) k5_tma_kernel(const K5Params p) {
    using namespace k5;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem &S = *reinterpret_cast<Smem *>(smem_raw);
    int32_t *cum_s = reinterpret_cast<int32_t *>(smem_raw + sizeof(Smem));
    int32_t *warp_tot = cum_s + (p.cum_global ? 0 : p.B);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kConsumers);  // every consumer thread releases its own loads
        }
        fence_mbar_init();
    }
    const int32_t *cum = p.cum_global ? p.cum_global : cum_s;
    // Every input (lengths, the prefix, the saved per-token arrays of the actor pass,
    // the logits) may come from the preceding kernel: wait for it before any read.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.cum_global) __syncthreads();
    else k5_build_prefix(p, cum_s, warp_tot);
    const int64_t N = cum[p.B - 1];
    const int64_t row_bytes = p.V * (int64_t)sizeof(Tin);

    if (warp == kConsumerWarps) {
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t j = blockIdx.x, rl = 0; j < N; j += gridDim.x, ++rl) {
                int b, t;
                locate_row(cum, p.B, j, b, t);
                const int64_t gi = (p.seq_offset + b) * (int64_t)p.T + t;
                const RowInfo ri = row_info(p, gi, __ldg(p.tokens + gi), cum[b] - (b > 0 ? cum[b - 1] : 0));
                RowInfo rix = ri;
                const char *src = p.base + logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.stride_b,
                                                             p.stride_t) * (int64_t)sizeof(Tin);
                int64_t ib = row_bytes;
                rix.h = 0;
                if (UNAL) {  // stream the aligned interior; load the head / tail here
                    rix.h = (int)((16u - (uint32_t)(reinterpret_cast<uintptr_t>(src) & 15u)) & 15u);
                    ib = (row_bytes - rix.h) & ~(int64_t)15;
                    const int head_e = rix.h / (int)sizeof(Tin);
                    const int tail_e = (int)((row_bytes - rix.h - ib) / (int64_t)sizeof(Tin));
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const int idx = k < head_e ? k : (k - head_e < tail_e ? (int)p.V - tail_e + (k - head_e) : -1);
                        rix.hx[k] = idx < 0 ? 0.f
                                    : sizeof(Tin) == 2
                                        ? __uint_as_float(((uint32_t)__ldg(reinterpret_cast<const unsigned short *>(src) + idx)) << 16)
                                        : __ldg(reinterpret_cast<const float *>(src) + idx);
                    }
                    src += rix.h;
                }
                for (int64_t off = 0; off < ib; off += kChunk) {
                    const uint32_t bytes = (uint32_t)min((int64_t)kChunk, ib - off);
                    mbar_wait(&S.empty[stage], phase ^ 1u);
                    if (off == 0) S.info[rl % kRowInfo] = rix;
                    mbar_arrive_expect_tx(&S.full[stage], bytes);
                    tma_load_1d(S.stage[stage], src + off, bytes, &S.full[stage], pol);
                    if (++stage == kStages) { stage = 0; phase ^= 1u; }
                }
            }
        }
        return;
    }

    const int ct = tid;
    int stage = 0;
    uint32_t phase = 0;
    const uint64_t c2p = pack2(p.c2x, p.c2x);
    for (int64_t j = blockIdx.x, rl = 0; j < N; j += gridDim.x, ++rl) {
        int b, t;
        locate_row(cum, p.B, j, b, t);
        Tin *orow = reinterpret_cast<Tin *>(p.out) +
                    logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.out_stride_b, p.out_stride_t);
        RowInfo ri;
        uint64_t nl2 = 0, A1p = 0, A0p = 0;
        int64_t ib = row_bytes;  // interior bytes of an unaligned row (set at its first chunk)
        for (int64_t off = 0; off < ib; off += kChunk) {
            mbar_wait(&S.full[stage], phase);
            if (off == 0) {
                ri = S.info[rl % kRowInfo];
                nl2 = pack2(-ri.l2, -ri.l2);
                A1p = pack2(ri.A1, ri.A1);
                A0p = pack2(ri.A0, ri.A0);
                if (UNAL) {
                    ib = (row_bytes - ri.h) & ~(int64_t)15;
                    // the head / tail elements, one per thread, written singly
                    const int head_e = ri.h / (int)sizeof(Tin);
                    const int tail_e = (int)((row_bytes - ri.h - ib) / (int64_t)sizeof(Tin));
                    int idx = -1;
                    if (ct < head_e) idx = ct;
                    else if (ct < head_e + tail_e) idx = (int)p.V - tail_e + (ct - head_e);
                    if (idx >= 0) {
                        const float t2 = fmaf(ri.hx[ct], p.c2x, -ri.l2);
                        float g = __fmul_rn(ex2(t2), GENT ? fmaf(ri.A1, t2, ri.A0) : ri.A0);  // no contraction: same bits on every path
                        if (idx == ri.y) g = __fadd_rn(g, ri.wt);
                        st_elem<Tin>(orow, idx, g);
                    }
                }
            }
            const int bytes = (int)min((int64_t)kChunk, ib - off);
            const int nvec = bytes >> 4;
            const uint8_t *sb = S.stage[stage];
            // owner of the target element reads it before the stage is released
            const int64_t ybyte = (int64_t)ri.y * (int64_t)sizeof(Tin) - (UNAL ? ri.h : 0);  // offset in the interior
            const bool own_y = ri.y >= 0 && (int64_t)ri.y < p.V && ybyte >= 0 && ybyte >= off && ybyte < off + bytes &&
                               (((int)(ybyte - off) >> 4) % kConsumers) == ct;
            float xy = 0.f;
            if (own_y) {
                const uint8_t *q = sb + (ybyte - off);
                xy = sizeof(Tin) == 2 ? __uint_as_float(((uint32_t)*reinterpret_cast<const uint16_t *>(q)) << 16)
                                      : *reinterpret_cast<const float *>(q);
            }
            uint4 v[kVPT];
#pragma unroll
            for (int k = 0; k < kVPT; ++k) {
                const int vi = ct + k * kConsumers;
                if (vi < nvec) v[k] = lds128(sb + vi * 16);
            }
            mbar_arrive(&S.empty[stage]);  // release: this thread's loads of the stage happen before
            if (++stage == kStages) { stage = 0; phase ^= 1u; }
            char *obase = reinterpret_cast<char *>(orow) + (UNAL ? ri.h : 0) + off;
            // dL/dx of one 16-byte vector (the same per-element operations as the fused pass)
            auto grad_vec = [&](const uint4 &vv, uint32_t (&o)[4]) {
                const uint32_t w4[4] = {vv.x, vv.y, vv.z, vv.w};
                if (sizeof(Tin) == 2) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t x = pack2(bf16lo(w4[q]), bf16hi(w4[q]));
                        const uint64_t t2 = ffma2(x, c2p, nl2);          // (z - lse) log2 e
                        float t0, t1;
                        unpack2(t2, t0, t1);
                        const uint64_t pr = pack2(ex2(t0), ex2(t1));     // p
                        const uint64_t g = fmul2(pr, GENT ? ffma2(A1p, t2, A0p) : A0p);
                        float g0, g1;
                        unpack2(g, g0, g1);
                        o[q] = f32x2_to_bf16x2(g0, g1);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        uint64_t x;
                        asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "r"(w4[2 * q]), "r"(w4[2 * q + 1]));
                        const uint64_t t2 = ffma2(x, c2p, nl2);
                        float t0, t1;
                        unpack2(t2, t0, t1);
                        const uint64_t pr = pack2(ex2(t0), ex2(t1));
                        const uint64_t g = fmul2(pr, GENT ? ffma2(A1p, t2, A0p) : A0p);
                        float g0, g1;
                        unpack2(g, g0, g1);
                        o[2 * q] = __float_as_uint(g0);
                        o[2 * q + 1] = __float_as_uint(g1);
                    }
                }
            };
            if (nvec == kVPT * kConsumers) {
                // full chunk: every thread owns kVPT vectors -- one straight-line block (no
                // per-vector branches), so the vectors' MUFU / FMA chains interleave
                uint32_t o[kVPT][4];
#pragma unroll
                for (int k = 0; k < kVPT; ++k) grad_vec(v[k], o[k]);
#pragma unroll
                for (int k = 0; k < kVPT; ++k)
                    stg128(obase + (ct + k * kConsumers) * 16, make_uint4(o[k][0], o[k][1], o[k][2], o[k][3]));
            } else {
#pragma unroll
                for (int k = 0; k < kVPT; ++k) {
                    const int vi = ct + k * kConsumers;
                    if (vi >= nvec) continue;
                    uint32_t o[4];
                    grad_vec(v[k], o);
                    stg128(obase + vi * 16, make_uint4(o[0], o[1], o[2], o[3]));
                }
            }
            // delta term at v = y: the owner of y's vector rewrites that element
            if (own_y) {
                const float t2 = fmaf(xy, p.c2x, -ri.l2);
                const float g = __fadd_rn(__fmul_rn(ex2(t2), GENT ? fmaf(ri.A1, t2, ri.A0) : ri.A0), ri.wt);  // not contracted
                st_elem<Tin>(orow, ri.y, g);
            }
        }
    }
    // zero the masked rows of the output block (t >= L_b)
    if (p.zero_masked && !p.cu_seqlens) {  // packed outputs have no masked rows
        const int64_t total = (int64_t)p.B * p.T;
        for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
            const int b = (int)(q / p.T), t = (int)(q % p.T);
            const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
            if (t < L) continue;
            char *orow = reinterpret_cast<char *>(p.out) +
                         ((int64_t)b * p.out_stride_b + (int64_t)t * p.out_stride_t) * (int64_t)sizeof(Tin);
            zero_row<Tin>(orow, row_bytes, ct, kConsumers);
        }
    }
}

// Generic path (unaligned rows): one row per CTA iteration, scalar accesses.
template <typename Tin, bool GENT = true>
__global__ void __launch_bounds__(256) k5_generic_kernel(const K5Params p) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    int32_t *cum_s = reinterpret_cast<int32_t *>(smem_raw);
    int32_t *warp_tot = cum_s + (p.cum_global ? 0 : p.B);
    const int32_t *cum = p.cum_global ? p.cum_global : cum_s;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // inputs may come from the preceding kernel
    if (p.cum_global) __syncthreads();
    else k5_build_prefix(p, cum_s, warp_tot);
    const int64_t total = (int64_t)p.B * p.T;
    for (int64_t q = blockIdx.x; q < total; q += gridDim.x) {
        const int b = (int)(q / p.T), t = (int)(q % p.T);
        const int L = cum[b] - (b > 0 ? cum[b - 1] : 0);
        if (t >= L) {
            if (p.cu_seqlens) continue;  // packed: no masked rows exist
            Tin *orow = reinterpret_cast<Tin *>(p.out) + (int64_t)b * p.out_stride_b + (int64_t)t * p.out_stride_t;
            if (p.zero_masked)
                for (int64_t v = threadIdx.x; v < p.V; v += blockDim.x) orow[v] = Tin(0);
            continue;
        }
        Tin *orow = reinterpret_cast<Tin *>(p.out) +
                    logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.out_stride_b, p.out_stride_t);
        const Tin *row = reinterpret_cast<const Tin *>(p.base) +
                         logits_row_offset(p.cu_seqlens, p.seq_offset, b, t, p.stride_b, p.stride_t);
        const int64_t gi = (p.seq_offset + b) * (int64_t)p.T + t;
        const k5::RowInfo ri = row_info(p, gi, __ldg(p.tokens + gi), L);
        for (int64_t v = threadIdx.x; v < p.V; v += blockDim.x) {
            float x;
            if (sizeof(Tin) == 2) x = __uint_as_float(((uint32_t)reinterpret_cast<const uint16_t *>(row)[v]) << 16);
            else x = reinterpret_cast<const float *>(row)[v];
            const float t2 = fmaf(x, p.c2x, -ri.l2);
            float g = __fmul_rn(ex2(t2), GENT ? fmaf(ri.A1, t2, ri.A0) : ri.A0);  // no contraction: same bits on every path
            if (v == ri.y) g = __fadd_rn(g, ri.wt);
            if (sizeof(Tin) == 2) {
                const uint32_t hb = f32x2_to_bf16x2(g, 0.f) & 0xffffu;
                reinterpret_cast<uint16_t *>(orow)[v] = (uint16_t)hb;
            } else {
                reinterpret_cast<float *>(orow)[v] = g;
            }
        }
    }
}

template <typename Tin>
static cudaError_t launch_k5_typed(const K5Params &p, bool tma, int num_sms, cudaStream_t s) {
    const int64_t rows = (int64_t)p.B * p.T;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.stream = s;
    if (tma) {
        const size_t smem = k5_smem_bytes(p.B);
        const bool gent = p.c2 != 0.0;
        auto kern = p.unaligned ? (gent ? k5_tma_kernel<Tin, true, true> : k5_tma_kernel<Tin, true, false>)
                                : (gent ? k5_tma_kernel<Tin, false, true> : k5_tma_kernel<Tin, false, false>);
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int64_t grid = num_sms;
        if (grid > rows) grid = rows;
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(k5::kThreads);
        cfg.dynamicSmemBytes = smem;
        return cudaLaunchKernelEx(&cfg, kern, p);
    }
    const size_t smem = sizeof(int32_t) * (size_t)((p.cum_global ? 0 : p.B) + 32);
    auto gkern = p.c2 != 0.0 ? k5_generic_kernel<Tin, true> : k5_generic_kernel<Tin, false>;
    cudaError_t e = cudaFuncSetAttribute(gkern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (int64_t)num_sms * 4;
    if (grid > rows) grid = rows;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    return cudaLaunchKernelEx(&cfg, gkern, p);
}

cudaError_t launch_k5(const K5Params &p, bool tma, int num_sms, cudaStream_t s) {
    return p.elt == 2 ? launch_k5_typed<uint16_t>(p, tma, num_sms, s) : launch_k5_typed<float>(p, tma, num_sms, s);
}

}  // namespace orl

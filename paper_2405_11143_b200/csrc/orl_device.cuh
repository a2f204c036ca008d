// orl_device.cuh -- sm_100a device helpers shared by the liborl kernels.
// PTX wrappers (mbarrier, 1-D TMA bulk copy, packed f32x2 math, bf16x2 max),
// the online (max, sum, moment) state of the streaming log-softmax, and the
// per-token KL estimators.  Product code only; nothing here is shared with
// the oracle (oracle/ has its own C implementation).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace orl {

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2 = 0.69314718055994530942;
// Initial running max (log2 units).  Finite so that (m_old - m_new) * s stays
// 0 * finite on the first chunk.  Every real logit scaled by inv_temp*log2e is
// far above it.
constexpr float kMInit = -1.0e38f;
// -inf logits are clamped to this (bf16 0xf149 = -9.95e29) so that
// exp2(t) == 0 AND exp2(t) * t == 0 (instead of 0 * -inf = NaN) in the
// entropy moment.  A whole row at the clamp is reported as non-finite.
constexpr uint32_t kNegClampBf16x2 = 0xf149f149u;
constexpr float kNegClampF32 = -9.953037915854457e29f;
// Rows whose scaled max is below this are "all -inf" rows (input error).
constexpr float kRowDeadLog2 = -1.0e29f;

// ------------------------------------------------------------- packed math
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// max of two bf16 pairs, NaN-propagating (a NaN logit must stay visible)
__device__ __forceinline__ uint32_t hmax2_nan(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float d;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^t for a packed pair on the FMA/ALU pipes (no MUFU): t clamped to
// [-126, 127], Cody-Waite split t = j + f with j = rint(t) (magic-number
// add), degree-5 polynomial for 2^f on [-1/2, 1/2] (max rel. error 2.3e-7 in
// fp32 Horner, ~MUFU.EX2 accuracy), exponent added with one LEA per lane.
// Used for a fixed fraction of the elements to offload the MUFU pipe.
__device__ __forceinline__ uint64_t poly_ex2x2(uint64_t tt) {
    float t0, t1;
    unpack2(tt, t0, t1);
    t0 = fminf(fmaxf(t0, -126.f), 127.f);
    t1 = fminf(fmaxf(t1, -126.f), 127.f);
    const uint64_t tc = pack2(t0, t1);
    const uint64_t mag = pack2(12582912.f, 12582912.f);   // 1.5 * 2^23
    const uint64_t r = fadd2(tc, mag);                     // low mantissa bits = rint(t)
    const uint64_t jf = fadd2(r, pack2(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(jf, pack2(-1.f, -1.f), tc);  // t - j in [-1/2, 1/2]
    uint64_t q = ffma2(pack2(1.3276358e-3f, 1.3276358e-3f), f, pack2(9.6755093e-3f, 9.6755093e-3f));
    q = ffma2(q, f, pack2(5.5507135e-2f, 5.5507135e-2f));
    q = ffma2(q, f, pack2(2.4022120e-1f, 2.4022120e-1f));
    q = ffma2(q, f, pack2(6.9314694e-1f, 6.9314694e-1f));
    q = ffma2(q, f, pack2(1.0000001f, 1.0000001f));
    float q0, q1, r0, r1;
    unpack2(q, q0, q1);
    unpack2(r, r0, r1);
    const uint32_t o0 = __float_as_uint(q0) + (__float_as_uint(r0) << 23);
    const uint32_t o1 = __float_as_uint(q1) + (__float_as_uint(r1) << 23);
    return pack2(__uint_as_float(o0), __uint_as_float(o1));
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// ------------------------------------------------------------- mbarrier / TMA
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t *bar, uint32_t count) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)), "r"(count)
        : "memory");
}
// 1-D bulk copy shared -> global (TMA engine), bulk-group completion.
__device__ __forceinline__ void tma_store_1d(void *gmem_dst, const void *smem_src, uint32_t bytes, uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes), "l"(policy)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .b64 st;\n\t"
        "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
            smem_u32(bar)),
        "r"(bytes)
        : "memory");
}
// Wait until the phase with parity `parity` of `bar` has completed.  The
// suspend-time hint lets the hardware park the warp until the phase flips
// instead of re-polling (fewer issue slots and less power while starved).
#ifndef ORL_MBAR_SUSPEND_NS
#define ORL_MBAR_SUSPEND_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#if ORL_MBAR_SUSPEND_NS > 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(ORL_MBAR_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_unchanged_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D bulk copy global -> shared (TMA engine), completion as tx bytes on `bar`.
__device__ __forceinline__ void tma_load_1d(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                            uint64_t *bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(const void *p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void stg128_cs(void *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
// Streaming store with an explicit L2 eviction policy (e.g. evict_first, so the
// dlogits of the fused actor pass do not push the rows it re-reads out of L2).
__device__ __forceinline__ void stg128_hint(void *p, uint4 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ uint32_t f32x2_to_bf16x2_rn(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ------------------------------------------------------------- online state
// Streaming log-sum-exp + first moment in log2 units:
//   m = running max of x*c (c = inv_temp*log2e),
//   s = sum 2^(x c - m),  u = sum 2^(x c - m) (x c - m).
// Then lse = ln2 (m + log2 s) and H = ln2 (log2 s - u/s).
struct Online {
    float m, s, u;
};

__device__ __forceinline__ Online online_merge(Online a, Online b) {
    float M = fmax_nan(a.m, b.m);
    float da = a.m - M, db = b.m - M;
    float ea = ex2(da), eb = ex2(db);
    Online r;
    r.m = M;
    r.s = a.s * ea + b.s * eb;
    r.u = ea * fmaf(da, a.s, a.u) + eb * fmaf(db, b.s, b.u);
    return r;
}

__device__ __forceinline__ Online warp_merge(Online v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Online o;
        o.m = __shfl_xor_sync(0xffffffffu, v.m, off);
        o.s = __shfl_xor_sync(0xffffffffu, v.s, off);
        o.u = __shfl_xor_sync(0xffffffffu, v.u, off);
        v = online_merge(v, o);
    }
    return v;
}

// ------------------------------------------------------------- KL estimators
// d = logp - logp_ref:  k1 = d, k2 = d^2/2, k3 = exp(-d) - 1 + d
__device__ __forceinline__ double kl_est(double d, int kind) {
    if (kind == 1) return d;
    if (kind == 2) return 0.5 * d * d;
    return exp(-d) - 1.0 + d;
}
__device__ __forceinline__ double kl_grad(double d, int kind) {
    if (kind == 1) return 1.0;
    if (kind == 2) return d;
    return 1.0 - exp(-d);
}

// Element offset of logits row (b, t) of a micro-batch: padded [B,T,V] views use
// (stride_b, stride_t); packed varlen logits (cu_seqlens != NULL, token offsets
// of the rank batch) put row (b,t) at (cu[so+b] - cu[so] + t) * stride_t.
__device__ __forceinline__ int64_t logits_row_offset(const int32_t *cu, int64_t so, int b, int t, int64_t sb,
                                                     int64_t st) {
    return cu ? ((int64_t)(__ldg(cu + so + b) - __ldg(cu + so)) + t) * st : (int64_t)b * sb + (int64_t)t * st;
}

// Valid-row enumeration: the micro-batch's valid rows (t < L_b) in
// (b,t) order, j = 0..N-1.  cum[b] = sum_{b'<=b} L_b' (inclusive).
__device__ __forceinline__ void locate_row(const int32_t *cum, int B, int64_t j, int &b, int &t) {
    int lo = 0, hi = B - 1;
    while (lo < hi) {  // first b with cum[b] > j
        int mid = (lo + hi) >> 1;
        if (cum[mid] > j) hi = mid;
        else lo = mid + 1;
    }
    b = lo;
    t = (int)(j - (lo > 0 ? cum[lo - 1] : 0));
}

}  // namespace orl

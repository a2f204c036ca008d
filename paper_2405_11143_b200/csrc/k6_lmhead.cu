// k6_lmhead.cu -- NEXT-4: the LM-head GEMM fused with the online log-sum-exp.
//
// z[r, v] = sum_k h[r, k] W[v, k] (the actor's LM head) is computed on
// the 5th-generation tensor cores (tcgen05.mma, bf16 x bf16 -> fp32 in TMEM)
// and reduced on the fly to the S1 online state (m, s, u) of each row
// (orl_device.cuh) -- the [R, V] logits never exist in HBM.  Work unit = one
// M-tile of h x one "split" of tiles_per_split 256-column vocab tiles; a unit
// writes one partial (m, s, u, z_y) per row, and K1's merge kernel
// (k1_logprobs.cu, k6_merge_kernel) combines the splits in a fixed order and
// runs the S1/S2/S3 or S7-S9 row epilogue.
//
// Two variants, both persistent (one CTA per SM walking units round-robin,
// split-major so the units in flight share a few L2-resident W tiles):
//   k6_lmhead_2sm_kernel (default): CTA pairs, tcgen05.mma.cta_group::2 with
//       M = 256 (128 rows per CTA), N = 256 split across the pair, 6-stage
//       32 KB/CTA TMA ring;
//   k6_lmhead_kernel (ORL_K6_2SM=0): one CTA, M = 128, N = 256, 4-stage
//       48 KB ring.
// Warp roles (192 threads per CTA):
//   warp 0      TMA producer: 2-D tensor-map loads (SWIZZLE_128B) of the A (h)
//               and B (W) k-blocks;
//   warp 1      TMEM allocator (512 columns = two 256-column fp32 accumulators)
//               and MMA issuer (one thread; the pair leader in the 2-SM kernel):
//               4 UMMAs (K = 16) per 64-wide k-block, tcgen05.commit ->
//               smem-slot release / accumulator ready;
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time from the lane
//               quarter the warp may access, online max/sum/moment in log2
//               units, target gather; the accumulator is released to the MMA
//               warp so tile i+1's MMAs overlap tile i's epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "orl_device.cuh"
#include "orl_internal.h"

namespace orl {
namespace {

constexpr int kBM = 128, kBN = kLmTileN, kBK = 64, kStages = 4, kUmmaK = 16;
constexpr uint32_t kBytesA = kBM * kBK * 2, kBytesB = kBN * kBK * 2, kStageBytes = kBytesA + kBytesB;
constexpr int kThreads6 = 192;
constexpr uint32_t kTmemCols = 2 * kBN;
static_assert(kTmemCols == 512, "two 256-column fp32 accumulators fill TMEM");
static_assert(kStageBytes % 1024 == 0, "SWIZZLE_128B tiles need 1024-byte alignment");

struct K6Bars {
    uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
    uint32_t tmem_base;
};
constexpr size_t kSmem6 = (size_t)kStages * kStageBytes + 1024 + sizeof(K6Bars);

// ----------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int x, int y,
                                            uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor of a K-major SWIZZLE_128B tile (rows of 64
// bf16 = 128 B, 8-row swizzle atoms 1024 B apart): start >> 4, LBO = 1
// (unused for swizzled K-major), SBO = 1024 B >> 4, version 1 (sm_100),
// layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// Instruction descriptor, kind::f16: D fp32 (bit 4), A and B bf16 (bits 7, 10),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, "
        "[%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// mbarrier wait with a suspend-time hint: the warp is parked until the phase
// completes (or the hint expires) instead of spinning -- the epilogue warps
// wait ~30 us per tile for the MMAs, and every issue slot they burn costs
// power the tensor cores need (this kernel runs at the 1 kW cap).
#ifndef ORL_K6_EPI_SLEEP_NS
#define ORL_K6_EPI_SLEEP_NS 20000
#endif
#ifndef ORL_K6_PROD_SLEEP_NS
#define ORL_K6_PROD_SLEEP_NS 0
#endif
template <int NS>
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
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

// Target token of hidden row r (or -1 when r is not a valid (b,t) of the call).
__device__ int row_target(const K6Params &p, int64_t r) {
    int b, t;
    if (p.cu_seqlens) {
        const int32_t *cu = p.cu_seqlens + p.seq_offset;
        const int32_t c0 = __ldg(cu);
        int lo = 0, hi = p.B - 1;  // last b with cu[b] - c0 <= r
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if ((int64_t)(__ldg(cu + mid) - c0) <= r) lo = mid;
            else hi = mid - 1;
        }
        b = lo;
        const int64_t tt = r - (int64_t)(__ldg(cu + b) - c0);
        if (tt < 0 || tt >= p.T) return -1;
        t = (int)tt;
    } else {
        b = (int)(r / p.T);
        t = (int)(r % p.T);
        if (b >= p.B) return -1;
    }
    int L = __ldg(p.lengths + p.seq_offset + b);
    L = L < 0 ? 0 : (L > p.T ? p.T : L);
    if (t >= L) return -1;
    return __ldg(p.tokens + (p.seq_offset + b) * (int64_t)p.T + t);
}

// Work-unit order: groups of `grp` M units (CTA-pair row blocks, or M-tiles in the
// 1-SM kernel) walk every vocab split before the next group starts; inside a group
// the M unit varies fastest, so the units in flight share one or two W splits and
// only the group's rows of h need to stay in L2.
__device__ __forceinline__ uint64_t k6_policy(int which) {
    return which == 1 ? l2_evict_last_policy() : which == 2 ? l2_evict_first_policy() : l2_evict_normal_policy();
}
__device__ __forceinline__ void unit_coords(int u, int m_units, int n_split, int grp, int &m, int &split) {
    const int per_group = grp * n_split;
    const int g = u / per_group;
    const int rem = u - g * per_group;
    const int gm = min(grp, m_units - g * grp);
    split = rem / gm;
    m = g * grp + (rem - split * gm);
}

// Persistent: one CTA per SM walks the work units u = blockIdx.x + k*gridDim.x,
// unit u = (split u / m_tiles, M-tile u % m_tiles).  Consecutive units share the
// vocab split, so the ~148 units in flight at any time touch only a few W
// tiles (L2-resident) while every M-tile of h stays in L2.  The TMA and MMA
// pipelines run across unit boundaries without draining.
__global__ void __launch_bounds__(kThreads6, 1)
    k6_lmhead_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const K6Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    K6Bars *bars = reinterpret_cast<K6Bars *>(sm + kStages * kStageBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = p.m_tiles * p.n_split;
    const int kblocks = (p.d + kBK - 1) / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tfull[a], 1);
            mbar_init(&bars->tempty[a], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tmap(&tmA);
            prefetch_tmap(&tmB);
            const uint64_t pol_a = k6_policy(p.pol_a);  // h: re-read for every vocab tile
            const uint64_t pol_b = k6_policy(p.pol_b);  // W: shared by the concurrent M units
            int stage = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int m_tile, split;
                unit_coords(u, p.m_tiles, p.n_split, p.m_group, m_tile, split);
                const int t_end = min(p.n_tiles, (split + 1) * p.tiles_per_split);
                for (int tile = split * p.tiles_per_split; tile < t_end; ++tile) {
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&bars->empty[stage], phase ^ 1u);
                        uint8_t *sa = sm + stage * kStageBytes;
                        mbar_arrive_expect_tx(&bars->full[stage], kStageBytes);
                        tma_load_2d(sa, &tmA, &bars->full[stage], kb * kBK, m_tile * kBM, pol_a);
                        tma_load_2d(sa + kBytesA, &tmB, &bars->full[stage], kb * kBK, tile * kBN, pol_b);
                        if (++stage == kStages) { stage = 0; phase ^= 1u; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0, i = 0;
            uint32_t phase = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int m_tile_, split;
                unit_coords(u, p.m_tiles, p.n_split, p.m_group, m_tile_, split);
                const int nt = min(p.n_tiles, (split + 1) * p.tiles_per_split) - split * p.tiles_per_split;
                for (int j = 0; j < nt; ++j, ++i) {
                    const int a = i & 1;
                    const uint32_t aphase = (uint32_t)(i >> 1) & 1u;
                    mbar_wait(&bars->tempty[a], aphase ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(a * kBN);
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&bars->full[stage], phase);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(sm + stage * kStageBytes);
                        const uint64_t da = sw128_kmajor_desc(sa), db = sw128_kmajor_desc(sa + kBytesA);
#pragma unroll
                        for (int k = 0; k < kBK / kUmmaK; ++k)  // +32 B along K inside the 128-B swizzle row
                            umma_bf16(d_tmem, da + 2 * k, db + 2 * k, (kb | k) != 0 ? 1u : 0u);
                        umma_commit(&bars->empty[stage]);
                        if (++stage == kStages) { stage = 0; phase ^= 1u; }
                    }
                    umma_commit(&bars->tfull[a]);
                }
            }
        }
    } else {
        // epilogue: warp w may read TMEM lanes 32 (w % 4) .. +31
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const float c2 = p.c2;
        int i = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int m_tile, split;
                unit_coords(u, p.m_tiles, p.n_split, p.m_group, m_tile, split);
            const int t_beg = split * p.tiles_per_split;
            const int nt = min(p.n_tiles, t_beg + p.tiles_per_split) - t_beg;
            const int64_t r = (int64_t)m_tile * kBM + row;
            const int y = r < p.R ? row_target(p, r) : -1;
            float m = kMInit, s = 0.f, uu = 0.f, tgt = __int_as_float(0x7fc00000);
            for (int j = 0; j < nt; ++j, ++i) {
                const int a = i & 1;
                const uint32_t aphase = (uint32_t)(i >> 1) & 1u;
                mbar_wait(&bars->tfull[a], aphase);
                tc_fence_after();
                const int n0 = (t_beg + j) * kBN;
#pragma unroll 1
                for (int c = 0; c < kBN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * kBN + c * 32), v);
                    const int col0 = n0 + c * 32;
                    const int nvalid = p.V - col0;  // columns >= V are TMA zero-fill: excluded
                    if ((unsigned)(y - col0) < 32u) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (jj == y - col0) tgt = __uint_as_float(v[jj]);
                    }
                    if (nvalid <= 0) continue;
                    float x[32];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj)
                        x[jj] = jj < nvalid ? __uint_as_float(v[jj]) : kNegClampF32;
                    float cm0 = x[0], cm1 = x[1];
#pragma unroll
                    for (int jj = 2; jj < 32; jj += 2) {
                        cm0 = fmax_nan(cm0, x[jj]);
                        cm1 = fmax_nan(cm1, x[jj + 1]);
                    }
                    const float mn = fmax_nan(m, fmax_nan(cm0, cm1) * c2);
                    const float dm = m - mn, rs = ex2(dm);
                    uu = rs * fmaf(dm, s, uu);
                    s = rs * s;
                    m = mn;
                    float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 32; jj += 2) {
                        const float t0 = fmaf(x[jj], c2, -m), t1 = fmaf(x[jj + 1], c2, -m);
                        const float e0 = ex2(t0), e1 = ex2(t1);
                        s0 += e0;
                        s1 += e1;
                        u0 = fmaf(e0, t0, u0);
                        u1 = fmaf(e1, t1, u1);
                    }
                    s += s0 + s1;
                    uu += u0 + u1;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->tempty[a]);
            }
            if (r < p.R) p.parts[(int64_t)split * p.part_stride + r] = make_float4(m, s, uu, tgt);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

// ------------------------------------------------------------------ 2-SM variant
// A CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile per UMMA
// (tcgen05.mma.cta_group::2, M = 256): CTA r holds rows 128 r .. of the A tile
// and rows 128 r .. of the B tile (the N split of the 2-SM MMA), so each SM
// streams 32 KB per k-block instead of 48 KB for the same MACs (B is no longer
// duplicated), and the pipeline can be 6 stages deep.  Only the leader (rank 0)
// issues MMAs; both CTAs' TMA loads complete on the leader's full barrier, the
// leader's commits arrive on both CTAs' empty / tmem-full barriers (multicast),
// and both CTAs' epilogues arrive on the leader's tmem-empty barrier.
constexpr int kStages2 = 6;
constexpr uint32_t kBytesA2 = kBM * kBK * 2, kBytesB2 = (kBN / 2) * kBK * 2, kStageBytes2 = kBytesA2 + kBytesB2;
static_assert(kStageBytes2 % 1024 == 0, "SWIZZLE_128B tiles need 1024-byte alignment");
struct K6Bars2 {
    uint64_t full[kStages2], empty[kStages2], tfull[2], tempty[2];
    uint32_t tmem_base;
};
constexpr size_t kSmem62 = (size_t)kStages2 * kStageBytes2 + 1024 + sizeof(K6Bars2);
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                             ((uint32_t)((2 * kBM) >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void *dst, const CUtensorMap *map, uint32_t bar_cluster, int x, int y,
                                                uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc2), "r"(accumulate)
        : "memory");
}
// commit the leader's MMAs to the barrier at this offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_2sm(uint64_t *bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __launch_bounds__(kThreads6, 1)
    k6_lmhead_2sm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const K6Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    K6Bars2 *bars = reinterpret_cast<K6Bars2 *>(sm + kStages2 * kStageBytes2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int m_pairs = (p.m_tiles + 1) >> 1;
    const int units = m_pairs * p.n_split;
    const int kblocks = (p.d + kBK - 1) / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tfull[a], 1);
            mbar_init(&bars->tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&bars->tmem_base)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync_all();
    __syncthreads();  // CTA-scope order for the tmem_base read (racecheck does not model the cluster barrier)
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            prefetch_tmap(&tmA);
            prefetch_tmap(&tmB);
            const uint64_t pol_a = k6_policy(p.pol_a);
            const uint64_t pol_b = k6_policy(p.pol_b);
            int stage = 0;
            uint32_t phase = 0;
            for (int u = cluster; u < units; u += nclusters) {
                int pm, split;
                unit_coords(u, m_pairs, p.n_split, p.m_group, pm, split);
                const int a_row = pm * 2 * kBM + (int)rank * kBM;
                const int t_end = min(p.n_tiles, (split + 1) * p.tiles_per_split);
                for (int tile = split * p.tiles_per_split; tile < t_end; ++tile) {
                    const int b_row = tile * kBN + (int)rank * (kBN / 2);
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait_sleep<ORL_K6_PROD_SLEEP_NS>(&bars->empty[stage], phase ^ 1u);
                        uint8_t *sa = sm + stage * kStageBytes2;
                        const uint32_t fb = map_to_rank(&bars->full[stage], 0);
                        if (leader) mbar_arrive_expect_tx(&bars->full[stage], 2 * kStageBytes2);
                        tma_load_2d_2sm(sa, &tmA, fb, kb * kBK, a_row, pol_a);
                        tma_load_2d_2sm(sa + kBytesA2, &tmB, fb, kb * kBK, b_row, pol_b);
                        if (++stage == kStages2) { stage = 0; phase ^= 1u; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            int stage = 0, i = 0;
            uint32_t phase = 0;
            for (int u = cluster; u < units; u += nclusters) {
                int pm_, split;
                unit_coords(u, m_pairs, p.n_split, p.m_group, pm_, split);
                const int nt = min(p.n_tiles, (split + 1) * p.tiles_per_split) - split * p.tiles_per_split;
                for (int j = 0; j < nt; ++j, ++i) {
                    const int a = i & 1;
                    const uint32_t aphase = (uint32_t)(i >> 1) & 1u;
                    mbar_wait(&bars->tempty[a], aphase ^ 1u);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(a * kBN);
                    for (int kb = 0; kb < kblocks; ++kb) {
                        mbar_wait(&bars->full[stage], phase);
                        tc_fence_after();
                        const uint32_t sa = smem_u32(sm + stage * kStageBytes2);
                        const uint64_t da = sw128_kmajor_desc(sa), db = sw128_kmajor_desc(sa + kBytesA2);
#pragma unroll
                        for (int k = 0; k < kBK / kUmmaK; ++k)
                            umma_bf16_2sm(d_tmem, da + 2 * k, db + 2 * k, (kb | k) != 0 ? 1u : 0u);
                        umma_commit_2sm(&bars->empty[stage]);
                        if (++stage == kStages2) { stage = 0; phase ^= 1u; }
                    }
                    umma_commit_2sm(&bars->tfull[a]);
                }
            }
        }
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;
        const float c2 = p.c2;
        const uint32_t tempty0 = map_to_rank(&bars->tempty[0], 0), tempty1 = map_to_rank(&bars->tempty[1], 0);
        int i = 0;
        for (int u = cluster; u < units; u += nclusters) {
            int pm, split;
                unit_coords(u, m_pairs, p.n_split, p.m_group, pm, split);
            const int t_beg = split * p.tiles_per_split;
            const int nt = min(p.n_tiles, t_beg + p.tiles_per_split) - t_beg;
            const int64_t r = (int64_t)pm * 2 * kBM + (int64_t)rank * kBM + row;
            const int y = r < p.R ? row_target(p, r) : -1;
            float m = kMInit, s = 0.f, uu = 0.f, tgt = __int_as_float(0x7fc00000);
            for (int j = 0; j < nt; ++j, ++i) {
                const int a = i & 1;
                const uint32_t aphase = (uint32_t)(i >> 1) & 1u;
                mbar_wait_sleep<ORL_K6_EPI_SLEEP_NS>(&bars->tfull[a], aphase);
                tc_fence_after();
                const int n0 = (t_beg + j) * kBN;
#pragma unroll 1
                for (int c = 0; c < kBN / 32; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(a * kBN + c * 32), v);
                    const int col0 = n0 + c * 32;
                    const int nvalid = p.V - col0;
                    if ((unsigned)(y - col0) < 32u) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            if (jj == y - col0) tgt = __uint_as_float(v[jj]);
                    }
                    if (nvalid <= 0) continue;
#ifdef ORL_K6_EPI_NOMATH  // diagnosis only: skip the online LSE math (wrong results)
                    if (v[0] != 0x7fc00001u) { s += __uint_as_float(v[1]); continue; }
#endif
                    float x[32];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj)
                        x[jj] = jj < nvalid ? __uint_as_float(v[jj]) : kNegClampF32;
                    float cm0 = x[0], cm1 = x[1];
#pragma unroll
                    for (int jj = 2; jj < 32; jj += 2) {
                        cm0 = fmax_nan(cm0, x[jj]);
                        cm1 = fmax_nan(cm1, x[jj + 1]);
                    }
                    const float mn = fmax_nan(m, fmax_nan(cm0, cm1) * c2);
                    const float dm = m - mn, rs = ex2(dm);
                    uu = rs * fmaf(dm, s, uu);
                    s = rs * s;
                    m = mn;
                    float s0 = 0.f, s1 = 0.f, u0 = 0.f, u1 = 0.f;
#pragma unroll
                    for (int jj = 0; jj < 32; jj += 2) {
                        const float t0 = fmaf(x[jj], c2, -m), t1 = fmaf(x[jj + 1], c2, -m);
                        const float e0 = ex2(t0), e1 = ex2(t1);
                        s0 += e0;
                        s1 += e1;
                        u0 = fmaf(e0, t0, u0);
                        u1 = fmaf(e1, t1, u1);
                    }
                    s += s0 + s1;
                    uu += u0 + u1;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(a ? tempty1 : tempty0);
            }
            if (r < p.R) p.parts[(int64_t)split * p.part_stride + r] = make_float4(m, s, uu, tgt);
        }
    }
    __syncwarp();        // reconverge the role warps before the .aligned cluster barrier
    tc_fence_before();
    cluster_sync_all();  // no CTA leaves while its peer may still touch its smem / barriers
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

bool make_map(CUtensorMap *m, const void *base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

void k6_plan(K6Params &p, int num_sms) {
    p.m_tiles = (int)((p.R + kBM - 1) / kBM);
    p.n_tiles = (int)((p.V + kBN - 1) / kBN);
    p.two_sm = 1;
    if (const char *e = getenv("ORL_K6_2SM")) p.two_sm = atoi(e) != 0;
    int tps = 4;  // vocab tiles per unit: small units balance the persistent CTAs
    if (const char *e = getenv("ORL_K6_TPS")) tps = atoi(e);
    if (tps < 1) tps = 1;
    if (tps > p.n_tiles) tps = p.n_tiles;
    p.tiles_per_split = tps;
    p.n_split = (p.n_tiles + tps - 1) / tps;
    const int m_units = p.two_sm ? (p.m_tiles + 1) / 2 : p.m_tiles;
    p.m_group = m_units;  // default: one group (every row block in flight)
    if (const char *e = getenv("ORL_K6_MGROUP")) p.m_group = atoi(e);
    if (p.m_group < 1 || p.m_group > m_units) p.m_group = m_units;
    p.pol_a = 1;  // h evict_last: re-read for every vocab tile of every split
    p.pol_b = 2;  // W evict_first: a split's tiles are used by the in-flight row blocks at once, then never
                  // again -- keeping them out of the way of h cuts DRAM re-reads (-4 % time sustained)
    if (const char *e = getenv("ORL_K6_POLA")) p.pol_a = atoi(e);
    if (const char *e = getenv("ORL_K6_POLB")) p.pol_b = atoi(e);
    if (p.two_sm) {
        const int64_t units = (int64_t)((p.m_tiles + 1) / 2) * p.n_split;
        p.grid = 2 * (int)std::min<int64_t>(units, num_sms / 2);
    } else {
        p.grid = (int)std::min<int64_t>((int64_t)p.m_tiles * p.n_split, num_sms);
    }
}

cudaError_t launch_k6(const K6Params &p, const void *hidden, int64_t ld_hidden, const void *weight,
                      int64_t ld_weight, cudaStream_t s) {
    CUtensorMap ma, mb;
    const int b_rows = p.two_sm ? kBN / 2 : kBN;
    if (!make_map(&ma, hidden, p.R, p.d, ld_hidden, kBM) || !make_map(&mb, weight, p.V, p.d, ld_weight, b_rows))
        return cudaErrorInvalidValue;
    if (p.grid < 1) return cudaErrorInvalidConfiguration;
    if (!p.two_sm) {
        cudaError_t e = cudaFuncSetAttribute(k6_lmhead_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem6);
        if (e != cudaSuccess) return e;
        k6_lmhead_kernel<<<(unsigned)p.grid, kThreads6, kSmem6, s>>>(ma, mb, p);
        return cudaGetLastError();
    }
    cudaError_t e = cudaFuncSetAttribute(k6_lmhead_2sm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem62);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.grid);
    cfg.blockDim = dim3(kThreads6);
    cfg.dynamicSmemBytes = kSmem62;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k6_lmhead_2sm_kernel, ma, mb, p);
}

}  // namespace orl

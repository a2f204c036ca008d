// k3_advantages.cu -- K3/K4: advantages over the rank-local batch.
//
//   GAE:  delta_t = r'_t + gamma V_{t+1} [t+1 < L] - V_t
//                 A_t = delta_t + gamma lambda A_{t+1},  A_{L} = 0,  R_t = A_t + V_t
//   REINFORCE++ (north star, Z23):  G_t = r'_t + gamma G_{t+1}
//   RPP-baseline: same with R_b - mu_g at t = L_b - 1
//   GRPO: A_b = (R_b - mu_g)/(sigma_g + 1e-8), constant group -> 0
//
// One CTA (256 threads) per response.  The backward recursion is an affine
// map per token (x -> delta_t + c x); each thread composes the maps of a
// contiguous chunk in fp64, a block-wide suffix scan of the chunk maps gives
// every chunk its carry-in, and a second pass writes A and R (fp32) from the
// fp64 carry.  Depth O(T/256 + log 256) instead of O(T), fp64 carry as the
// 1e-5 bar at T=8192, gamma=lambda=1 requires.
// The CTA also forms the fp64 whitening partial (n_b, mean_b, M2_b) of the
// stored fp32 advantages (two-pass within the response).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "orl_internal.h"

namespace orl {

constexpr int kK3Threads = 256;

__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < kK3Threads / 32; ++q) s += sh[q];  // fixed order
    return s;
}

__global__ void __launch_bounds__(kK3Threads) k3_kernel(const K3Params p) {
    __shared__ double sh_m[kK3Threads], sh_b[kK3Threads];
    __shared__ double sh_red[kK3Threads / 32];
    __shared__ double sh_seq[2];
    const int b = blockIdx.x, tid = threadIdx.x;
    int L = p.lengths[b];
    if (L < 0 || L > p.T) {
        if (tid == 0) atomicAdd(&p.err[2], 1ull);
        L = L < 0 ? 0 : p.T;
    }
    const int64_t row = (int64_t)b * p.T;
    const bool grpo = p.kind == 1;
    const bool gae = p.kind == 0;
    const bool base = p.kind == 3;

    // ---- group statistics (GRPO, RPP-baseline), fp64, thread 0 -------------
    if (tid == 0 && (grpo || base)) {
        const int g0 = (b / p.G) * p.G;
        double mx = p.seq_reward[g0], mn = mx, sum = 0.0;
        for (int j = 0; j < p.G; ++j) {
            const double r = p.seq_reward[g0 + j];
            mx = fmax(mx, r);
            mn = fmin(mn, r);
            sum += r;
        }
        const double mu = sum / (double)p.G;
        double ss = 0.0;
        for (int j = 0; j < p.G; ++j) {
            const double r = (double)p.seq_reward[g0 + j] - mu;
            ss += r * r;
        }
        const double sigma = sqrt(ss / (double)p.G);
        const double Rb = p.seq_reward[b];
        sh_seq[0] = grpo ? ((mx == mn) ? 0.0 : (Rb - mu) / (sigma + 1e-8)) : mu;
        if (p.keep && b == g0) p.keep[b / p.G] = (mx - mn >= 1e-12) ? 1 : 0;
    }
    __syncthreads();

    if (grpo) {
        const float a = (float)sh_seq[0];
        const float alo = p.adv_lo ? (float)(sh_seq[0] - (double)a) : 0.f;
        for (int t = tid; t < p.T; t += kK3Threads) {
            const float v = t < L ? a : 0.f;
            p.adv[row + t] = v;
            if (p.adv_lo) p.adv_lo[row + t] = t < L ? alo : 0.f;
            if (p.ret) p.ret[row + t] = v;
        }
        if (tid == 0) {
            double *o = p.seq_part + 3 * (int64_t)b;
            o[0] = (double)L;
            o[1] = L > 0 ? (double)a + (double)alo : 0.0;
            o[2] = 0.0;
        }
        return;
    }

    const double c = gae ? p.gamma * p.lambda : p.gamma;
    const double mu_g = base ? sh_seq[0] : 0.0;
    // delta_t in fp64 from the fp32 inputs
    auto delta = [&](int t) -> double {
        double d = (double)p.shaped[row + t];
        if (base && t == L - 1) d -= mu_g;
        if (gae) {
            const double vn = (t + 1 < L) ? (double)p.values[row + t + 1] : 0.0;
            d += p.gamma * vn - (double)p.values[row + t];
        }
        return d;
    };
    const int per = (L + kK3Threads - 1) / kK3Threads;
    const int beg = min(L, tid * per), end = min(L, beg + per);

    // pass 1: chunk map x -> M x + Bc over tokens [beg, end)
    double M = 1.0, Bc = 0.0;
    for (int t = end - 1; t >= beg; --t) {
        Bc = delta(t) + c * Bc;
        M *= c;
    }
    // suffix composition F_k = f_k o f_{k+1} o ... (inclusive), fixed shape
    sh_m[tid] = M;
    sh_b[tid] = Bc;
    __syncthreads();
    for (int off = 1; off < kK3Threads; off <<= 1) {
        double m2 = 1.0, b2 = 0.0;
        if (tid + off < kK3Threads) { m2 = sh_m[tid + off]; b2 = sh_b[tid + off]; }
        __syncthreads();
        // (M, Bc) o (m2, b2): x -> Bc + M (b2 + m2 x)
        Bc = Bc + M * b2;
        M = M * m2;
        sh_m[tid] = M;
        sh_b[tid] = Bc;
        __syncthreads();
    }
    const double carry = (tid + 1 < kK3Threads) ? sh_b[tid + 1] : 0.0;  // A at t = end

    // pass 2: write A (fp32, plus the fp32 residual when adv_lo is given), R; local sum
    // of the stored advantages (the values the actor pass will whiten)
    double A = carry, lsum = 0.0;
    for (int t = end - 1; t >= beg; --t) {
        A = delta(t) + c * A;
        const float af = (float)A;
        p.adv[row + t] = af;
        double As = (double)af;
        if (p.adv_lo) {
            const float lo = (float)(A - (double)af);
            p.adv_lo[row + t] = lo;
            As += (double)lo;
        }
        if (p.ret) p.ret[row + t] = gae ? (float)(A + (double)p.values[row + t]) : af;
        lsum += As;
    }
    for (int t = L + tid; t < p.T; t += kK3Threads) {
        p.adv[row + t] = 0.f;
        if (p.adv_lo) p.adv_lo[row + t] = 0.f;
        if (p.ret) p.ret[row + t] = 0.f;
    }
    // whitening partial of this response: n, mean, M2 (two-pass, fp64)
    const double S = block_sum(lsum, sh_red);
    const double mean = L > 0 ? S / (double)L : 0.0;
    double lss = 0.0;
    for (int t = beg; t < end; ++t) {
        const double d = (double)p.adv[row + t] + (p.adv_lo ? (double)p.adv_lo[row + t] : 0.0) - mean;  // own writes
        lss += d * d;
    }
    const double M2 = block_sum(lss, sh_red);
    if (tid == 0) {
        double *o = p.seq_part + 3 * (int64_t)b;
        o[0] = (double)L;
        o[1] = mean;
        o[2] = M2;
    }
}

cudaError_t launch_k3(const K3Params &p, cudaStream_t s) {
    k3_kernel<<<p.B, kK3Threads, 0, s>>>(p);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- whitening
// Chan et al. pairwise merge of (n, mean, M2); fixed order -> deterministic.
__device__ __forceinline__ void chan_merge(double &n, double &mean, double &M2, double nb,
                                           double meanb, double M2b) {
    if (nb <= 0.0) return;
    if (n <= 0.0) { n = nb; mean = meanb; M2 = M2b; return; }
    const double nt = n + nb;
    const double d = meanb - mean;
    mean = mean + d * (nb / nt);
    M2 = M2 + M2b + d * d * (n * nb / nt);
    n = nt;
}

// Rank-local whitening partial (n, mean, M2, sequences with L_b > 0) of the
// per-sequence partials, 256 threads; thread 0 returns it in out[0..3].
__device__ void whiten_local_block(const double *seq_part, int B, double *out) {
    __shared__ double sn[256], sm[256], s2[256], sc[256];
    const int tid = threadIdx.x;
    const int per = (B + 255) / 256;
    const int beg = min(B, tid * per), end = min(B, beg + per);
    double n = 0.0, mean = 0.0, M2 = 0.0, nseq = 0.0;
    for (int q = beg; q < end; ++q) {
        chan_merge(n, mean, M2, seq_part[3 * q], seq_part[3 * q + 1], seq_part[3 * q + 2]);
        nseq += seq_part[3 * q] > 0.0 ? 1.0 : 0.0;
    }
    sn[tid] = n; sm[tid] = mean; s2[tid] = M2; sc[tid] = nseq;
    __syncthreads();
    // fixed-shape pairwise tree (deterministic, log depth): slot i absorbs i + h
    for (int h = 128; h >= 1; h >>= 1) {
        if (tid < h) {
            double a = sn[tid], am = sm[tid], a2 = s2[tid];
            chan_merge(a, am, a2, sn[tid + h], sm[tid + h], s2[tid + h]);
            sn[tid] = a; sm[tid] = am; s2[tid] = a2;
            sc[tid] += sc[tid + h];
        }
        __syncthreads();
    }
    if (tid == 0) {
        out[0] = sn[0]; out[1] = sm[0]; out[2] = s2[0];
        out[3] = sc[0];   // sequences with L_b > 0
    }
}

__global__ void whiten_local_kernel(const double *seq_part, int B, double *slot) {
    whiten_local_block(seq_part, B, slot);
}

cudaError_t launch_whiten_local(const double *seq_part, int B, double *gather_slot, cudaStream_t s) {
    whiten_local_kernel<<<1, 256, 0, s>>>(seq_part, B, gather_slot);
    return cudaGetLastError();
}

// Rank-ordered Chan merge of the gathered [world][4] partials (one thread).
__device__ void whiten_merge_body(const double *gather, int world, int want, double *whiten, double *flags) {
    double N = 0.0, mu = 0.0, M2 = 0.0, S = 0.0;
    for (int r = 0; r < world; ++r) {
        chan_merge(N, mu, M2, gather[4 * r], gather[4 * r + 1], gather[4 * r + 2]);
        S += gather[4 * r + 3];
    }
    const bool apply = want && N >= 2.0;
    whiten[0] = N;
    whiten[1] = apply ? mu : 0.0;
    whiten[2] = apply ? sqrt(M2 / N) : 0.0;
    whiten[3] = apply ? 1.0 : 0.0;
    whiten[4] = S;
    flags[0] = (want && N < 2.0) ? 1.0 : 0.0;
}

__global__ void whiten_merge_kernel(const double *gather, int world, int want, double *whiten,
                                    double *flags) {
    whiten_merge_body(gather, world, want, whiten, flags);
}

cudaError_t launch_whiten_merge(const double *gather, int world, int want_whiten, double *whiten,
                                double *flags, cudaStream_t s) {
    whiten_merge_kernel<<<1, 1, 0, s>>>(gather, world, want_whiten, whiten, flags);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- statistics
__device__ __forceinline__ double stats_pack_value(const double *acc, const unsigned long long *err, int k) {
    return k < kNumPartials ? acc[k] : (k >= 16 && k < 16 + kNumErr) ? (double)err[k - 16] : 0.0;
}

__global__ void stats_pack_kernel(const double *acc, const unsigned long long *err, double *out) {
    const int k = threadIdx.x;
    if (k < kStatsSlots) out[k] = stats_pack_value(acc, err, k);
}

cudaError_t launch_stats_pack(const double *acc, const unsigned long long *err, double *out,
                              cudaStream_t s) {
    stats_pack_kernel<<<1, 32, 0, s>>>(acc, err, out);
    return cudaGetLastError();
}

// S10: rank-ordered sum of the gathered partials, then the means.
// loss_agg = 1 (NEXT-2, Z31): policy/value/entropy/kl are means over the N_seq
// sequences of per-sequence token means; shares and ratio stay token means.
__device__ void stats_final_body(const double *gather, int world, const double *whiten,
                                 double *flags, double c1, double c2, double beta_loss,
                                 int kl_in_loss, int loss_agg, double *st) {
    double t[kStatsSlots];
    for (int k = 0; k < kStatsSlots; ++k) t[k] = 0.0;
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < kStatsSlots; ++k) t[k] += gather[kStatsSlots * r + k];
    const double N = t[0], S = whiten[4];
    const bool ok = N > 0.0;
    const bool sm = loss_agg == 1 && S > 0.0;
    st[0] = N;
    st[1] = !ok ? 0.0 : sm ? -t[11] / S : -t[1] / N;
    st[2] = !ok ? 0.0 : sm ? t[12] / S : t[2] / N;
    st[3] = !ok ? 0.0 : sm ? t[13] / S : t[3] / N;
    st[4] = !ok ? 0.0 : sm ? t[14] / S : t[4] / N;
    st[5] = ok ? t[7] / N : 0.0;
    st[6] = ok ? t[5] / N : 0.0;
    st[7] = ok ? t[6] / N : 0.0;
    st[8] = ok ? t[8] / N : 0.0;
    st[9] = st[1] + c1 * st[2] - c2 * st[3] + (kl_in_loss ? beta_loss * st[4] : 0.0);
    st[10] = whiten[1];
    st[11] = whiten[2];
    st[12] = t[9];
    st[13] = t[10] + t[17];
    st[14] = t[16];
    st[15] = flags[0];
    flags[1] = t[18] + t[19];  // invalid lengths + non-prefix mask rows (ORL_E_MASK)
    flags[3] = t[20];          // LM-head rows missing from the hidden matrix (ORL_E_SHAPE)
}

__global__ void stats_final_kernel(const double *gather, int world, const double *whiten,
                                   double *flags, double c1, double c2, double beta_loss,
                                   int kl_in_loss, int loss_agg, double *st) {
    stats_final_body(gather, world, whiten, flags, c1, c2, beta_loss, kl_in_loss, loss_agg, st);
}

cudaError_t launch_stats_final(const double *gather, int world, const double *whiten,
                               const double *flags, double c1, double c2, double beta_loss,
                               int kl_in_loss, int loss_agg, double *stats_out, cudaStream_t s) {
    stats_final_kernel<<<1, 1, 0, s>>>(gather, world, whiten, const_cast<double *>(flags), c1, c2,
                                       beta_loss, kl_in_loss, loss_agg, stats_out);
    return cudaGetLastError();
}

// ------------------------------------------------- C1 / C2 over peer memory
// Each collective is ONE kernel: the rank's partial is formed (S6: Chan merge of
// the per-sequence moments; S10: the packed loss accumulators), stored into slot
// [parity][rank] of every rank's exchange buffer over NVLink (plain 64-bit
// stores to peer memory), published with a release store of the epoch into the
// peer's flag [parity][rank]; the kernel then waits (acquire loads of its own
// flags) until every rank's epoch has arrived and merges the slots in rank order
// with the same code as the NCCL path -- every rank computes bit-identical
// results.  Slots alternate by epoch parity: a rank can only write epoch e + 2
// after all ranks published e + 1, i.e. after they finished reading epoch e.
static_assert(kXS - kXW == 2 * kPeerMax * 4 && kXFW - kXS == 2 * kPeerMax * kStatsSlots, "exchange layout");

__device__ __forceinline__ void st_relaxed_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Thread-0 exchange: push `n` words of `mine` to slot (par, rank) of every rank,
// publish, wait for every rank, copy the world x n gathered words into `gath`
// (rank-major).  Returns false on timeout (the missing slots read as NaN).
__device__ bool peer_exchange(const PeerArgs &pa, int data_off, int flag_off, int n, const double *mine,
                              double *gath) {
    const unsigned long long epoch = *pa.epoch + 1ull;  // same sequence on every rank
    const int par = (int)(epoch & 1ull);
    const int slot = data_off + par * kPeerMax * n;
    for (int r = 0; r < pa.world; ++r)
        for (int k = 0; k < n; ++k)
            st_relaxed_sys(pa.x[r] + slot + pa.rank * n + k, (unsigned long long)__double_as_longlong(mine[k]));
    __threadfence_system();
    for (int r = 0; r < pa.world; ++r) st_release_sys(pa.x[r] + flag_off + par * kPeerMax + pa.rank, epoch);
    bool ok = true;
    const unsigned long long *own = pa.x[pa.rank];
    for (int r = 0; r < pa.world; ++r) {
        long long spins = 0;
        bool arrived = true;
        while (ld_acquire_sys(own + flag_off + par * kPeerMax + r) != epoch) {
            if (++spins > pa.spin_limit) { arrived = false; break; }
            __nanosleep(256);
        }
        ok = ok && arrived;
        for (int k = 0; k < n; ++k)
            gath[r * n + k] = arrived ? __longlong_as_double((long long)ld_relaxed_sys(own + slot + r * n + k))
                                      : __longlong_as_double(0x7ff8000000000000ll);
    }
    *pa.epoch = epoch;
    return ok;
}

__global__ void whiten_peer_kernel(const double *seq_part, int B, const PeerArgs pa, int want, double *whiten,
                                   double *flags) {
    __shared__ double mine[4];
    __shared__ double gath[kPeerMax * 4];
    whiten_local_block(seq_part, B, mine);
    if (threadIdx.x == 0) {
        const bool ok = peer_exchange(pa, kXW, kXFW, 4, mine, gath);
        whiten_merge_body(gath, pa.world, want, whiten, flags);
        if (!ok) flags[2] += 1.0;
    }
}

cudaError_t launch_whiten_peer(const double *seq_part, int B, const PeerArgs &pa, int want, double *whiten,
                               double *flags, cudaStream_t s) {
    whiten_peer_kernel<<<1, 256, 0, s>>>(seq_part, B, pa, want, whiten, flags);
    return cudaGetLastError();
}

__global__ void stats_peer_kernel(const double *acc, const unsigned long long *err, const PeerArgs pa,
                                  const double *whiten, double *flags, double c1, double c2, double beta_loss,
                                  int kl_in_loss, int loss_agg, double *st) {
    __shared__ double mine[kStatsSlots];
    __shared__ double gath[kPeerMax * kStatsSlots];
    if (threadIdx.x < kStatsSlots) mine[threadIdx.x] = stats_pack_value(acc, err, threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool ok = peer_exchange(pa, kXS, kXFS, kStatsSlots, mine, gath);
        stats_final_body(gath, pa.world, whiten, flags, c1, c2, beta_loss, kl_in_loss, loss_agg, st);
        if (!ok) flags[2] += 1.0;
    }
}

cudaError_t launch_stats_peer(const double *acc, const unsigned long long *err, const PeerArgs &pa,
                              const double *whiten, double *flags, double c1, double c2, double beta_loss,
                              int kl_in_loss, int loss_agg, double *stats_out, cudaStream_t s) {
    stats_peer_kernel<<<1, 32, 0, s>>>(acc, err, pa, whiten, flags, c1, c2, beta_loss, kl_in_loss, loss_agg,
                                       stats_out);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ masks -> lengths
// Z10: the path's masks are right-padded prefixes.  One CTA per row: L_b = index of the
// first 0 (T if none); a 1 after that is a non-prefix mask, counted in err[3] (reported
// by orl_finalize as ORL_E_MASK) -- the row then keeps its leading prefix.
__global__ void __launch_bounds__(256) mask_lengths_kernel(const uint8_t *mask, int64_t T, int32_t *lengths,
                                                           unsigned long long *err) {
    __shared__ int first_zero, last_one;
    const int64_t b = blockIdx.x;
    if (threadIdx.x == 0) {
        first_zero = (int)T;
        last_one = -1;
    }
    __syncthreads();
    const uint8_t *row = mask + b * T;
    int fz = (int)T, lo = -1;
    for (int64_t t = threadIdx.x; t < T; t += blockDim.x) {
        if (row[t]) lo = (int)t;
        else if (fz == (int)T) fz = (int)t;
    }
    if (fz < (int)T) atomicMin(&first_zero, fz);
    if (lo >= 0) atomicMax(&last_one, lo);
    __syncthreads();
    if (threadIdx.x == 0) {
        lengths[b] = first_zero;
        if (last_one > first_zero && err) atomicAdd(&err[3], 1ull);
    }
}

cudaError_t launch_mask_lengths(const uint8_t *mask, int64_t B, int64_t T, int32_t *lengths,
                                unsigned long long *err, cudaStream_t s) {
    if (B <= 0) return cudaSuccess;
    mask_lengths_kernel<<<(unsigned)B, 256, 0, s>>>(mask, T, lengths, err);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ DAPO re-roll list
// NEXT-2: the indices of the kept groups in increasing order and their count,
// one CTA, fixed-order block scan (deterministic); the caller re-samples the rest.
__global__ void __launch_bounds__(1024) keep_compact_kernel(const uint8_t *keep, int64_t n, int32_t *idx,
                                                            int32_t *count) {
    __shared__ int32_t warp_tot[32];
    __shared__ int32_t base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) base = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const int64_t g = c0 + tid;
        const int k = (g < n && keep[g]) ? 1 : 0;
        int incl = k;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const int v = warp_tot[w];
                warp_tot[w] = run;
                run += v;
            }
        }
        __syncthreads();
        if (k) idx[base + warp_tot[warp] + incl - 1] = (int32_t)g;
        __syncthreads();
        if (tid == blockDim.x - 1) base += warp_tot[warp] + incl;
        __syncthreads();
    }
    if (tid == 0) *count = base;
}

cudaError_t launch_keep_compact(const uint8_t *keep, int64_t n, int32_t *idx, int32_t *count, cudaStream_t s) {
    keep_compact_kernel<<<1, 1024, 0, s>>>(keep, n, idx, count);
    return cudaGetLastError();
}

}  // namespace orl

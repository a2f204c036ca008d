// power_path.cu -- does K1's load path cost power?  The same streaming math as K1's
// logprob pass (per bf16 pair: unpack, FFMA2, 2 x MUFU.EX2, FADD2 into packed sums) over
// an 8.4 GB buffer, fed (a) by a 1-D TMA bulk-copy ring into shared memory + ld.shared
// (K1's path: 1 producer + 16 consumer warps, 6 x 32 KB stages) or (b) by direct
// ld.global.v4 into registers with the next iteration's loads issued before the current
// math (16 warps per SM).  Cool (first launches) and power-capped (after a warm-up,
// blocks of launches alternated) times per launch; the power cap is what the bench sees.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o power_path tools/power_path.cu && ./power_path
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
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
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// K1's per-word body: one bf16 pair -> sum of 2^(x c - m)
__device__ __forceinline__ void body(uint32_t w, uint64_t c2p, uint64_t nm, uint64_t &s) {
    uint64_t x;
    asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\tmov.b64 %0, {lo, hi};\n\t}"
        : "=l"(x) : "r"(w));
    const uint64_t t = ffma2(x, c2p, nm);
    float t0, t1;
    unpack2(t, t0, t1);
    s = fadd2(s, pack2(ex2(t0), ex2(t1)));
}

constexpr int kChunk = 32768, kStages = 6, kCW = 16;

__global__ void __launch_bounds__((kCW + 1) * 32, 1) tma_math(const char *base, size_t bytes, float *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + kStages * kChunk);
    uint64_t *empty = full + kStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(kCW * 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t nch = bytes / kChunk;
    if (warp == kCW) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int stage = 0;
            uint32_t phase = 0;
            for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                             ::"r"(smem_u32(&empty[stage])), "r"(phase ^ 1u) : "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])),
                             "r"(kChunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                             " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sm + stage * kChunk)), "l"(base + c * kChunk),
                             "r"(kChunk), "r"(smem_u32(&full[stage])), "l"(pol) : "memory");
                if (++stage == kStages) { stage = 0; phase ^= 1u; }
            }
        }
        return;
    }
    const uint64_t c2p = pack2(1.4426950f, 1.4426950f), nm = pack2(-8.f, -8.f);
    uint64_t sA = 0, sB = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x) {
        asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                     ::"r"(smem_u32(&full[stage])), "r"(phase) : "memory");
        const uint4 *q = reinterpret_cast<const uint4 *>(sm + stage * kChunk);
        uint4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = q[tid + k * kCW * 32];
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
        if (++stage == kStages) { stage = 0; phase ^= 1u; }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            body(v[k].x, c2p, nm, sA);
            body(v[k].y, c2p, nm, sB);
            body(v[k].z, c2p, nm, sA);
            body(v[k].w, c2p, nm, sB);
        }
    }
    float a, b;
    unpack2(fadd2(sA, sB), a, b);
    if (a + b == 1234.5f) out[0] = a;
}

// direct loads: each CTA walks the same 32 KB chunks (grid-stride), thread tid owns
// vectors tid + k * 512 of a chunk; chunk c+1's loads are issued before chunk c's math
__global__ void __launch_bounds__(kCW * 32, 1) ldg_math(const char *base, size_t bytes, float *out) {
    const int tid = threadIdx.x;
    const size_t nch = bytes / kChunk;
    const uint64_t c2p = pack2(1.4426950f, 1.4426950f), nm = pack2(-8.f, -8.f);
    uint64_t sA = 0, sB = 0;
    auto ld = [&](size_t c, uint4 (&v)[4]) {
        const uint4 *q = reinterpret_cast<const uint4 *>(base + c * kChunk);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(q + tid + k * kCW * 32));
    };
    size_t c = blockIdx.x;
    if (c >= nch) return;
    uint4 cur[4], nxt[4];
    ld(c, cur);
    for (; c < nch; c += gridDim.x) {
        const size_t cn = c + gridDim.x;
        if (cn < nch) ld(cn, nxt);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            body(cur[k].x, c2p, nm, sA);
            body(cur[k].y, c2p, nm, sB);
            body(cur[k].z, c2p, nm, sA);
            body(cur[k].w, c2p, nm, sB);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) cur[k] = nxt[k];
    }
    float a, b;
    unpack2(fadd2(sA, sB), a, b);
    if (a + b == 1234.5f) out[0] = a;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = (size_t)8 * 4096 * 128256 * 2 / kChunk * kChunk;  // one grpo micro-batch
    char *buf;
    float *out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 0x3f, bytes);
    const size_t smem = kStages * kChunk + 2 * kStages * 8;
    cudaFuncSetAttribute(tma_math, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    auto A = [&]() { tma_math<<<sms, (kCW + 1) * 32, smem>>>(buf, bytes, out); };
    auto B = [&]() { ldg_math<<<sms, kCW * 32>>>(buf, bytes, out); };
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto block = [&](auto f, int n) {
        cudaEventRecord(e0);
        for (int i = 0; i < n; ++i) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms * 1e3 / n;
    };
    auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    };
    for (int w = 0; w < 3; ++w) { A(); B(); }
    cudaDeviceSynchronize();
    std::vector<double> ca, cb;
    for (int r = 0; r < 5; ++r) {
        ca.push_back(block(A, 3));
        cb.push_back(block(B, 3));
    }
    printf("cool: tma+lds %.1f us/launch (%.0f GB/s)   ldg %.1f us/launch (%.0f GB/s)  [%s]\n", med(ca),
           bytes / med(ca) / 1e3, med(cb), bytes / med(cb) / 1e3, cudaGetErrorString(cudaGetLastError()));
    auto t0 = std::chrono::steady_clock::now();
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 20.0) { block(A, 20); block(B, 20); }
    std::vector<double> ha, hb;
    for (int r = 0; r < 20; ++r) {
        ha.push_back(block(A, 15));
        hb.push_back(block(B, 15));
    }
    printf("hot:  tma+lds %.1f us/launch (%.0f GB/s)   ldg %.1f us/launch (%.0f GB/s)\n", med(ha), bytes / med(ha) / 1e3,
           med(hb), bytes / med(hb) / 1e3);
    return 0;
}

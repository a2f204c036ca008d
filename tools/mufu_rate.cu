// mufu_rate.cu -- MUFU.EX2 throughput on this GPU: how many ex2.approx.ftz.f32
// per SM clock can warps sustain, alone and mixed with the FMA-pipe work of K1's
// inner loops (per element pair: unpack, FFMA2, 2 x EX2, FADD2, FFMA2)?
// Sets the compute ceiling of the fused actor pass (2 exps per logit).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate tools/mufu_rate.cu && ./mufu_rate
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
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
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// MODE 0: independent ex2 chains only.  MODE 1: K1's forward pair body.
template <int MODE>
__global__ void kern(int iters, float seed, float *out, unsigned long long *clk) {
    const unsigned long long t0 = clock64();
    float acc = 0.f;
    if (MODE == 0) {
        float x[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = -1e-3f * (threadIdx.x + k) + seed;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) x[k] = ex2(x[k]) - 1.0f;  // dependent chain per k
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += x[k];
    } else {
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) w[k] = 0x3f803f80u ^ (threadIdx.x * 977u + k * 131u);
        const uint64_t c2p = pack2(-0.5f, -0.5f), m = pack2(seed, seed);
        uint64_t sA = 0, sB = 0, uA = 0, uB = 0;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const uint64_t x = pack2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u));
                const uint64_t t = ffma2(x, c2p, m);
                float t0, t1;
                unpack2(t, t0, t1);
                const uint64_t e = pack2(ex2(t0), ex2(t1));
                if (k & 1) { sA = fadd2(sA, e); uA = ffma2(e, t, uA); }
                else { sB = fadd2(sB, e); uB = ffma2(e, t, uB); }
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) w[k] += 0x00010001u;
        }
        float a, b;
        unpack2(fadd2(fadd2(sA, sB), fadd2(uA, uB)), a, b);
        acc = a + b;
    }
    const unsigned long long t1 = clock64();
    if (acc == 1234.5f) out[0] = acc;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    unsigned long long *clk, h[1024];
    cudaMalloc(&out, 4);
    cudaMalloc(&clk, 1024 * 8);
    const int iters = 4096;
    for (int mode = 0; mode < 2; ++mode) {
        for (int warps : {4, 8, 16, 24, 32}) {
            auto run = [&]() {
                if (mode == 0) kern<0><<<sms, warps * 32>>>(iters, 0.5f, out, clk);
                else kern<1><<<sms, warps * 32>>>(iters, 0.5f, out, clk);
            };
            run();
            cudaDeviceSynchronize();
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            run();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
            double cyc = 0;
            for (int i = 0; i < sms; ++i) cyc += h[i];
            cyc /= sms;
            const double ex2_per_sm = (double)warps * 32 * iters * 16 * (mode == 0 ? 1 : 2);
            printf("%s warps/SM %2d: %.2f ex2/clk/SM (%.1f us, %.0f MHz effective)\n",
                   mode == 0 ? "ex2 only   " : "K1 pair body", warps, ex2_per_sm / cyc, ms * 1e3,
                   cyc / (ms * 1e3));
        }
    }
    return 0;
}

// read_bw.cu -- what read-only streaming bandwidth can a B200 sustain?
// Measures (a) LDG.128 grid-stride reads, (b) a 1-D TMA bulk-copy ring into
// shared memory (K1's producer/consumer skeleton without the math), for a
// few grid shapes.  Used to set the ceiling K1 is compared against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw tools/read_bw.cu && ./read_bw
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void ldg_kernel(const uint4 *__restrict__ p, size_t n, uint32_t *out) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int U = 8;
    for (; i + (U - 1) * stride < n; i += U * stride) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint4 *q = p + i + k * stride;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(q));
        }
#pragma unroll
        for (int k = 0; k < U; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    for (; i < n; i += stride) acc ^= p[i].x;
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int CHUNK, int STAGES, int CWARPS>
__global__ void tma_kernel(const char *base, size_t row_bytes, size_t nrows, uint32_t *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * CHUNK);
    uint64_t *empty = full + STAGES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(CWARPS));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == CWARPS) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int stage = 0;
            uint32_t phase = 0;
            for (size_t r = blockIdx.x; r < nrows; r += gridDim.x)
                for (size_t off = 0; off < row_bytes; off += CHUNK) {
                    uint32_t bytes = (uint32_t)min((size_t)CHUNK, row_bytes - off);
                    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                                 ::"r"(smem_u32(&empty[stage])), "r"(phase ^ 1u) : "memory");
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                                 ::"r"(smem_u32(&full[stage])), "r"(bytes) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                                 " [%0], [%1], %2, [%3], %4;"
                                 ::"r"(smem_u32(sm + stage * CHUNK)), "l"(base + r * row_bytes + off), "r"(bytes),
                                 "r"(smem_u32(&full[stage])), "l"(pol) : "memory");
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
        }
        return;
    }
    uint32_t acc = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (size_t r = blockIdx.x; r < nrows; r += gridDim.x)
        for (size_t off = 0; off < row_bytes; off += CHUNK) {
            asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                         ::"r"(smem_u32(&full[stage])), "r"(phase) : "memory");
            const uint4 *q = reinterpret_cast<const uint4 *>(sm + stage * CHUNK);
            for (int i = tid; i < CHUNK / 16; i += CWARPS * 32) {
                uint4 v = q[i];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
            if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
    if (acc == 0x12345678u) out[0] = acc;
}

template <int CHUNK, int STAGES, int CWARPS>
void run_tma(const char *buf, size_t row_bytes, size_t nrows, uint32_t *out, int ctas_per_sm, int sms) {
    size_t smem = STAGES * CHUNK + 2 * STAGES * 8;
    auto k = tma_kernel<CHUNK, STAGES, CWARPS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k<<<grid, (CWARPS + 1) * 32, smem>>>(buf, row_bytes, nrows, out);
    cudaEventRecord(a);
    const int it = 10;
    for (int w = 0; w < it; ++w) k<<<grid, (CWARPS + 1) * 32, smem>>>(buf, row_bytes, nrows, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double gbs = (double)row_bytes * nrows * it / (ms / 1e3) / 1e9;
    printf("tma chunk=%6d stages=%d cwarps=%2d ctas/sm=%d : %8.1f GB/s  (%s)\n", CHUNK, STAGES, CWARPS,
           ctas_per_sm, gbs, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t row_bytes = 128256 * 2, nrows = 8192 * 4;  // 8.4 GB
    char *buf;
    uint32_t *out;
    cudaMalloc(&buf, row_bytes * nrows);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, row_bytes * nrows);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int cps : {1, 2, 4, 8}) {
        int grid = sms * cps;
        for (int w = 0; w < 3; ++w) ldg_kernel<<<grid, 512>>>((const uint4 *)buf, row_bytes * nrows / 16, out);
        cudaEventRecord(a);
        for (int w = 0; w < 10; ++w) ldg_kernel<<<grid, 512>>>((const uint4 *)buf, row_bytes * nrows / 16, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("ldg   512 thr x %d ctas/sm           : %8.1f GB/s\n", cps,
               (double)row_bytes * nrows * 10 / (ms / 1e3) / 1e9);
    }
    run_tma<16384, 6, 8>(buf, row_bytes, nrows, out, 2, sms);
    run_tma<16384, 12, 8>(buf, row_bytes, nrows, out, 1, sms);
    run_tma<32768, 6, 8>(buf, row_bytes, nrows, out, 1, sms);
    run_tma<16384, 4, 4>(buf, row_bytes, nrows, out, 3, sms);
    run_tma<8192, 8, 4>(buf, row_bytes, nrows, out, 3, sms);
    run_tma<16384, 6, 16>(buf, row_bytes, nrows, out, 2, sms);
    run_tma<65536, 3, 8>(buf, row_bytes, nrows, out, 1, sms);
    return 0;
}

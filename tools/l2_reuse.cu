// l2_reuse.cu -- how far back can a streaming kernel re-read its own rows from
// L2 on a B200?  Every CTA (one per SM) TMA-loads row i (first touch, from HBM)
// and then row i-d again (second touch); the time of the 2x traffic tells how
// much of the re-read hit L2.  Informs the fused actor forward+backward (K1
// mode 2), which re-reads a row ~1-2 rows (per CTA) after its first touch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_reuse tools/l2_reuse.cu && ./l2_reuse
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int CHUNK = 32768, STAGES = 6;

__global__ void __launch_bounds__(288, 1) reuse_kernel(const char *base, size_t row_bytes, int rows_per_cta, int d,
                                                       int pol_first_kind, uint32_t *out) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + STAGES * CHUNK);
    uint64_t *empty = full + STAGES;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // schedule: for i: load row i (first), then if i >= d: load row i-d (second)
    if (warp == 8) {
        if (lane == 0) {
            uint64_t pol1, pol2;
            if (pol_first_kind == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol1));
            else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol1));
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol2));
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0; i < rows_per_cta + d; ++i) {
                for (int pass = 0; pass < 2; ++pass) {
                    const int r = pass == 0 ? i : i - d;
                    if (pass == 0 && i >= rows_per_cta) continue;
                    if (pass == 1 && (r < 0 || d == 0)) continue;
                    const char *src = base + ((size_t)r * gridDim.x + blockIdx.x) * row_bytes;
                    for (size_t off = 0; off < row_bytes; off += CHUNK) {
                        uint32_t bytes = (uint32_t)min((size_t)CHUNK, row_bytes - off);
                        asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                                     ::"r"(smem_u32(&empty[stage])), "r"(phase ^ 1u) : "memory");
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                                     ::"r"(smem_u32(&full[stage])), "r"(bytes) : "memory");
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                                     " [%0], [%1], %2, [%3], %4;"
                                     ::"r"(smem_u32(sm + stage * CHUNK)), "l"(src + off), "r"(bytes),
                                     "r"(smem_u32(&full[stage])), "l"(pass == 0 ? pol1 : pol2) : "memory");
                        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                    }
                }
            }
        }
        return;
    }
    uint32_t acc = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (int i = 0; i < rows_per_cta + d; ++i)
        for (int pass = 0; pass < 2; ++pass) {
            const int r = pass == 0 ? i : i - d;
            if (pass == 0 && i >= rows_per_cta) continue;
            if (pass == 1 && (r < 0 || d == 0)) continue;
            for (size_t off = 0; off < row_bytes; off += CHUNK) {
                asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W;}"
                             ::"r"(smem_u32(&full[stage])), "r"(phase) : "memory");
                const uint4 *q = reinterpret_cast<const uint4 *>(sm + stage * CHUNK);
                for (int k = tid; k < CHUNK / 16; k += 256) acc ^= q[k].x;
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
        }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t row_bytes = 128256 * 2;
    const int rows_per_cta = 64;
    const size_t total = row_bytes * rows_per_cta * sms;
    char *buf;
    uint32_t *out;
    cudaMalloc(&buf, total);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 1, total);
    const size_t smem = STAGES * CHUNK + 2 * STAGES * 8;
    cudaFuncSetAttribute(reuse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int pol = 1; pol <= 2; ++pol)
        for (int d : {0, 1, 2, 3, 4, 6, 8}) {
            for (int w = 0; w < 2; ++w) reuse_kernel<<<sms, 288, smem>>>(buf, row_bytes, rows_per_cta, d, pol, out);
            cudaEventRecord(a);
            reuse_kernel<<<sms, 288, smem>>>(buf, row_bytes, rows_per_cta, d, pol, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = (double)total * (d > 0 ? 2 : 1);
            printf("first-touch %s  d=%d rows (%.0f MB chip-wide between touches): %.3f ms, %.1f GB/s of requested bytes\n",
                   pol == 1 ? "evict_last  " : "evict_normal", d, d * row_bytes * sms / 1e6, ms, bytes / (ms / 1e3) / 1e9);
        }
    return 0;
}

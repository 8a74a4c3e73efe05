// Microbenchmark: tcgen05.mma kind::i8 issue/throughput vs N (M = 128, K = 32),
// A from TMEM (TS) or shared memory (SS).  One CTA per SM, one issuing thread,
// back-to-back MMAs into 1..4 accumulators; prints clocks per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tcmb scripts/tc_microbench.cu && ./tcmb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N, bool TS, int NACC, int KIND>
__global__ void bench(int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t taddr;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // KIND 0: i8 (s32 acc), 1: f16 (f32 acc), 2: tf32 (f32 acc), 3: bf16 (f32 acc)
    const uint32_t fmt = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10)) : KIND == 1 ? (1u << 4)
                       : KIND == 2 ? ((1u << 4) | (2u << 7) | (2u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10));
    const uint32_t idesc = fmt | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bd = desc(smem_u32(sm), N * 16, 128);
    const uint64_t ad = desc(smem_u32(sm) + 32768, 128 * 16, 128);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t acc = (uint32_t)((j % NACC) * N);
#define MMA_CASE(K, KS)                                                                                     \
                if (KIND == K) {                                                                                \
                    if (TS)                                                                                     \
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::" KS \
                                     " [%0], [%1], %2, %3, p;\n}\n" ::"r"(acc), "r"(448u), "l"(bd), "r"(idesc), "r"(1)); \
                    else                                                                                        \
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::" KS \
                                     " [%0], %1, %2, %3, p;\n}\n" ::"r"(acc), "l"(ad), "l"(bd), "r"(idesc), "r"(1)); \
                }
                MMA_CASE(0, "i8")
                MMA_CASE(1, "f16")
                MMA_CASE(2, "tf32")
                MMA_CASE(3, "f16")
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)) : "memory");
        t1 = clock64();
        out[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u));
}

template <int N, bool TS, int NACC, int KIND = 0>
void run(unsigned long long* d) {
    const int reps = 2000;
    auto k = bench<N, TS, NACC, KIND>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<148, 128, 64 * 1024>>>(reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double per = avg / (reps * 16.0);
    const double ideal = 128.0 * N / 256;  // every kind: M=128 x N x (32 bytes of K) per N/2 clk
    printf("kind %d N=%3d %s nacc=%d: %6.2f clk/MMA  (ideal %5.1f)  eff %.2f  %s\n", KIND, N, TS ? "TS" : "SS", NACC, per, ideal, ideal / per, cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 148 * 8);
    run<48, true, 4, 0>(d);
    run<96, true, 4, 0>(d);
    run<112, true, 4, 0>(d);
    run<128, true, 2, 0>(d);
    run<48, true, 4, 1>(d);
    run<64, true, 4, 1>(d);
    run<96, true, 4, 1>(d);
    run<128, true, 2, 1>(d);
    run<192, true, 2, 1>(d);
    run<256, true, 1, 1>(d);
    run<128, false, 2, 1>(d);
    run<256, false, 1, 1>(d);
    run<64, true, 4, 2>(d);
    run<128, true, 2, 2>(d);
    run<256, true, 1, 2>(d);
    run<128, true, 2, 3>(d);
    return 0;
}

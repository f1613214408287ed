// Per-stage overhead probe (whole-warp elect.sync issue): 8 TS MMAs (N = 144) per stage plus
// (mode bits) 1: one tcgen05.commit, 2: two try_waits on a completed barrier, 4: tcgen05.fence::after.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__global__ void probe(int N, int NS, int mode, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar, done[4], ready;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&done[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ready)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&ready)));   // phase 0 complete
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot;
    const uint32_t idesc = (1u << 4) | (uint32_t(N >> 3) << 17) | (8u << 24);
    const uint64_t bd0 = desc(su32(sm + 32768));
    if (warp == 0) {
        long long t0, t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
        for (int st = 0; st < NS; ++st) {
            if (mode & 4) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t en = (st > 0 || kk > 0) ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + h * 160),
                                 "r"(tb + 320 + h * 32 + kk * 8), "l"(bd0 + kk * 2), "r"(idesc), "r"(en) : "memory");
                }
                if ((mode & 2) && kk == 1) {
                    asm volatile("{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n}" ::"r"(su32(&ready)) : "memory");
                    asm volatile("{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}" ::"r"(su32(&ready)) : "memory");
                }
            }
            if (mode & 1)
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&done[st & 3])) : "memory");
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(su32(&bar)));
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
        if (lane == 0) out[0] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int NS = 64;
    for (int N : {16, 144})
        for (int mode : {0, 1, 2, 4, 7}) {
            long long h;
            probe<<<1, 128, 100000>>>(N, NS, mode, d);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("N=%3d mode=%d (commit=%d waits=%d fence=%d): %7.1f cycles/stage %s\n", N, mode, mode & 1,
                   (mode >> 1) & 1, (mode >> 2) & 1, double(h) / NS, cudaGetErrorString(cudaGetLastError()));
        }
}

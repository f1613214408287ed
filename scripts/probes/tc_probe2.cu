// Issue-overhead probe: lane-0-only issue vs whole-warp issue with an elect.sync-guarded MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
template <int MODE>
__global__ void probe(int N, int NI, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
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
    long long t0 = 0, t1 = 0;
    if (MODE == 0 ? threadIdx.x == 0 : warp == 0) {
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
        for (int i = 0; i < NI; i += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t en = (i + u) > 1 ? 1u : 0u;
                if (MODE == 0) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + (u & 1) * 160),
                                 "r"(tb + 384 + (u & 3) * 8), "l"(bd0 + (u & 3) * 2), "r"(idesc), "r"(en));
                } else {
                    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + (u & 1) * 160),
                                 "r"(tb + 384 + (u & 3) * 8), "l"(bd0 + (u & 3) * 2), "r"(idesc), "r"(en));
                }
            }
        }
        if (MODE == 0 || lane == 0)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
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
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int NI = 512;
    for (int N : {16, 64, 144}) {
        long long h;
        probe<0><<<1, 128, 100000>>>(N, NI, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("lane0  N=%3d : %6.1f cycles/MMA\n", N, double(h) / NI);
        probe<1><<<1, 128, 100000>>>(N, NI, d); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("elect  N=%3d : %6.1f cycles/MMA %s\n", N, double(h) / NI, cudaGetErrorString(cudaGetLastError()));
    }
}

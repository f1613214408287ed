// tcgen05 issue-rate probe (tuning only): one CTA issues NI MMAs back to back and times
// them with clock64 until the commit's mbarrier completes.  Modes: SS / TS (A from TMEM),
// N, number of accumulators the MMAs alternate over.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

__global__ void probe(int mode, int N, int nacc, int NI, long long* out, int M, int commit_every, int bg) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t dummy[4];
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&dummy[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot;
    __shared__ volatile int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (warp >= 1 && bg) {
        uint32_t r[16];
        for (int i = 0; i < 16; ++i) r[i] = i * threadIdx.x;
        uint32_t acc = 0;
        while (!stop) {
            if (bg == 1) {
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tb + ((warp & 3) * 32 << 16) + 448),
                    "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
                    "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            } else if (bg == 2) {
                for (int k = 0; k < 64; ++k) acc = acc * 1664525u + r[k & 15];
            } else {
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1;\n\tselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(su32(&dummy[3])));
                acc += ok;
            }
        }
        if (acc == 12345) out[3] = acc;
    }
    if (mode >= 2 ? warp == 0 : threadIdx.x == 0) {
        const bool conv = mode >= 2;
        const uint32_t idesc = (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
        const uint32_t a_s = su32(sm), b_s = su32(sm + 32768);
        long long t0, t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0));
        const uint64_t bd0 = desc(b_s, 16, 1024);
        const uint64_t ad0 = desc(a_s, 16, 1024);
        const uint32_t acc1 = nacc > 1 ? (N <= 128 ? 128u : 160u) : 0u;
        if (mode == 0) {
            for (int i = 0; i < NI; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t en = (i + u) > 0 ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tb + ((u & 1) ? acc1 : 0u)),
                                 "l"(ad0 + u * 2), "l"(bd0 + u * 2), "r"(idesc), "r"(en));
                }
            }
        } else {
            for (int i = 0; i < NI; i += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t en = (i + u) > 0 ? 1u : 0u;
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tb + ((u & 1) ? acc1 : 0u)),
                                 "r"(tb + 384 + u * 8), "l"(bd0 + u * 2), "r"(idesc), "r"(en));
                }
                if (commit_every && ((i + 4) % commit_every) == 0) {
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&dummy[(i / commit_every) & 3])));
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&dummy[((i / commit_every) + 1) & 3])));
                }
            }
        }
        long long ti;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(ti));
        if ((threadIdx.x & 31) == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
            su32(&bar)));
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1));
        if ((threadIdx.x & 31) == 0) { out[0] = ti - t0; out[1] = t1 - t0; }
        stop = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int NI = 512;
    printf("mode N nacc : issue_cycles/MMA  total_cycles/MMA  (floor 128*N/256 = N/2)\n");
    const char* bgn[4] = {"none", "sttm", "alu", "trywait-spin"};
    for (int bg = 0; bg < 4; ++bg)
        for (int ce : {0, 8})
            for (int N : {16, 144}) {
                probe<<<1, 128, 100000>>>(1, N, 2, NI, d, 128, ce, bg);
                long long h[2];
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                cudaError_t e = cudaGetLastError();
                printf("TS N=%3d commit_every=%d bg=%-12s : %8.1f %8.1f %s\n", N, ce, bgn[bg], double(h[0]) / NI,
                       double(h[1]) / NI, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}

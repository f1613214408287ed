// cta_group::2 semantics probe: a CTA pair computes D[256][N] = A[256][16] * B[N][16]^T with
// A in TMEM (128 rows per CTA), B K-major SW128 in smem (N/2 rows per CTA), one MMA issued by
// the leader, commit multicast to both CTAs; each CTA reads its 128 rows of D.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
    return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(64) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__device__ __forceinline__ float aval(int m, int k) { return float(((m * 7 + k * 3) % 11) - 5) * 0.25f; }
__device__ __forceinline__ float bval(int n, int k) { return float(((n * 5 + k * 2) % 9) - 4) * 0.5f; }

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(float* out) {
    __shared__ __align__(1024) uint8_t bsm[16384];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B half: rows n = rank * N/2 + r, r < N/2; K-major SW128: row r at r*128 B, 16-byte chunk c^(r&7)
    for (int i = threadIdx.x; i < (N / 2) * 16; i += blockDim.x) {     // 16 k per row (32 B = chunks 0, 1)
        const int r = i / 16, k = i % 16;
        const int n = int(rank) * (N / 2) + r;
        const int chunk = k / 8, within = k % 8;
        const uint32_t off = uint32_t(r) * 128u + uint32_t(((chunk ^ (r & 7)) << 4)) + uint32_t(within * 2);
        *reinterpret_cast<__half*>(bsm + off) = __float2half(bval(n, k));
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot;
    // A rows of this CTA: TMEM lane l = row rank*128 + l; 16 k packed as 8 columns at col 256
    {
        const int l = warp * 32 + lane;
        const int m = int(rank) * 128 + l;
        uint32_t r[8];
        for (int c = 0; c < 8; ++c) {
            __half2 h = __floats2half2_rn(aval(m, 2 * c), aval(m, 2 * c + 1));
            r[c] = *reinterpret_cast<uint32_t*>(&h);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tb + (uint32_t(warp * 32) << 16) + 256u),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (rank == 0 && warp == 0) {
        const uint32_t idesc = (1u << 4) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
        const uint64_t bd = desc(su32(bsm));
        asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tb), "r"(tb + 256u), "l"(bd),
                     "r"(idesc), "r"(0u) : "memory");
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}"
                     ::"r"(su32(&bar)), "h"((unsigned short)3) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    {
        const int l = warp * 32 + lane;
        for (int c0 = 0; c0 < N; c0 += 8) {
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(tb + (uint32_t(warp * 32) << 16) + uint32_t(c0)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int j = 0; j < 8; ++j) out[(int(rank) * 128 + l) * N + c0 + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int N>
int run() {
    float* d;
    cudaMalloc(&d, 256 * N * 4);
    cudaMemset(d, 0xFF, 256 * N * 4);
    probe<N><<<2, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    float* h = new float[256 * N];
    cudaMemcpy(h, d, 256 * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < 16; ++k)
                ref += double(float(((m * 7 + k * 3) % 11) - 5) * 0.25f) * double(float(((n * 5 + k * 2) % 9) - 4) * 0.5f);
            maxerr = fmax(maxerr, fabs(ref - h[m * N + n]));
        }
    printf("N=%d: %s, max err %g (D[0][0]=%g D[255][N-1]=%g)\n", N, cudaGetErrorString(e), maxerr, h[0], h[256 * N - 1]);
    return maxerr < 1e-3 ? 0 : 1;
}
int main() { return run<32>() | run<144>(); }

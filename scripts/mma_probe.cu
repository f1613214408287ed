#include <stdint.h>
#include <stdio.h>
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__global__ void k(const uint32_t* in, int* out, int iters) {
    int d0[4] = {0,0,0,0}, d1[4] = {0,0,0,0}, d2[4]={0,0,0,0}, d3[4]={0,0,0,0};
    uint32_t a = in[threadIdx.x], b = in[threadIdx.x + 32];
    for (int i = 0; i < iters; ++i) {
        mma_u8s8(d0, a, 0, a ^ i, 0, b, b ^ i);
        mma_u8s8(d1, a ^ 1, 0, a, 0, b, b);
        mma_u8s8(d2, a ^ 2, 0, a, 0, b ^ 3, b);
        mma_u8s8(d3, a ^ 3, 0, a, 0, b, b ^ 5);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = d0[0] + d1[1] + d2[2] + d3[3] + d0[3];
}
int main() {
    uint32_t* in; int* out; cudaMalloc(&in, 4096); cudaMalloc(&out, 148 * 8 * 1024 * 4);
    cudaMemset(in, 1, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps = 4; warps <= 32; warps *= 2) {
        k<<<148, warps * 32>>>(in, out, 1000);
        cudaEventRecord(e0);
        k<<<148, warps * 32>>>(in, out, 10000);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double mmas = 148.0 * warps * 10000 * 4;
        printf("warps/SM %d: %.3f ms, %.2f mma/clk/SM at 1.9GHz, %.1f TOPS\n", warps, ms, mmas / (ms * 1e-3) / 148 / 1.9e9, mmas * 4096 * 2 / (ms * 1e-3) / 1e12);
    }
    return 0;
}

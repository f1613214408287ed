// quant.cu -- group-wise 4-bit quantize / dequantize / KV-append kernels (sm_100a).
//
// FlexGen Sec. 4: per group of g = 64 contiguous
// elements, x_quant = round((x - min) / (max - min) * (2^b - 1)), b = 4.
// The fp32 operation order is fixed (reading B): a = RN(x - min),
// u = RN(a / r) with IEEE division, t = RN(u * 15), code = RNE(clamp(t, 0, 15)).
// Every float op below is an explicit round-to-nearest intrinsic and this TU
// is compiled with -fmad=false, so nothing is contracted into an FMA.
//
// Mapping: 4 lanes per group, 16 elements (32 B of fp16) per lane, two 128-bit
// loads; group min/max by two xor-shuffles; each lane stores 8 B of packed
// codes (a warp writes 256 contiguous bytes); lane 0 of the group stores the
// half2 {scale, min}.  HBM-bound: 2 B read + 0.5625 B written per element.
#include <cuda_fp16.h>
#include <stdint.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void h2_to_f(uint32_t w, float& lo, float& hi) {
    __half2 h = *reinterpret_cast<__half2*>(&w);
    float2 f = __half22float2(h);   // exact
    lo = f.x;
    hi = f.y;
}

__device__ __forceinline__ int64_t dst_row(int64_t row, const RowMap& m) {
    if (m.n_new == 0) return row;
    int64_t bh = row / m.n_new;
    return bh * m.t_cap + m.pos + (row - bh * m.n_new);
}

// Code of one element (reading B): every step one IEEE round-to-nearest op.
__device__ __forceinline__ uint32_t code_of(float x, float mn, float r) {
    float a = __fsub_rn(x, mn);
    float u = __fdiv_rn(a, r);
    float t = __fmul_rn(u, 15.0f);
    t = fminf(fmaxf(t, 0.0f), 15.0f);                         // reading D (a no-op)
    return __float_as_uint(__fadd_rn(t, 8388608.0f)) & 0xFu;  // 2^23 + RNE(t)
}

__global__ void __launch_bounds__(kThreads)
quantize_kernel(const __half* __restrict__ x0, uint8_t* __restrict__ codes0, __half2* __restrict__ meta0,
                const __half* __restrict__ x1, uint8_t* __restrict__ codes1, __half2* __restrict__ meta1,
                int64_t rows, int64_t cols, RowMap map) {
    const __half* x = blockIdx.y ? x1 : x0;
    uint8_t* codes = blockIdx.y ? codes1 : codes0;
    __half2* meta = blockIdx.y ? meta1 : meta0;

    const int lane = threadIdx.x & 31;
    const int part = lane & 3;
    const int64_t gpr = cols / kGroup;
    const int64_t total = rows * gpr;
    const int64_t warp0 = (int64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * kThreads) >> 5;

    for (int64_t wg = warp0 * 8; wg < total; wg += nwarps * 8) {   // warp-uniform loop
        const int64_t g = wg + (lane >> 2);
        const bool valid = g < total;
        float v[16];
        if (valid) {
            const int64_t row = g / gpr, k = g - row * gpr;
            const __half* p = x + row * cols + k * kGroup + part * 16;
            uint4 a = ld_stream(p), b = ld_stream(p + 8);
            h2_to_f(a.x, v[0], v[1]);   h2_to_f(a.y, v[2], v[3]);
            h2_to_f(a.z, v[4], v[5]);   h2_to_f(a.w, v[6], v[7]);
            h2_to_f(b.x, v[8], v[9]);   h2_to_f(b.y, v[10], v[11]);
            h2_to_f(b.z, v[12], v[13]); h2_to_f(b.w, v[14], v[15]);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.0f;
        }
        float mn = v[0], mx = v[0];
#pragma unroll
        for (int j = 1; j < 16; ++j) { mn = fminf(mn, v[j]); mx = fmaxf(mx, v[j]); }
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, 2));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        if (!valid) continue;
        mn = (mn == 0.0f) ? 0.0f : mn;            // reading P: -0 -> +0
        const float r = __fsub_rn(mx, mn);        // RN32(max - min)
        uint32_t lo = 0, hi = 0;
        __half scale16 = __float2half_rn(0.0f);
        if (r != 0.0f) {                          // reading C: degenerate group -> codes 0
            scale16 = __float2half_rn(__fdiv_rn(r, 15.0f));
#pragma unroll
            for (int j = 0; j < 8; ++j) lo |= code_of(v[j], mn, r) << (4 * j);
#pragma unroll
            for (int j = 0; j < 8; ++j) hi |= code_of(v[8 + j], mn, r) << (4 * j);
        }
        const int64_t row = g / gpr, k = g - row * gpr;
        const int64_t drow = dst_row(row, map);
        *reinterpret_cast<uint2*>(codes + drow * (cols / 2) + k * (kGroup / 2) + part * 8) = make_uint2(lo, hi);
        if (part == 0) meta[drow * gpr + k] = __halves2half2(scale16, __float2half_rn(mn));
    }
}

// out = f16(clamp(fmaf(code, scale, min), +-65504))   (reading R)
__global__ void __launch_bounds__(kThreads)
dequantize_kernel(const uint8_t* __restrict__ codes, const __half2* __restrict__ meta,
                  __half* __restrict__ out, int64_t rows, int64_t cols) {
    const int lane = threadIdx.x & 31;
    const int part = lane & 3;
    const int64_t gpr = cols / kGroup;
    const int64_t total = rows * gpr;
    const int64_t t0 = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nthr = int64_t(gridDim.x) * kThreads;
    for (int64_t t = t0; t < total * 4; t += nthr) {
        const int64_t g = t >> 2;
        const int64_t row = g / gpr, k = g - row * gpr;
        uint2 c = *reinterpret_cast<const uint2*>(codes + row * (cols / 2) + k * (kGroup / 2) + part * 8);
        float2 sm = __half22float2(meta[g]);
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t w = j < 4 ? c.x : c.y;
            int s = (j & 3) * 8;
            float c0 = __uint_as_float(0x4B000000u | ((w >> s) & 0xFu)) - 8388608.0f;        // exact
            float c1 = __uint_as_float(0x4B000000u | ((w >> (s + 4)) & 0xFu)) - 8388608.0f;
            float y0 = fminf(fmaxf(__fmaf_rn(c0, sm.x, sm.y), -65504.0f), 65504.0f);
            float y1 = fminf(fmaxf(__fmaf_rn(c1, sm.x, sm.y), -65504.0f), 65504.0f);
            __half2 h = __halves2half2(__float2half_rn(y0), __float2half_rn(y1));
            o[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + row * cols + k * kGroup + part * 16);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace

cudaError_t launch_quantize(const void* x, int64_t rows, int64_t cols, void* codes, void* meta,
                            const void* x2, void* codes2, void* meta2, RowMap map,
                            cudaStream_t stream) {
    const int64_t groups = rows * (cols / kGroup);
    if (groups == 0) return cudaSuccess;
    int64_t blocks = (groups * 4 + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    dim3 grid(unsigned(blocks), x2 ? 2u : 1u);
    quantize_kernel<<<grid, kThreads, 0, stream>>>(
        static_cast<const __half*>(x), static_cast<uint8_t*>(codes), static_cast<__half2*>(meta),
        static_cast<const __half*>(x2), static_cast<uint8_t*>(codes2), static_cast<__half2*>(meta2),
        rows, cols, map);
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const void* codes, const void* meta, int64_t rows, int64_t cols,
                              void* out, cudaStream_t stream) {
    const int64_t groups = rows * (cols / kGroup);
    if (groups == 0) return cudaSuccess;
    int64_t blocks = (groups * 4 + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    dequantize_kernel<<<unsigned(blocks), kThreads, 0, stream>>>(
        static_cast<const uint8_t*>(codes), static_cast<const __half2*>(meta),
        static_cast<__half*>(out), rows, cols);
    return cudaGetLastError();
}

}  // namespace flexq

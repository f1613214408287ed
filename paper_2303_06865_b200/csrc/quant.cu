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
// The KV append is the same kernel writing into the chunked cache layout.
#include <cuda_fp16.h>
#include <stdint.h>

#include <mutex>

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

// Byte offsets of the packed codes (8 B per lane) and of the half2 meta of
// source group g.  Plain tensors: row-major [rows][cols/2] codes, [rows][cols/64]
// meta.  KV append: the chunked cache layout of include/flexq.h; source row
// r = bh * n_new + t goes to token pos + t of head bh, K (kv = 0) or V (kv = 1).
struct PlainDst {
    __device__ __forceinline__ void operator()(uint32_t g, uint32_t /*gpr*/, int /*kv*/, int64_t& codes_off,
                                               int64_t& meta_off) const {
        codes_off = int64_t(g) * (kGroup / 2);
        meta_off = int64_t(g) * 4;
    }
    // the lane's 16 codes (8 bytes, element 2i in the low nibble of byte i)
    __device__ __forceinline__ void store_codes(uint8_t* base, int64_t co, int part, int /*kv*/, uint32_t lo,
                                                uint32_t hi) const {
        *reinterpret_cast<uint2*>(base + co + part * 8) = make_uint2(lo, hi);
    }
};
// Unsigned division by a runtime constant d < 2^31 via multiply-high
// (Granlund-Montgomery): q = (umulhi(x, mul) + x) >> shift for x < 2^31.
struct FastDiv {
    uint32_t d, mul, shift;
    static FastDiv make(uint32_t d) {
        FastDiv f;
        f.d = d;
        f.shift = 0;
        while ((1ull << f.shift) < d) ++f.shift;
        f.mul = uint32_t(((1ull << 32) * ((1ull << f.shift) - d)) / d + 1);
        return f;
    }
    __device__ __forceinline__ uint32_t div(uint32_t x) const { return (__umulhi(x, mul) + x) >> shift; }
};

struct KvChunkDst {
    KvDst d;
    FastDiv nnew;   // divisor n_new
    int gpr_log2;   // log2(groups per row) (head_dim / 64 = 1 or 2)
    int cb;         // code bytes per token (D/2)
    int v_tm;       // 1: V token-major like K (FLEXQ_KV_TOKEN_MAJOR); 0: V quad-interleaved (FLEXQ_KV_DENSE)
    // codes_off: K (and token-major V) -> byte offset of the token's codes of group k;
    //            quad V -> byte offset of the first column-pair word of group k in the token's
    //               quad, plus the token's byte lane (t % 4)   (include/flexq.h layout).
    __device__ __forceinline__ void operator()(uint32_t g, uint32_t /*gpr*/, int kv, int64_t& codes_off,
                                               int64_t& meta_off) const {
        const uint32_t row = g >> gpr_log2, k = g & ((1u << gpr_log2) - 1u);
        const uint32_t bh = nnew.div(row);
        const int64_t t = d.pos + (row - bh * nnew.d);
        const int64_t chunk = int64_t(bh) * d.chunks + (t >> 5);
        const int slot = int(t & (kChunk - 1));
        const int mb = cb / 8;                                            // meta bytes per token
        const int64_t base = chunk * (kChunk * (cb + mb));                // kv_chunk_bytes(2 cb)
        if (kv == 0 || v_tm)
            codes_off = base + slot * cb + k * (kGroup / 2);
        else   // word (quad, first pair of group k), plus the token's byte lane; + the quad's swizzle
            codes_off = (base + ((slot >> 2) * cb + k * (kGroup / 2)) * 4 + (slot & 3)) * 4 + ((slot >> 2) & 3);
        meta_off = base + kChunk * cb + slot * mb + k * 4;
    }
    __device__ __forceinline__ void store_codes(uint8_t* base, int64_t co, int part, int kv, uint32_t lo,
                                                uint32_t hi) const {
        if (kv == 0 || v_tm) {
            *reinterpret_cast<uint2*>(base + co + part * 8) = make_uint2(lo, hi);
        } else {   // V: byte i (column pair part*8 + i of the group) -> word (quad, pair ^ (swz << 3)), byte t % 4
            const int swz = int(co & 3);   // V offsets carry the swizzle (quad & 3) in 2 low bits (operator())
            uint8_t* p = base + (co >> 2) + (part ^ swz) * 32;
#pragma unroll
            for (int i = 0; i < 4; ++i) p[4 * i] = uint8_t(lo >> (8 * i));
#pragma unroll
            for (int i = 0; i < 4; ++i) p[16 + 4 * i] = uint8_t(hi >> (8 * i));
        }
    }
};

// Division u = RN(a / r) by one correctly rounded reciprocal per group and a
// Markstein correction per element: y = RN(1/r), q0 = RN(a*y),
// e = fma(-q0, r, a) (exact), u = RN(q0 + e*y).  Markstein's theorem (y within
// 1/2 ulp of 1/r, q0 within 1 ulp of a/r, no over/underflow: here
// a in [0, 131008], r in [2^-24, 131008]) makes u the IEEE quotient; the
// host test tests/test_division.py checks it on 4e7 samples of the exact
// operand domain, and the GPU parity tests compare every code with the
// oracle's true division.  u in [0, 1] => t = RN(15 u) in [0, 15], so the
// clamp of reading D is a no-op and is not repeated here.
//
// Codes of 8 consecutive elements -> one packed 32-bit word.  Each code is
// produced as the float 2^23 + c (RNE to integer via the magic add); Horner
// packing acc = acc * 16 + bits over the 8 floats' bit patterns leaves the
// constant 0x4B000000 * (1 + 16) mod 2^32 = 0xFB000000 on top of the packed
// codes (the 0x4B000000 * 16^j terms for j >= 2 vanish mod 2^32).
__device__ __forceinline__ uint32_t codes8(const float2 (&x)[4], float mn, float r, float y) {
    const float2 nmn = make_float2(-mn, -mn), yy = make_float2(y, y), nr = make_float2(-r, -r);
    uint32_t acc = 0;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
        const float2 a = __fadd2_rn(x[k], nmn);            // RN(x - min)
        const float2 q0 = __fmul2_rn(a, yy);               // RN(a * y)
        const float2 e = __ffma2_rn(q0, nr, a);            // a - q0 r, exact
        const float2 u = __ffma2_rn(e, yy, q0);            // RN(a / r)
        // t = RN(u * 15) and the magic add stay scalar __fmul_rn / __fadd_rn: ptxas
        // contracts a packed mul.rn.f32x2 + add.rn.f32x2 pair into one FFMA2 (single
        // rounding), which breaks RNE at exact .5 ties (reading A); the scalar
        // round-to-nearest intrinsics are never merged.
        const float t0 = __fmul_rn(u.x, 15.0f), t1 = __fmul_rn(u.y, 15.0f);
        const float b0 = __fadd_rn(t0, 8388608.0f), b1 = __fadd_rn(t1, 8388608.0f);   // 2^23 + RNE(t)
        acc = acc * 16u + __float_as_uint(b1);
        acc = acc * 16u + __float_as_uint(b0);
    }
    return acc - 0xFB000000u;
}

__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// blockIdx.y selects source x0 -> (codes0, meta0) or x1 -> (codes1, meta1):
// byte base pointers of the destination (the same cache buffer for codes and
// meta of the KV cache).
template <class Dst>
__global__ void __launch_bounds__(kThreads)
quantize_kernel(const __half* __restrict__ x0, const __half* __restrict__ x1, uint8_t* __restrict__ codes0,
                uint8_t* __restrict__ meta0, uint8_t* __restrict__ codes1, uint8_t* __restrict__ meta1,
                int64_t rows, int64_t cols, Dst dst) {
    const int kv = blockIdx.y;
    const __half* x = kv ? x1 : x0;
    uint8_t* codes_base = kv ? codes1 : codes0;
    uint8_t* meta_base = kv ? meta1 : meta0;

    const int lane = threadIdx.x & 31;
    const int part = lane & 3;
    const uint32_t gpr = uint32_t(cols / kGroup);
    const uint32_t total = uint32_t(rows * gpr);
    const uint32_t warp0 = (blockIdx.x * kThreads + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * kThreads) >> 5;

    for (uint32_t wg = warp0 * 8; wg < total; wg += nwarps * 8) {   // warp-uniform loop
        const uint32_t g = wg + (lane >> 2);
        const bool valid = g < total;
        uint4 va = make_uint4(0, 0, 0, 0), vb = va;
        if (valid) {
            const __half* p = x + int64_t(g) * kGroup + part * 16;
            va = ld_stream(p);
            vb = ld_stream(p + 8);
        }
        // O3: exact group min / max on the fp16 values (half2 min/max), then 2 shuffles
        const __half2 h[8] = {u2h(va.x), u2h(va.y), u2h(va.z), u2h(va.w),
                              u2h(vb.x), u2h(vb.y), u2h(vb.z), u2h(vb.w)};
        __half2 lo = __hmin2(__hmin2(__hmin2(h[0], h[1]), __hmin2(h[2], h[3])),
                             __hmin2(__hmin2(h[4], h[5]), __hmin2(h[6], h[7])));
        __half2 hi = __hmax2(__hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])),
                             __hmax2(__hmax2(h[4], h[5]), __hmax2(h[6], h[7])));
        __half2 mm = __halves2half2(__hmin(__low2half(lo), __high2half(lo)),
                                    __hmax(__low2half(hi), __high2half(hi)));   // (min, max)
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
            const __half2 t = u2h(__shfl_xor_sync(0xffffffffu, h2u(mm), o));
            mm = __halves2half2(__hmin(__low2half(mm), __low2half(t)), __hmax(__high2half(mm), __high2half(t)));
        }
        if (!valid) continue;
        float mn = __low2float(mm);   // exact (an fp16 value)
        const float mx = __high2float(mm);
        mn = (mn == 0.0f) ? 0.0f : mn;            // reading P: -0 -> +0
        const float r = __fsub_rn(mx, mn);        // RN32(max - min)
        uint32_t wlo = 0, whi = 0;
        __half scale16 = __float2half_rn(0.0f);
        if (r != 0.0f) {                          // reading C: degenerate group -> codes 0
            // RN(r / 15) by one Markstein step on RN(1/15): equal to the IEEE quotient for every
            // fp32 r in the operand range (tests/test_division.py, exhaustive), ~15 instructions
            // cheaper than __fdiv_rn
            constexpr float kInv15 = 0.0666666701436042785645f;   // RN(1/15) = 0x3D888889
            const float s0 = __fmul_rn(r, kInv15);
            scale16 = __float2half_rn(__fmaf_rn(__fmaf_rn(-s0, 15.0f, r), kInv15, s0));
            const float y = __frcp_rn(r);
            float2 f[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) f[j] = __half22float2(h[j]);
            wlo = codes8(f, mn, r, y);
#pragma unroll
            for (int j = 0; j < 4; ++j) f[j] = __half22float2(h[4 + j]);
            whi = codes8(f, mn, r, y);
        }
        int64_t co, mo;
        dst(g, gpr, kv, co, mo);
        dst.store_codes(codes_base, co, part, kv, wlo, whi);
        if (part == 0) *reinterpret_cast<__half2*>(meta_base + mo) = __halves2half2(scale16, __float2half_rn(mn));
    }
}

// out = f16(clamp(fmaf(code, scale, min), +-65504))   (reading R)
// The nibble n at bit position 4k of a word becomes the float 2^23 + n 16^k
// with one LOP3; subtracting 2^23 is exact, and (n 16^k) * (scale 16^-k) is
// the exact product n * scale, so one FFMA2 gives fmaf(n, scale, min) for two
// elements.  cvt.rn.satfinite clamps to +-65504 exactly like the clamp + RN.
__device__ __forceinline__ uint32_t magic_reg() {
    uint32_t m;
    asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(m));
    return m;
}
template <uint32_t M>
__device__ __forceinline__ float nib(uint32_t w, uint32_t magic) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(M), "r"(magic));  // (a & b) | c
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t sat_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
__device__ __forceinline__ void deq8(uint32_t w, uint32_t magic, const float2 (&s)[4], float2 m2, uint32_t* o) {
    const uint32_t w4 = w >> 4;   // odd nibbles
    const float2 bias = make_float2(-8388608.0f, -8388608.0f);
    // pairs (even nibble, odd nibble) of each byte: bytes 0..3 -> columns (0,1) (2,3) (4,5) (6,7)
    const float2 f0 = __fadd2_rn(make_float2(nib<0x0000000Fu>(w, magic), nib<0x0000000Fu>(w4, magic)), bias);
    const float2 f1 = __fadd2_rn(make_float2(nib<0x00000F00u>(w, magic), nib<0x00000F00u>(w4, magic)), bias);
    const float2 f2 = __fadd2_rn(make_float2(nib<0x000F0000u>(w, magic), nib<0x000F0000u>(w4, magic)), bias);
    const uint32_t w16 = w >> 16, w20 = w >> 20;
    const float2 f3 = __fadd2_rn(make_float2(nib<0x00000F00u>(w16, magic), nib<0x00000F00u>(w20, magic)), bias);
    float2 y;
    y = __ffma2_rn(f0, s[0], m2); o[0] = sat_pack(y.x, y.y);
    y = __ffma2_rn(f1, s[1], m2); o[1] = sat_pack(y.x, y.y);
    y = __ffma2_rn(f2, s[2], m2); o[2] = sat_pack(y.x, y.y);
    y = __ffma2_rn(f3, s[3], m2); o[3] = sat_pack(y.x, y.y);
}

#ifndef FLEXQ_DEQ_UNROLL
#define FLEXQ_DEQ_UNROLL 4      // group-parts per thread per iteration: loads issued together
#endif
#ifndef FLEXQ_DEQ_CS
#define FLEXQ_DEQ_CS 1          // streaming (evict-first) stores of the fp16 output
#endif
__device__ __forceinline__ void st_out(uint4* p, uint4 v) {
#if FLEXQ_DEQ_CS
    __stcs(p, v);
#else
    *p = v;
#endif
}

__global__ void __launch_bounds__(kThreads)
dequantize_kernel(const uint8_t* __restrict__ codes, const __half2* __restrict__ meta,
                  __half* __restrict__ out, int64_t rows, int64_t cols) {
    constexpr int U = FLEXQ_DEQ_UNROLL;
    const int64_t total = rows * (cols / kGroup) * 4;       // group parts (16 elements each)
    const int64_t t0 = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nthr = int64_t(gridDim.x) * kThreads;
    const uint32_t magic = magic_reg();
    for (int64_t tb = t0; tb < total; tb += nthr * U) {
        uint2 c[U];
        float2 sm[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {          // all loads of the U parts first (memory-level parallelism)
            const int64_t t = tb + int64_t(u) * nthr;
            if (t < total) {
                c[u] = __ldcs(reinterpret_cast<const uint2*>(codes + (t >> 2) * (kGroup / 2) + (t & 3) * 8));
                sm[u] = __half22float2(meta[t >> 2]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t t = tb + int64_t(u) * nthr;
            if (t >= total) break;
            // scale * 16^-k for the nibble positions used by deq8: (0,0), (8,8), (16,16), (8,8)
            const float2 s[4] = {make_float2(sm[u].x, sm[u].x),
                                 make_float2(sm[u].x * 0.00390625f, sm[u].x * 0.00390625f),
                                 make_float2(sm[u].x * 1.52587890625e-05f, sm[u].x * 1.52587890625e-05f),
                                 make_float2(sm[u].x * 0.00390625f, sm[u].x * 0.00390625f)};
            const float2 m2 = make_float2(sm[u].y, sm[u].y);
            uint32_t o[8];
            deq8(c[u].x, magic, s, m2, o);
            deq8(c[u].y, magic, s, m2, o + 4);
            uint4* dst = reinterpret_cast<uint4*>(out + (t >> 2) * kGroup + (t & 3) * 16);
            st_out(dst, make_uint4(o[0], o[1], o[2], o[3]));
            st_out(dst + 1, make_uint4(o[4], o[5], o[6], o[7]));
        }
    }
}

// ------------------------------------------------------------------ other (b, g): NEXT-3 variants
// Same fp32 sequence as the b = 4, g = 64 kernel with 2^b - 1 levels (reading B), for
// b in {2, 3, 8} (and 4) and g in {32, 64, 128}.  G / 16 lanes per group, 16 elements per
// lane; codes are a little-endian bit stream per row, so a lane's 16 codes are the
// 2b bytes at (16 * element index) * b / 8 -- byte aligned for every b.
template <int B>
__device__ __forceinline__ void store_bits(uint8_t* p, uint64_t lo, uint64_t hi) {
    if constexpr (B == 2) {
        *reinterpret_cast<uint32_t*>(p) = uint32_t(lo);
    } else if constexpr (B == 3) {                      // 6 bytes at a 2-byte aligned offset
        uint16_t* q = reinterpret_cast<uint16_t*>(p);
        q[0] = uint16_t(lo);
        q[1] = uint16_t(lo >> 16);
        q[2] = uint16_t(lo >> 32);
    } else if constexpr (B == 4) {
        *reinterpret_cast<uint64_t*>(p) = lo;
    } else {
        *reinterpret_cast<uint4*>(p) = make_uint4(uint32_t(lo), uint32_t(lo >> 32), uint32_t(hi), uint32_t(hi >> 32));
    }
}

// Destination of group g's codes (lane `part`'s 2b bytes) and half2 meta.  Plain tensors:
// [rows][cols * b / 8] bit-stream rows and [rows][cols / g] meta.
template <int B, int G>
struct PlainBitsDst {
    __device__ __forceinline__ void operator()(int64_t g, int part, int64_t& co, int64_t& mo) const {
        co = (g * G + part * 16) * B / 8;
        mo = g * 4;
    }
};
// KV append of the variants: the chunked cache layout of include/flexq.h with CB = D b / 8 code
// bytes (the token's row as a little-endian bit stream, K and V alike) and MB = 4 D / g meta
// bytes per token; chunk = [codes 32 x CB][meta 32 x MB].  Source row r = bh * n_new + t goes to
// token pos + t of head bh.
template <int B, int G>
struct KvBitsDst {
    int64_t pos, chunks;
    FastDiv nnew;
    int gpr_log2, cb, mb;
    __device__ __forceinline__ void operator()(int64_t g, int part, int64_t& co, int64_t& mo) const {
        const uint32_t row = uint32_t(g >> gpr_log2), k = uint32_t(g) & ((1u << gpr_log2) - 1u);
        const uint32_t bh = nnew.div(row);
        const int64_t t = pos + (row - bh * nnew.d);
        const int64_t base = (int64_t(bh) * chunks + (t >> 5)) * (kChunk * (cb + mb));
        const int slot = int(t & (kChunk - 1));
        co = base + slot * cb + (int64_t(k) * G + part * 16) * B / 8;
        mo = base + kChunk * cb + slot * mb + k * 4;
    }
};

// blockIdx.y selects source x0 -> (codes0, meta0) or x1 -> (codes1, meta1) (byte bases)
template <int B, int G, class Dst>
__global__ void __launch_bounds__(kThreads)
quantize_generic_kernel(const __half* __restrict__ x0, const __half* __restrict__ x1, uint8_t* __restrict__ codes0,
                        uint8_t* __restrict__ meta0, uint8_t* __restrict__ codes1, uint8_t* __restrict__ meta1,
                        int64_t groups, Dst dst) {
    const int kv = blockIdx.y;
    const __half* x = kv ? x1 : x0;
    uint8_t* codes = kv ? codes1 : codes0;
    uint8_t* meta = kv ? meta1 : meta0;
    constexpr int L = G / 16;                     // lanes per group
    constexpr float kLevels = float((1 << B) - 1);
    const int lane = threadIdx.x & 31;
    const int part = lane & (L - 1);
    const int64_t warp0 = (int64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int64_t nwarps = (int64_t(gridDim.x) * kThreads) >> 5;
    for (int64_t wg = warp0 * (32 / L); wg < groups; wg += nwarps * (32 / L)) {   // warp-uniform loop
        const int64_t g = wg + lane / L;
        const bool valid = g < groups;
        uint4 va = make_uint4(0, 0, 0, 0), vb = va;
        if (valid) {
            const __half* p = x + g * G + part * 16;
            va = ld_stream(p);
            vb = ld_stream(p + 8);
        }
        const __half2 h[8] = {u2h(va.x), u2h(va.y), u2h(va.z), u2h(va.w),
                              u2h(vb.x), u2h(vb.y), u2h(vb.z), u2h(vb.w)};
        __half2 lo2 = __hmin2(__hmin2(__hmin2(h[0], h[1]), __hmin2(h[2], h[3])),
                              __hmin2(__hmin2(h[4], h[5]), __hmin2(h[6], h[7])));
        __half2 hi2 = __hmax2(__hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])),
                              __hmax2(__hmax2(h[4], h[5]), __hmax2(h[6], h[7])));
        __half2 mm = __halves2half2(__hmin(__low2half(lo2), __high2half(lo2)),
                                    __hmax(__low2half(hi2), __high2half(hi2)));   // (min, max), exact
#pragma unroll
        for (int o = 1; o < L; o <<= 1) {
            const __half2 t = u2h(__shfl_xor_sync(0xffffffffu, h2u(mm), o));
            mm = __halves2half2(__hmin(__low2half(mm), __low2half(t)), __hmax(__high2half(mm), __high2half(t)));
        }
        if (!valid) continue;
        float mn = __low2float(mm);
        const float mx = __high2float(mm);
        mn = (mn == 0.0f) ? 0.0f : mn;            // reading P
        const float r = __fsub_rn(mx, mn);        // RN32(max - min)
        uint64_t plo = 0, phi = 0;
        __half scale16 = __float2half_rn(0.0f);
        if (r != 0.0f) {                          // reading C
            // RN(r / (2^b - 1)) by one Markstein step on RN(1 / (2^b - 1)): equal to the IEEE quotient
            // for every fp32 r in the operand range and b in {2, 3, 4, 8} (tests/test_division.py)
            constexpr float kInvLevels = 1.0f / kLevels;
            const float s0 = __fmul_rn(r, kInvLevels);
            scale16 = __float2half_rn(__fmaf_rn(__fmaf_rn(-s0, kLevels, r), kInvLevels, s0));
            const float y = __frcp_rn(r);
            const float2 nmn = make_float2(-mn, -mn), yy = make_float2(y, y), nr = make_float2(-r, -r);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                // the b = 4 kernel's packed sequence: a, q0, e, u two elements at a time (each a single
                // rounding, no two of them contractible); t and the magic add stay scalar (a packed
                // mul + add pair is contracted into one FFMA2 by ptxas, see codes8)
                const float2 a = __fadd2_rn(__half22float2(h[j]), nmn);   // RN(x - min)
                const float2 q0 = __fmul2_rn(a, yy);
                const float2 er = __ffma2_rn(q0, nr, a);                  // exact
                const float2 u = __ffma2_rn(er, yy, q0);                  // RN(a / r)  (Markstein)
                const float us[2] = {u.x, u.y};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float t = __fmul_rn(us[e], kLevels);                  // RN(u (2^b - 1))
                    const uint32_t c = __float_as_uint(__fadd_rn(t, 8388608.0f)) & 0xFFu;   // RNE(t)
                    const int idx = 2 * j + e;
                    if (B * idx < 64)
                        plo |= uint64_t(c) << (B * idx);
                    else
                        phi |= uint64_t(c) << (B * idx - 64);
                }
            }
        }
        int64_t co, mo;
        dst(g, part, co, mo);
        store_bits<B>(codes + co, plo, phi);
        if (part == 0) *reinterpret_cast<__half2*>(meta + mo) = __halves2half2(scale16, __float2half_rn(mn));
    }
}

// out = f16(clamp(fmaf(code, scale, min), +-65504))   (O7, any b)
template <int B, int G>
__global__ void __launch_bounds__(kThreads)
dequantize_generic_kernel(const uint8_t* __restrict__ codes, const __half2* __restrict__ meta,
                          __half* __restrict__ out, int64_t groups) {
    constexpr int L = G / 16;
    const int64_t nthr = int64_t(gridDim.x) * kThreads;
    for (int64_t t = int64_t(blockIdx.x) * kThreads + threadIdx.x; t < groups * L; t += nthr) {
        const int64_t g = t / L;
        const int part = int(t % L);
        const uint8_t* p = codes + (g * G + part * 16) * B / 8;
        uint64_t lo = 0, hi = 0;
        if constexpr (B == 2) {
            lo = *reinterpret_cast<const uint32_t*>(p);
        } else if constexpr (B == 3) {
            const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
            lo = uint64_t(q[0]) | (uint64_t(q[1]) << 16) | (uint64_t(q[2]) << 32);
        } else if constexpr (B == 4) {
            lo = *reinterpret_cast<const uint64_t*>(p);
        } else {
            const uint4 v = *reinterpret_cast<const uint4*>(p);
            lo = uint64_t(v.x) | (uint64_t(v.y) << 32);
            hi = uint64_t(v.z) | (uint64_t(v.w) << 32);
        }
        const float2 sm = __half22float2(meta[g]);
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float v[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int idx = 2 * j + e;
                const uint32_t c = uint32_t((B * idx < 64 ? (lo >> (B * idx)) : (hi >> (B * idx - 64))) &
                                            ((1u << B) - 1u));
                v[e] = __fmaf_rn(float(c), sm.x, sm.y);
            }
            o[j] = sat_pack(v[0], v[1]);
        }
        uint4* dst = reinterpret_cast<uint4*>(out + g * G + part * 16);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

int num_sms() { return device_sm_count(); }

}  // namespace

template <int B, int G>
cudaError_t launch_quantize_bg(const void* x, int64_t groups, void* codes, void* meta, cudaStream_t stream) {
    int64_t blocks = (groups * (G / 16) + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    uint8_t* c = static_cast<uint8_t*>(codes);
    uint8_t* m = static_cast<uint8_t*>(meta);
    quantize_generic_kernel<B, G, PlainBitsDst<B, G>><<<unsigned(blocks), kThreads, 0, stream>>>(
        static_cast<const __half*>(x), nullptr, c, m, nullptr, nullptr, groups, PlainBitsDst<B, G>{});
    return cudaGetLastError();
}
template <int B, int G>
cudaError_t launch_append_kv_bg(const void* k, const void* v, int64_t rows, int head_dim, void* k_cache,
                                void* v_cache, KvDst d, cudaStream_t stream) {
    const int64_t groups = rows * (head_dim / G);
    int64_t blocks = (groups * (G / 16) + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    int gl = 0;
    while ((G << gl) < head_dim) ++gl;
    const KvBitsDst<B, G> dst{d.pos, d.chunks, FastDiv::make(uint32_t(d.n_new)), gl, head_dim * B / 8,
                              4 * head_dim / G};
    uint8_t* kc = static_cast<uint8_t*>(k_cache);
    uint8_t* vc = static_cast<uint8_t*>(v_cache);
    quantize_generic_kernel<B, G, KvBitsDst<B, G>><<<dim3(unsigned(blocks), 2u), kThreads, 0, stream>>>(
        static_cast<const __half*>(k), static_cast<const __half*>(v), kc, kc, vc, vc, groups, dst);
    return cudaGetLastError();
}
template <int B, int G>
cudaError_t launch_dequantize_bg(const void* codes, const void* meta, int64_t groups, void* out,
                                 cudaStream_t stream) {
    int64_t blocks = (groups * (G / 16) + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    dequantize_generic_kernel<B, G><<<unsigned(blocks), kThreads, 0, stream>>>(
        static_cast<const uint8_t*>(codes), static_cast<const __half2*>(meta), static_cast<__half*>(out), groups);
    return cudaGetLastError();
}

#define FLEXQ_BG_SWITCH(bits, group, CALL)                                                         \
    switch (bits * 1000 + group) {                                                                 \
        case 2032: return CALL(2, 32); case 2064: return CALL(2, 64); case 2128: return CALL(2, 128); \
        case 3032: return CALL(3, 32); case 3064: return CALL(3, 64); case 3128: return CALL(3, 128); \
        case 4032: return CALL(4, 32); case 4128: return CALL(4, 128);                             \
        case 8032: return CALL(8, 32); case 8064: return CALL(8, 64); case 8128: return CALL(8, 128); \
        default: return cudaErrorInvalidValue;                                                     \
    }

cudaError_t launch_quantize(const void* x, int64_t rows, int64_t cols, int bits, int group, void* codes, void* meta,
                            cudaStream_t stream) {
    if (bits != kBits || group != kGroup) {
        const int64_t groups = rows * (cols / group);
        if (groups == 0) return cudaSuccess;
#define Q_CALL(b, g) launch_quantize_bg<b, g>(x, groups, codes, meta, stream)
        FLEXQ_BG_SWITCH(bits, group, Q_CALL)
#undef Q_CALL
    }
    const int64_t groups = rows * (cols / kGroup);
    if (groups == 0) return cudaSuccess;
    int64_t blocks = (groups * 4 + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    quantize_kernel<PlainDst><<<unsigned(blocks), kThreads, 0, stream>>>(
        static_cast<const __half*>(x), nullptr, static_cast<uint8_t*>(codes), static_cast<uint8_t*>(meta), nullptr,
        nullptr, rows, cols, PlainDst{});
    return cudaGetLastError();
}

cudaError_t launch_append_kv(const void* k, const void* v, int64_t rows, int head_dim, int bits, int group,
                             void* k_cache, void* v_cache, KvDst d, cudaStream_t stream, bool v_tm) {
    if (rows == 0) return cudaSuccess;
    if (bits != kBits || group != kGroup) {
#define A_CALL(b, g) launch_append_kv_bg<b, g>(k, v, rows, head_dim, k_cache, v_cache, d, stream)
        FLEXQ_BG_SWITCH(bits, group, A_CALL)
#undef A_CALL
    }
    const int64_t groups = rows * (head_dim / kGroup);
    int64_t blocks = (groups * 4 + kThreads - 1) / kThreads;
    const int64_t cap = int64_t(num_sms()) * 8;
    if (blocks > cap) blocks = cap;
    dim3 grid(unsigned(blocks), 2u);
    quantize_kernel<KvChunkDst><<<grid, kThreads, 0, stream>>>(
        static_cast<const __half*>(k), static_cast<const __half*>(v), static_cast<uint8_t*>(k_cache),
        static_cast<uint8_t*>(k_cache), static_cast<uint8_t*>(v_cache), static_cast<uint8_t*>(v_cache), rows,
        head_dim, KvChunkDst{d, FastDiv::make(uint32_t(d.n_new)), head_dim == 128 ? 1 : 0, head_dim / 2, v_tm ? 1 : 0});
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const void* codes, const void* meta, int64_t rows, int64_t cols, int bits, int group,
                              void* out, cudaStream_t stream) {
    if (bits != kBits || group != kGroup) {
        const int64_t groups = rows * (cols / group);
        if (groups == 0) return cudaSuccess;
#define D_CALL(b, g) launch_dequantize_bg<b, g>(codes, meta, groups, out, stream)
        FLEXQ_BG_SWITCH(bits, group, D_CALL)
#undef D_CALL
    }
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

// attn_common.cuh -- shared pieces of the decode-attention kernels (dense and
// Top-K sparse): stage geometry of the chunked KV cache, PTX helpers (mbarrier,
// 1-D TMA bulk copy), the nibble -> float unpack, and the per-iteration K-score
// and P.V bodies.  See decode_attention.cu for the design notes.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

// One stage = NCH consecutive 32-token chunks of one cache (K or V); its smem
// image has the HBM layout: per chunk [codes 32 x D/2][meta 32 x D/16].
template <int D, int NCH>
struct Cfg {
    static constexpr int LPT = D / 32;                 // lanes per token
    static constexpr int TPI = 32 / LPT;               // tokens per warp iteration
    static constexpr int CH = kChunk * NCH;            // tokens per stage
    static constexpr int CB = D / 2;                   // code bytes per token
    static constexpr int MB = D / 16;                  // meta bytes per token (D/64 half2)
    static constexpr int ITERS = CH / TPI;
    static constexpr int CHB = kChunk * (CB + MB);     // chunk bytes (18 D)
    static constexpr int OFF_M = kChunk * CB;          // meta inside a chunk
    static constexpr int OFF_Q = NCH * CHB;
    static constexpr int OFF_NEW = OFF_Q + 2 * D;      // fused append: k_new, v_new rows (fp16)
    static constexpr int STAGE = OFF_NEW + 4 * D;      // + q [+ k_new, v_new] for the unit's first stage
    static constexpr int CPL_WORDS = D / 64;           // V pass: column-pair words per lane per quad
    static_assert(STAGE % 16 == 0 && CHB % 16 == 0, "stage alignment");
    static_assert(kChunk % TPI == 0, "an iteration stays inside one chunk");
    // byte offsets of iteration i's codes / meta rows (token slot 0 of the iteration)
    static constexpr int code_off(int i) { return (i * TPI / kChunk) * CHB + (i * TPI % kChunk) * CB; }
    static constexpr int meta_off(int i) { return (i * TPI / kChunk) * CHB + OFF_M + (i * TPI % kChunk) * MB; }
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 1-D TMA bulk store shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
    return *reinterpret_cast<const uint4*>(p);
}

#ifndef FLEXQ_H16_UNPACK
#define FLEXQ_H16_UNPACK 0
#endif

// Nibble -> float conversion of one 32-bit code word (8 codes, columns e = 0..7
// of the word).  Two implementations (FLEXQ_H16_UNPACK):
//  1: fp16 magic.  (w & 0x000F000F) | 0x64006400 is the half2
//    (1024 + c0, 1024 + c4) in ONE LOP3 for two codes; the mixed-precision
//    add.rn.f32.f16 (SASS FHADD, FMA pipe) subtracts 1024 exactly while widening
//    to fp32.  Pairs: f[0] = (c0, c4), f[1] = 16 (c1, c5), f[2] = (c2, c6),
//    f[3] = 16 (c3, c7)  (w >> 8 supplies c2, c3, c6, c7).
//  0 (default): fp32 magic.  (w & 0xF<<4e) | 0x4B000000 = 2^23 + c_e 16^e (one LOP3 per
//    code, e = 5..7 from w >> 12), one FADD2 removes 2^23 per pair.
//    Pairs: f[0] = (c0, 16 c1), f[1] = (256 c2, 4096 c3), f[2] = (65536 c4, 256 c5),
//    f[3] = (4096 c6, 65536 c7).
// Either way the value is exact; the power-of-two factor is folded into q on
// the K side and removed once per unit on the V side (inv_shift).  The magic
// constant lives in a register so that (w & mask) | magic is a single LOP3.
__device__ __forceinline__ uint32_t magic_reg() {
    uint32_t m;
#if FLEXQ_H16_UNPACK
    asm volatile("mov.b32 %0, 0x64006400;" : "=r"(m));
#else
    asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(m));
#endif
    return m;
}
template <uint32_t M>
__device__ __forceinline__ uint32_t lop_and_or(uint32_t w, uint32_t magic) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(M), "r"(magic));  // (a & b) | c
    return r;
}
__device__ __forceinline__ float2 fhadd2(uint32_t h2, float b) {   // (f32(h.lo) + b, f32(h.hi) + b)
    unsigned short lo, hi;
    asm("mov.b32 {%0,%1}, %2;" : "=h"(lo), "=h"(hi) : "r"(h2));
    float x, y;
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(x) : "h"(lo), "f"(b));
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(y) : "h"(hi), "f"(b));
    return make_float2(x, y);
}
// -1024.0f held in a register (FHADD has no immediate form; a compile-time
// constant gets re-materialised with a MOV before every FHADD).
__device__ __forceinline__ float neg1024_reg() {
    float r;
    asm volatile("mov.b32 %0, 0xC4800000;" : "=f"(r));
    return r;
}
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t magic, float2 (&f)[4]) {
#if FLEXQ_H16_UNPACK
    const uint32_t w8 = w >> 8;
    float nb;   // -1024 (register); passed through an empty asm so it is not re-materialised
    asm("mov.b32 %0, %1;" : "=f"(nb) : "r"(magic ^ 0x64006400u ^ 0xC4800000u));
    f[0] = fhadd2(lop_and_or<0x000F000Fu>(w, magic), nb);    // (c0, c4)
    f[1] = fhadd2(lop_and_or<0x00F000F0u>(w, magic), nb);    // 16 (c1, c5)
    f[2] = fhadd2(lop_and_or<0x000F000Fu>(w8, magic), nb);   // (c2, c6)
    f[3] = fhadd2(lop_and_or<0x00F000F0u>(w8, magic), nb);   // 16 (c3, c7)
#else
    const uint32_t w12 = w >> 12;
    const float2 bias = make_float2(-8388608.0f, -8388608.0f);
    f[0] = __fadd2_rn(make_float2(__uint_as_float(lop_and_or<0x0000Fu>(w, magic)),
                                  __uint_as_float(lop_and_or<0x000F0u>(w, magic))), bias);
    f[1] = __fadd2_rn(make_float2(__uint_as_float(lop_and_or<0x00F00u>(w, magic)),
                                  __uint_as_float(lop_and_or<0x0F000u>(w, magic))), bias);
    f[2] = __fadd2_rn(make_float2(__uint_as_float(lop_and_or<0xF0000u>(w, magic)),
                                  __uint_as_float(lop_and_or<0x00F00u>(w12, magic))), bias);
    f[3] = __fadd2_rn(make_float2(__uint_as_float(lop_and_or<0x0F000u>(w12, magic)),
                                  __uint_as_float(lop_and_or<0xF0000u>(w12, magic))), bias);
#endif
}
// 2^-k of the two codes of pair p (order of unpack8).
__device__ __forceinline__ float2 inv_shift(int pair) {
#if FLEXQ_H16_UNPACK
    return (pair & 1) ? make_float2(0.0625f, 0.0625f) : make_float2(1.0f, 1.0f);
#else
    switch (pair) {
        case 0: return make_float2(1.0f, 0.0625f);
        case 1: return make_float2(0.00390625f, 0.000244140625f);
        case 2: return make_float2(1.52587890625e-05f, 0.00390625f);
        default: return make_float2(0.000244140625f, 1.52587890625e-05f);
    }
#endif
}
// Word-local column of element h (0 = .x, 1 = .y) of pair p (order of unpack8).
__host__ __device__ constexpr int pair_col(int p, int h) {
#if FLEXQ_H16_UNPACK
    return p + 4 * h;
#else
    return 2 * p + h;
#endif
}

struct Params {
    const __half* q;
    const uint8_t* kc;   // chunked K cache
    const uint8_t* vc;   // chunked V cache
    __half* out;
    uint32_t* ctrl;      // [0] next ticket, [1] finished warps
    uint32_t* tickets;   // per (b, h): finished splits
    float* part;         // [unit][D] partial numerators
    float2* ml;          // [unit] (m, l)
    int bh_total, chunks, cur_len, nsplit, split_len;
    float qscale;        // log2(e) / sqrt(D)
    const __half* k_new; // fused append (NEXT-3): token cur_len - 1 of every (b, h), [B H][D];
    const __half* v_new; //   nullptr = the cache already holds it
    uint8_t* kc_w;       // writable aliases of kc / vc for the fused append
    uint8_t* vc_w;
};

#ifndef FLEXQ_K_IDP4A
#define FLEXQ_K_IDP4A 1
#endif

// The lane's view of q for pass 1 (FLEXQ_K_IDP4A):
//  0: qp[4w + p] = q * qscale * 2^-k at the columns of pair p of word w
//     (unpack8 order), qsum = sum q * qscale; the dot product runs on FFMA2.
//  1 (default): q as a 24-bit fixed-point integer per lane (scale 2^(23 - e), |q| < 2^e),
//     split into three byte limbs packed to match the codes' lo / hi nibbles;
//     the dot product runs on IDP.4A (exact in int32; q values within 2^-14 of
//     the lane's max are represented exactly, smaller ones to 2^-23 of the max).
struct KQuery {
#if FLEXQ_K_IDP4A
    uint32_t lo[3][4], hi[3][4];   // limb L of the q bytes at the lo / hi nibble columns of word w
    float pscale;                  // qscale * 2^(e - 23)
#else
    float2 qp[16];
#endif
    float qsum;                    // sum of q * qscale over the lane's 32 columns
};

__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
    int r;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// q (fp16, 64 B of the lane's 32 columns at qs) -> KQuery.
__device__ __forceinline__ void load_q(const uint8_t* qs, float qscale, KQuery& kq) {
    const __half* qh = reinterpret_cast<const __half*>(qs);
#if FLEXQ_K_IDP4A
    float q[32], mx = 0.0f, sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        q[j] = __half2float(qh[j]);
        mx = fmaxf(mx, fabsf(q[j]));
        sum += q[j];
    }
    int e = 0;
    frexpf(mx, &e);                                   // mx < 2^e (mx = 0 -> e = 0)
    const float up = ldexpf(1.0f, 23 - e);
    kq.pscale = qscale * ldexpf(1.0f, e - 23);
    kq.qsum = sum * qscale;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int L = 0; L < 3; ++L) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int ql = __float2int_rn(q[8 * w + 2 * b] * up);       // exact scaling, |.| < 2^23
                const int qh2 = __float2int_rn(q[8 * w + 2 * b + 1] * up);
                const uint32_t bl = uint32_t(ql >> (8 * L)) & 0xFFu;         // limb 2 keeps the sign byte
                const uint32_t bh = uint32_t(qh2 >> (8 * L)) & 0xFFu;
                lo |= bl << (8 * b);
                hi |= bh << (8 * b);
            }
            kq.lo[L][w] = lo;
            kq.hi[L][w] = hi;
        }
    }
#else
    float acc = 0.0f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float x = __half2float(qh[8 * w + pair_col(p, 0)]) * qscale;
            const float y = __half2float(qh[8 * w + pair_col(p, 1)]) * qscale;
            acc += x + y;
            const float2 sh = inv_shift(p);
            kq.qp[4 * w + p] = make_float2(x * sh.x, y * sh.y);
        }
    }
    kq.qsum = acc;
#endif
}

// Pass 1, one warp iteration (tokens i*TPI + [0, TPI) of the stage): scores -> smem (log2 domain).
// lc / lm: the lane's byte offsets inside a token row (codes / meta).
template <int D, int NCH, bool FULL>
__device__ __forceinline__ void k_iter(int i, const KQuery& kq, const uint8_t* sb, float* sc, int t0, int tl,
                                       int n, int lc, int lm, int sg, uint32_t magic, float& mx) {
    using C = Cfg<D, NCH>;
    const int tok = i * C::TPI + tl;
    const uint4 kw = lds128(sb + C::code_off(i) + lc);
    const float2 km = __half22float2(*reinterpret_cast<const __half2*>(sb + C::meta_off(i) + lm));
#if FLEXQ_K_IDP4A
    const uint32_t wv[4] = {kw.x, kw.y, kw.z, kw.w};
    uint32_t a0 = 0, a1 = 0;
    int a2 = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const uint32_t lo = wv[w] & 0x0F0F0F0Fu;         // codes of columns 0, 2, 4, 6 as bytes
        const uint32_t hi = (wv[w] >> 4) & 0x0F0F0F0Fu;  // columns 1, 3, 5, 7
        a0 = dp4a_uu(lo, kq.lo[0][w], a0);
        a0 = dp4a_uu(hi, kq.hi[0][w], a0);
        a1 = dp4a_uu(lo, kq.lo[1][w], a1);
        a1 = dp4a_uu(hi, kq.hi[1][w], a1);
        a2 = dp4a_us(lo, kq.lo[2][w], a2);
        a2 = dp4a_us(hi, kq.hi[2][w], a2);
    }
    const float P = fmaf(float(a2), 65536.0f, fmaf(float(a1), 256.0f, float(a0)));
    float s = fmaf(km.x, P * kq.pscale, km.y * kq.qsum);
    (void)magic;
#else
    float2 d0 = make_float2(0.0f, 0.0f), d1 = d0;
    float2 f[4];
    unpack8(kw.x, magic, f);
    d0 = __ffma2_rn(kq.qp[0], f[0], d0); d1 = __ffma2_rn(kq.qp[1], f[1], d1);
    d0 = __ffma2_rn(kq.qp[2], f[2], d0); d1 = __ffma2_rn(kq.qp[3], f[3], d1);
    unpack8(kw.y, magic, f);
    d0 = __ffma2_rn(kq.qp[4], f[0], d0); d1 = __ffma2_rn(kq.qp[5], f[1], d1);
    d0 = __ffma2_rn(kq.qp[6], f[2], d0); d1 = __ffma2_rn(kq.qp[7], f[3], d1);
    unpack8(kw.z, magic, f);
    d0 = __ffma2_rn(kq.qp[8], f[0], d0); d1 = __ffma2_rn(kq.qp[9], f[1], d1);
    d0 = __ffma2_rn(kq.qp[10], f[2], d0); d1 = __ffma2_rn(kq.qp[11], f[3], d1);
    unpack8(kw.w, magic, f);
    d0 = __ffma2_rn(kq.qp[12], f[0], d0); d1 = __ffma2_rn(kq.qp[13], f[1], d1);
    d0 = __ffma2_rn(kq.qp[14], f[2], d0); d1 = __ffma2_rn(kq.qp[15], f[3], d1);
    d0 = __fadd2_rn(d0, d1);
    float s = fmaf(km.x, d0.x + d0.y, km.y * kq.qsum);
#endif
#pragma unroll
    for (int o = 1; o < C::LPT; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (FULL || tok < n) {
        mx = fmaxf(mx, s);
        if (sg == 0) sc[t0 + tok] = s;
    }
}

// ---------------------------------------------------------------- pass 1 on the tensor cores
// FLEXQ_K_MMA=1 (default): the scores of 16 tokens at a time as one integer
// matrix product on IMMA (mma.sync m16n8k32, u8 codes x s8 q digits, exact
// int32 accumulation):
//   A (16 x 32, u8)  = the codes of 16 tokens (rows) x 32 elements (k), straight
//                      from the smem stage: a code word's low nibbles (w & 0x0F0F0F0F)
//                      and high nibbles ((w >> 4) & 0x0F0F0F0F) are 4 bytes of A each;
//   B (32 x 8, s8)   = q as a 23-bit fixed-point integer per 64-element group
//                      (scale 2^(22 - E_g), |q| < 2^E_g), split into three signed
//                      base-256 digits; column n = (digit, group) (3 G columns used);
//   C (16 x 8, s32)  = per token, the dot products of its codes with each digit
//                      of each group's q.
// The element order along k is any permutation applied to both operands alike
// (a dot product does not care): k-step s, lane quad-index j covers the word
// w = j KS + s of the token row, k positions 4j..4j+3 its even columns,
// 16+4j..16+4j+3 its odd columns.  Epilogue per token (each lane holds two C
// columns of two tokens; a 2-step quad reduction adds them up):
//   score = sum_g scale_g * 2^(E_g - 22) qscale * (C_g0 + 2^8 C_g1 + 2^16 C_g2)
//           + sum_g min_g * qscale * sum_{j in g} q_j              (log2 domain).
// Column map: D = 128: n = 0..5 -> (d0,g0) (d1,g0) (d2,g0) (d2,g1) (d0,g1) (d1,g1);
// D = 64: n = 0..2 -> d0, d1, d2.  So lane tig 0 and 2 combine their two columns
// in int32 (C_d0 + 2^8 C_d1 < 2^31), tig 1 holds the two d2 columns, tig 3
// (zero columns) adds the min term.
#ifndef FLEXQ_K_MMA
#define FLEXQ_K_MMA 1
#endif

__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>
struct KFrag {
    static constexpr int KS = D / 32;   // k-steps per token row
    uint32_t b[KS][2];                  // B fragment (q digits of the lane's column)
    int k256;                           // 256: combine the lane's two C columns in int32
    float wA, wB, bA, bB;               // v = fma(x0, wA, bA) hA + fma(x1, wB, bB) hB
    int offA, offB;                     // byte offsets of hA / hB in the token's meta
};

// q (fp16 [D] at qs, smem) -> the lane's KFrag.
template <int D>
__device__ __forceinline__ void load_q_mma(const uint8_t* qs, float qscale, int lane, KFrag<D>& kf) {
    constexpr int KS = D / 32, G = D / 64, NE = 8 * KS;   // elements per lane
    constexpr int JG = 4 / G;                             // quad lanes per group
    const int n = lane >> 2, j = lane & 3;
    const __half* qh = reinterpret_cast<const __half*>(qs) + NE * j;   // words j KS .. j KS + KS - 1
    float q[NE], mx = 0.0f, sum = 0.0f;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
        q[i] = __half2float(qh[i]);
        mx = fmaxf(mx, fabsf(q[i]));
        sum += q[i];
    }
#pragma unroll
    for (int o = 1; o < JG; o <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    int e = 0;
    frexpf(mx, &e);                                      // mx < 2^e (mx = 0 -> e = 0)
    const float up = ldexpf(1.0f, 22 - e);   // |Q| < 2^22: the signed top digit stays in [-64, 64]
    const int gl = j / JG;                               // the group of the lane's words
    // column n of B: digit n % 3 of group n / 3 (D = 128: n = 3 is (d2, g1), 4 / 5 are d0 / d1 of g1)
    int dig = -1, grp = -1;
    if (G == 2) {
        dig = n < 3 ? n : (n == 3 ? 2 : (n == 4 ? 0 : (n == 5 ? 1 : -1)));
        grp = n < 3 ? 0 : (n < 6 ? 1 : -1);
    } else if (n < 3) {
        dig = n;
        grp = 0;
    }
    const bool live = dig >= 0 && grp == gl;
#pragma unroll
    for (int s = 0; s < KS; ++s) {
        uint32_t b0 = 0, b1 = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int Q0 = __float2int_rn(q[8 * s + 2 * i] * up);       // exact scaling, |Q| < 2^22
            const int Q1 = __float2int_rn(q[8 * s + 2 * i + 1] * up);
            // signed base-256 digits: Q = d0 + 2^8 d1 + 2^16 d2, each in [-128, 127]
            const int a0 = (Q0 << 24) >> 24, r0 = (Q0 - a0) >> 8, a1 = (r0 << 24) >> 24, a2 = (r0 - a1) >> 8;
            const int c0 = (Q1 << 24) >> 24, r1 = (Q1 - c0) >> 8, c1 = (r1 << 24) >> 24, c2 = (r1 - c1) >> 8;
            const int x = dig == 0 ? a0 : (dig == 1 ? a1 : a2);
            const int y = dig == 0 ? c0 : (dig == 1 ? c1 : c2);
            b0 |= (uint32_t(x) & 0xFFu) << (8 * i);
            b1 |= (uint32_t(y) & 0xFFu) << (8 * i);
        }
        kf.b[s][0] = live ? b0 : 0u;
        kf.b[s][1] = live ? b1 : 0u;
    }
    // per-group weights from the quad lanes that own each group
    const float w_l = qscale * ldexpf(1.0f, e - 22);   // this lane's group weight
    const float s_l = sum * qscale;
    const float w0 = __shfl_sync(0xffffffffu, w_l, lane & ~3);
    const float s0 = __shfl_sync(0xffffffffu, s_l, lane & ~3);
    const float w1 = __shfl_sync(0xffffffffu, w_l, (lane & ~3) | 2);
    const float s1 = __shfl_sync(0xffffffffu, s_l, (lane & ~3) | 2);
    kf.wA = kf.wB = kf.bA = kf.bB = 0.0f;
    kf.k256 = 0;
    kf.offA = 0;
    kf.offB = 2;
    if (G == 2) {
        if (j == 0) { kf.k256 = 256; kf.wA = w0; kf.offA = 0; }
        if (j == 1) { kf.wA = w0 * 65536.0f; kf.offA = 0; kf.wB = w1 * 65536.0f; kf.offB = 4; }
        if (j == 2) { kf.k256 = 256; kf.wA = w1; kf.offA = 4; }
        if (j == 3) { kf.bA = s0; kf.offA = 2; kf.bB = s1; kf.offB = 6; }
    } else {
        if (j == 0) { kf.k256 = 256; kf.wA = w0; kf.offA = 0; }
        if (j == 1) { kf.wA = w0 * 65536.0f; kf.offA = 0; }
        if (j == 3) { kf.bA = s0; kf.offA = 2; }
    }
}

// Pass 1, one 16-token block `blk` of the stage (tokens 16 blk + [0, 16)): scores -> smem.
template <int D, int NCH>
__device__ __forceinline__ void k_block_mma(int blk, const KFrag<D>& kf, const uint8_t* sb, float* sc, int t0,
                                            int n, int lane, float& mx) {
    using C = Cfg<D, NCH>;
    constexpr int KS = D / 32;
    const int r = lane >> 2, j = lane & 3;
    const int tok = blk * 16 + r;                       // stage-relative token of row r (row r + 8: tok + 8)
    const uint8_t* ch = sb + (tok >> 5) * C::CHB;       // a 16-token block never straddles a chunk
    const int slot = tok & 31;
    const uint8_t* cr = ch + slot * C::CB + j * (4 * KS);
    uint32_t w0[KS], w8[KS];
    if constexpr (KS == 4) {
        const uint4 x = lds128(cr), y = lds128(cr + 8 * C::CB);
        w0[0] = x.x; w0[1] = x.y; w0[2] = x.z; w0[3] = x.w;
        w8[0] = y.x; w8[1] = y.y; w8[2] = y.z; w8[3] = y.w;
    } else {
        const uint2 x = *reinterpret_cast<const uint2*>(cr), y = *reinterpret_cast<const uint2*>(cr + 8 * C::CB);
        w0[0] = x.x; w0[1] = x.y;
        w8[0] = y.x; w8[1] = y.y;
    }
    int c[4] = {0, 0, 0, 0};
#pragma unroll
    for (int s = 0; s < KS; ++s)
        mma_u8s8(c, w0[s] & 0x0F0F0F0Fu, w8[s] & 0x0F0F0F0Fu, (w0[s] >> 4) & 0x0F0F0F0Fu,
                 (w8[s] >> 4) & 0x0F0F0F0Fu, kf.b[s][0], kf.b[s][1]);
    const uint8_t* mr = ch + C::OFF_M + slot * C::MB;
    const float hA0 = __half2float(*reinterpret_cast<const __half*>(mr + kf.offA));
    const float hB0 = __half2float(*reinterpret_cast<const __half*>(mr + kf.offB));
    const float hA8 = __half2float(*reinterpret_cast<const __half*>(mr + 8 * C::MB + kf.offA));
    const float hB8 = __half2float(*reinterpret_cast<const __half*>(mr + 8 * C::MB + kf.offB));
    float v0 = fmaf(fmaf(float(c[0] + kf.k256 * c[1]), kf.wA, kf.bA), hA0, fmaf(float(c[1]), kf.wB, kf.bB) * hB0);
    float v8 = fmaf(fmaf(float(c[2] + kf.k256 * c[3]), kf.wA, kf.bA), hA8, fmaf(float(c[3]), kf.wB, kf.bB) * hB8);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 1);
    v8 += __shfl_xor_sync(0xffffffffu, v8, 1);
    v0 += __shfl_xor_sync(0xffffffffu, v0, 2);
    v8 += __shfl_xor_sync(0xffffffffu, v8, 2);
    if (tok < n) {
        mx = fmaxf(mx, v0);
        if (j == 0) sc[t0 + tok] = v0;
    }
    if (tok + 8 < n) {
        mx = fmaxf(mx, v8);
        if (j == 1) sc[t0 + tok + 8] = v8;
    }
}

// acc_j += (p scale) c_j over the lane's 32 columns, bias += p min, l += p.
__device__ __forceinline__ void v_accum(float2 (&acc)[16], float& l, float& bsum, uint4 vw, float2 vm, float p,
                                        uint32_t magic) {
    l += p;
    const float a = p * vm.x;
    bsum = fmaf(p, vm.y, bsum);
    const float2 a2 = make_float2(a, a);
    float2 f[4];
    unpack8(vw.x, magic, f);
    acc[0] = __ffma2_rn(a2, f[0], acc[0]); acc[1] = __ffma2_rn(a2, f[1], acc[1]);
    acc[2] = __ffma2_rn(a2, f[2], acc[2]); acc[3] = __ffma2_rn(a2, f[3], acc[3]);
    unpack8(vw.y, magic, f);
    acc[4] = __ffma2_rn(a2, f[0], acc[4]); acc[5] = __ffma2_rn(a2, f[1], acc[5]);
    acc[6] = __ffma2_rn(a2, f[2], acc[6]); acc[7] = __ffma2_rn(a2, f[3], acc[7]);
    unpack8(vw.z, magic, f);
    acc[8] = __ffma2_rn(a2, f[0], acc[8]); acc[9] = __ffma2_rn(a2, f[1], acc[9]);
    acc[10] = __ffma2_rn(a2, f[2], acc[10]); acc[11] = __ffma2_rn(a2, f[3], acc[11]);
    unpack8(vw.w, magic, f);
    acc[12] = __ffma2_rn(a2, f[0], acc[12]); acc[13] = __ffma2_rn(a2, f[1], acc[13]);
    acc[14] = __ffma2_rn(a2, f[2], acc[14]); acc[15] = __ffma2_rn(a2, f[3], acc[15]);
}

// Pass 2, one warp iteration: acc_j += (p scale) c_j, bias += p min for TPI tokens.
template <int D, int NCH, bool FULL>
__device__ __forceinline__ void v_iter(int i, float2 (&acc)[16], float& l, float& bsum, const uint8_t* sb,
                                       const float* sc, float M, int t0, int tl, int n, int lc, int lm,
                                       uint32_t magic) {
    using C = Cfg<D, NCH>;
    const int tok = i * C::TPI + tl;
    const uint4 vw = lds128(sb + C::code_off(i) + lc);
    float2 vm = __half22float2(*reinterpret_cast<const __half2*>(sb + C::meta_off(i) + lm));
    float p = ex2(sc[t0 + tok] - M);
    if (!FULL) {
        const bool valid = tok < n;
        p = valid ? p : 0.0f;
        vm.x = valid ? vm.x : 0.0f;
        vm.y = valid ? vm.y : 0.0f;
    }
    v_accum(acc, l, bsum, vw, vm, p, magic);
}

// ---------------------------------------------------------------- pass 2 (dense): V
// V chunk codes are quad-interleaved (include/flexq.h): word (quad qd, column pair pj)
// holds, in byte k, token 4qd+k's codes of columns 2pj (low nibble) and 2pj+1 (high).
// So w & 0x0F0F0F0F is column 2pj of 4 tokens as bytes and (w >> 4) & 0x0F0F0F0F
// column 2pj+1: IDP.4A against the 4 tokens' weights needs no transposition.
// Lane l owns columns [CPL l, CPL (l+1)) (CPL = D/32; one quantization group).
// Per stage the weights a_t = p_t scale_tg of each group are turned into 24-bit
// fixed point against the stage's max (scale 2^(23-e)), split into 3 byte limbs
// (smem table [group][quad][limb]); int32 limb sums are flushed to fp32 per stage.
template <int D, int NCH>
constexpr int kLimbWords = (D / 64) * (NCH * kChunk / 4) * 4;   // [group][quad][4 words]

template <int D>
struct VAcc {
    static constexpr int CPL = D / 32;   // columns per lane
    float acc[CPL];                      // sum_t a_t c_tj, fp32
    float l, bsum[D / 64];               // the lane's tokens: sum p, sum p min_g
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = 0.0f;
        l = 0.0f;
#pragma unroll
        for (int g = 0; g < D / 64; ++g) bsum[g] = 0.0f;
    }
    // warp-reduce l and the lane's group bias; v[c] = acc + bias (unnormalised); returns col0
    __device__ __forceinline__ int finish(int lane, float (&v)[32], float& lsum) {
        float b[D / 64];
#pragma unroll
        for (int g = 0; g < D / 64; ++g) b[g] = bsum[g];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
            for (int g = 0; g < D / 64; ++g) b[g] += __shfl_xor_sync(0xffffffffu, b[g], o);
        }
        lsum = l;
        const int col0 = lane * CPL;
        const float bias = (D / 64 == 1 || col0 < 64) ? b[0] : b[D / 64 - 1];
#pragma unroll
        for (int c = 0; c < CPL; ++c) v[c] = acc[c] + bias;
        return col0;
    }
};

// Pass 2 stage pre-pass: weights a_tg = p_t scale_tg of the stage's tokens as
// 24-bit fixed point (scale 2^(23 - e_g), a < 2^e_g per group) in the limb
// table [group][quad][limb 0..2, pad][token byte]; l += p, bias_g += p min_g
// on the lane's tokens; inv[g] = 2^(e_g - 23).
template <int D, int NCH>
__device__ __forceinline__ void v_weights(float& l, float (&bsum)[D / 64], const uint8_t* sb, const float* sc, float M,
                                          int n, int lane, uint32_t* limbs, float (&inv)[D / 64]) {
    using C = Cfg<D, NCH>;
    constexpr int G = D / 64;           // groups per token
    constexpr int Q = C::CH / 4;        // quads per stage
    constexpr int TPL = C::CH / 32;     // tokens per lane in the weight pre-pass
    // ---- weights: lane handles tokens lane + 32 i of the stage
    float a[TPL][G];
    float amax[G];
#pragma unroll
    for (int g = 0; g < G; ++g) amax[g] = 0.0f;
#pragma unroll
    for (int i = 0; i < TPL; ++i) {
        const int t = lane + 32 * i;
        const bool valid = t < n;
        const float p = valid ? ex2(sc[t] - M) : 0.0f;
        l += p;
        const uint8_t* mrow = sb + (t / kChunk) * C::CHB + C::OFF_M + (t % kChunk) * C::MB;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float2 sm = __half22float2(*reinterpret_cast<const __half2*>(mrow + 4 * g));
            sm.x = valid ? sm.x : 0.0f;
            sm.y = valid ? sm.y : 0.0f;
            a[i][g] = p * sm.x;
            bsum[g] = fmaf(p, sm.y, bsum[g]);
            amax[g] = fmaxf(amax[g], a[i][g]);
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) amax[g] = fmaxf(amax[g], __shfl_xor_sync(0xffffffffu, amax[g], o));
        int e = 0;
        frexpf(amax[g], &e);                      // amax < 2^e (0 -> e = 0)
        const float up = ldexpf(1.0f, 23 - e);
        inv[g] = ldexpf(1.0f, e - 23);
        uint8_t* tb = reinterpret_cast<uint8_t*>(limbs + g * Q * 4);
#pragma unroll
        for (int i = 0; i < TPL; ++i) {
            const int t = lane + 32 * i;
            const uint32_t ai = uint32_t(__float2int_rn(a[i][g] * up));     // < 2^23, >= 0
            uint8_t* q = tb + (t >> 2) * 16 + (t & 3);                        // [quad][limb word][token byte]
            q[0] = uint8_t(ai);
            q[4] = uint8_t(ai >> 8);
            q[8] = uint8_t(ai >> 16);
        }
    }
    __syncwarp();
}

template <int D, int NCH>
__device__ __forceinline__ void v_stage(VAcc<D>& va, const uint8_t* sb, const float* sc, float M, int n, int lane,
                                        uint32_t* limbs) {
    using C = Cfg<D, NCH>;
    constexpr int G = D / 64;           // groups per token
    constexpr int Q = C::CH / 4;        // quads per stage
    float inv[G];
    v_weights<D, NCH>(va.l, va.bsum, sb, sc, M, n, lane, limbs, inv);
    // ---- IDP.4A over quads: lane's CPL columns = CPL/2 column-pair words per quad
    constexpr int W = C::CPL_WORDS;
    const int g = (lane * (D / 32)) / 64;
    uint32_t s0[2 * W], s1[2 * W], s2[2 * W];
#pragma unroll
    for (int c = 0; c < 2 * W; ++c) { s0[c] = 0u; s1[c] = 0u; s2[c] = 0u; }
    const uint32_t* lt = limbs + g * Q * 4;
#pragma unroll 4
    for (int qd = 0; qd < Q; ++qd) {
        const uint4 lm = *reinterpret_cast<const uint4*>(lt + qd * 4);       // limbs 0..2 (+ pad)
        const uint8_t* crow = sb + (qd / 8) * C::CHB + ((qd % 8) * C::CB + ((lane * W) ^ ((qd & 3) << 3))) * 4;
        uint32_t wv[W];
        if constexpr (W == 2) {
            const uint2 x = *reinterpret_cast<const uint2*>(crow);
            wv[0] = x.x;
            wv[W - 1] = x.y;
        } else {
            wv[0] = *reinterpret_cast<const uint32_t*>(crow);
        }
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const uint32_t lo = wv[w] & 0x0F0F0F0Fu;
            const uint32_t hi = (wv[w] >> 4) & 0x0F0F0F0Fu;
            s0[2 * w] = dp4a_uu(lo, lm.x, s0[2 * w]);
            s1[2 * w] = dp4a_uu(lo, lm.y, s1[2 * w]);
            s2[2 * w] = dp4a_uu(lo, lm.z, s2[2 * w]);
            s0[2 * w + 1] = dp4a_uu(hi, lm.x, s0[2 * w + 1]);
            s1[2 * w + 1] = dp4a_uu(hi, lm.y, s1[2 * w + 1]);
            s2[2 * w + 1] = dp4a_uu(hi, lm.z, s2[2 * w + 1]);
        }
    }
    // ---- flush: acc += (s2 2^16 + s1 2^8 + s0) * 2^(e - 23)
#pragma unroll
    for (int c = 0; c < 2 * W; ++c) {
        const float f = fmaf(float(s2[c]), 65536.0f, fmaf(float(s1[c]), 256.0f, float(s0[c])));
        va.acc[c] = fmaf(f, (G == 1 || g == 0) ? inv[0] : inv[G - 1], va.acc[c]);
    }
    __syncwarp();   // limb table reuse by the next stage
}

// ---------------------------------------------------------------- pass 2 on the tensor cores
// FLEXQ_V_MMA=1 (default): P.V of each 32-token k-step as IMMA m16n8k32 (u8 x u8,
// exact int32):
//   A (16 x 32) = V codes: row r <-> column 2 p (low nibbles, w & 0x0F0F0F0F),
//                 row r + 8 <-> column 2 p + 1 (high nibbles, w & 0xF0F0F0F0 = 16 c),
//                 p = PPL r + u for tile u; k <-> tokens: positions 4j..4j+3 are the
//                 4 tokens of quad 8s + j (one quad-interleaved word), 16+4j.. quad 8s+4+j;
//   B (32 x 8)  = the weight limbs a_tg (v_weights' table, one word per quad and limb);
//                 column n = (limb, group) as in pass 1's map;
//   C (16 x 8)  = per column, per (limb, group) partial sums; only the column's own
//                 group is kept.  Flushed to fp32 once per stage (the fixed-point scale
//                 is per stage); limbs and nibble positions are combined at the end of
//                 the unit, with a quad reduction.
#ifndef FLEXQ_V_MMA
#define FLEXQ_V_MMA 1
#endif

__device__ __forceinline__ void mma_u8u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>
struct VAccM {
    static constexpr int PPL = D / 16;   // tiles (column pairs per lane row)
    float acc[PPL][4];                   // fp32 partials of C, per tile / C register
    float l, bsum[D / 64];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int u = 0; u < PPL; ++u)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[u][i] = 0.0f;
        l = 0.0f;
#pragma unroll
        for (int g = 0; g < D / 64; ++g) bsum[g] = 0.0f;
    }
};

// pass 1's (limb, group) map of C column n (-1: unused)
template <int D>
__device__ __forceinline__ void col_role(int n, int& limb, int& grp) {
    if (D == 128) {
        limb = n < 3 ? n : (n == 3 ? 2 : (n == 4 ? 0 : (n == 5 ? 1 : -1)));
        grp = n < 3 ? 0 : (n < 6 ? 1 : -1);
    } else {
        limb = n < 3 ? n : -1;
        grp = n < 3 ? 0 : -1;
    }
}

// Fixed-point scale for a block of non-negative weights with maximum bit
// pattern mb: e = floor(log2(amax)) + 1 (amax < 2^e); up = 2^(23 - e),
// inv = 2^(e - 23), built from the exponent field (no frexpf / ldexpf slow
// paths).  amax < 2^-103 (or 0) gives up = inv = 0: such weights are below
// 2^-100 of the unit's largest p (= 1) and drop out.
__device__ __forceinline__ void fixed_scale(uint32_t mb, float& up, float& inv) {
    const int eb = int((mb >> 23) & 0xFFu);
    up = eb < 24 ? 0.0f : __int_as_float((276 - eb) << 23);
    inv = eb < 24 ? 0.0f : __int_as_float((eb - 22) << 23);
}

// Weight pre-pass of the MMA pass 2 (same table as v_weights): lane (quad qd,
// group g) computes the 4 weights of its quad, the per-group exponent comes
// from one REDUX max on the float bits (a >= 0, so the bit patterns order like
// the values), and the three limb words are assembled with PRMT and stored as
// one 16-byte row [limb0, limb1, limb2, 0] of the table.
template <int D, int NCH>
__device__ __forceinline__ void v_weights_quad(float& l, float (&bsum)[D / 64], const uint8_t* sb, const float* sc,
                                               float M, int n, int lane, uint32_t* limbs, float (&inv)[D / 64]) {
    using C = Cfg<D, NCH>;
    constexpr int G = D / 64, Q = C::CH / 4;
    static_assert(Q * G <= 32, "one (quad, group) per lane");
    const int qd = lane % Q, g = lane / Q;
    const bool act = g < G;
    const float4 s4 = *reinterpret_cast<const float4*>(sc + 4 * qd);
    const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
    float a[4], amax = 0.0f, ps = 0.0f, bs = 0.0f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int t = 4 * qd + k;
        const bool valid = act && t < n;
        const float p = valid ? ex2(sv[k] - M) : 0.0f;
        const float2 sm = __half22float2(*reinterpret_cast<const __half2*>(
            sb + (t / kChunk) * C::CHB + C::OFF_M + (t % kChunk) * C::MB + 4 * (act ? g : 0)));
        a[k] = valid ? p * sm.x : 0.0f;
        bs = valid ? fmaf(p, sm.y, bs) : bs;
        ps += p;
        amax = fmaxf(amax, a[k]);
    }
    if (g == 0) l += ps;                      // p is counted once (lanes of group 1 repeat the quad)
#pragma unroll
    for (int gg = 0; gg < G; ++gg) if (g == gg) bsum[gg] += bs;
    float up = 0.0f;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        const uint32_t mb = __reduce_max_sync(0xffffffffu, (g == gg) ? __float_as_uint(amax) : 0u);
        float u;
        fixed_scale(mb, u, inv[gg]);
        up = (g == gg) ? u : up;
    }
    if (act) {
        const uint32_t q0 = uint32_t(__float2int_rn(a[0] * up)), q1 = uint32_t(__float2int_rn(a[1] * up));
        const uint32_t q2 = uint32_t(__float2int_rn(a[2] * up)), q3 = uint32_t(__float2int_rn(a[3] * up));
        const uint32_t l01 = __byte_perm(q0, q1, 0x5140), l23 = __byte_perm(q2, q3, 0x5140);   // bytes 0, 1
        const uint32_t h01 = __byte_perm(q0, q1, 0x7362), h23 = __byte_perm(q2, q3, 0x7362);   // bytes 2, 3
        *reinterpret_cast<uint4*>(limbs + (g * Q + qd) * 4) =
            make_uint4(__byte_perm(l01, l23, 0x5410), __byte_perm(l01, l23, 0x7632), __byte_perm(h01, h23, 0x5410), 0u);
    }
    __syncwarp();
}

// The lane's fixed roles in pass 2 (computed once per kernel).
template <int D>
struct VLane {
    int tab;          // word offset of the lane's B column (limb, group) in a stage's limb table
    bool live;        // the lane's B column is used
    int g0, g1;       // group of the weights in C columns 2j, 2j+1 (-1: unused column)
    float w0, w1;     // end-of-unit limb weights of those columns (0: other group / unused)
    int gr;           // group of the lane row's output columns
    int hx;           // D = 128: byte XOR of the half-block order (16 for odd rows)
};
template <int D, int NCH>
__device__ __forceinline__ VLane<D> v_lane(int lane) {
    constexpr int Q = Cfg<D, NCH>::CH / 4, PPL = D / 16;
    const int r = lane >> 2, j = lane & 3;
    VLane<D> v;
    int limb, grp, l0, l1;
    col_role<D>(r, limb, grp);
    v.live = grp >= 0;
    v.tab = v.live ? grp * Q * 4 + limb : 0;
    col_role<D>(2 * j, l0, v.g0);
    col_role<D>(2 * j + 1, l1, v.g1);
    v.gr = (2 * PPL * r) / 64;
    v.w0 = (v.g0 == v.gr) ? float(1 << (8 * l0)) : 0.0f;
    v.w1 = (v.g1 == v.gr) ? float(1 << (8 * l1)) : 0.0f;
    v.hx = (D == 128 && (r & 1)) ? 16 : 0;
    return v;
}

template <int D, int NCH>
__device__ __forceinline__ void v_stage_mma(VAccM<D>& va, const VLane<D>& vl, const uint8_t* sb, const float* sc,
                                            float M, int n, int lane, uint32_t* limbs) {
    using C = Cfg<D, NCH>;
    constexpr int G = D / 64, PPL = D / 16;
    float inv[G];
    v_weights_quad<D, NCH>(va.l, va.bsum, sb, sc, M, n, lane, limbs, inv);
    const int r = lane >> 2, j = lane & 3;
    const uint32_t* lt = limbs + vl.tab;
    int c[PPL][4];
#pragma unroll
    for (int u = 0; u < PPL; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) c[u][i] = 0;
#pragma unroll
    for (int s = 0; s < C::CH / 32; ++s) {
        if (32 * s >= n) break;
        const uint32_t b0 = vl.live ? lt[(8 * s + j) * 4] : 0u;
        const uint32_t b1 = vl.live ? lt[(8 * s + 4 + j) * 4] : 0u;
        const uint8_t* ch = sb + s * C::CHB;      // quads 8s .. 8s + 7 = chunk s
        // the swizzled layout puts pair p of quad q at p ^ ((q & 3) << 3): quads j and 4 + j
        // share the swizzle j.  D = 128: the lane's 8 pairs (two 16-B halves) start at
        // 8 (r ^ j); odd rows read their upper half first (vl.hx = 16) so the 8 lanes of an
        // LDS.128 phase hit 8 distinct 16-B bank groups.  D = 64: 4 pairs at 4 (r ^ 2j).
        const int blk = D == 128 ? PPL * (r ^ j) : PPL * (r ^ (2 * j));
        const uint8_t* wa = ch + (j * C::CB + blk) * 4;
        const uint8_t* wb = ch + ((4 + j) * C::CB + blk) * 4;
        uint32_t xa[PPL], xb[PPL];
#pragma unroll
        for (int h = 0; h < PPL / 4; ++h) {
            const int off = (16 * h) ^ vl.hx;
            const uint4 ua = lds128(wa + off), ub = lds128(wb + off);
            xa[4 * h] = ua.x; xa[4 * h + 1] = ua.y; xa[4 * h + 2] = ua.z; xa[4 * h + 3] = ua.w;
            xb[4 * h] = ub.x; xb[4 * h + 1] = ub.y; xb[4 * h + 2] = ub.z; xb[4 * h + 3] = ub.w;
        }
#pragma unroll
        for (int u = 0; u < PPL; ++u)
            mma_u8u8(c[u], xa[u] & 0x0F0F0F0Fu, xa[u] & 0xF0F0F0F0u, xb[u] & 0x0F0F0F0Fu, xb[u] & 0xF0F0F0F0u, b0,
                     b1);
    }
    // flush: C column n = 2j + {0, 1} holds weights of group g0 / g1
    const float i0 = vl.g0 < 0 ? 0.0f : (vl.g0 == 0 ? inv[0] : inv[G - 1]);
    const float i1 = vl.g1 < 0 ? 0.0f : (vl.g1 == 0 ? inv[0] : inv[G - 1]);
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
        va.acc[u][0] = fmaf(float(c[u][0]), i0, va.acc[u][0]);
        va.acc[u][1] = fmaf(float(c[u][1]), i1, va.acc[u][1]);
        va.acc[u][2] = fmaf(float(c[u][2]), i0, va.acc[u][2]);
        va.acc[u][3] = fmaf(float(c[u][3]), i1, va.acc[u][3]);
    }
    __syncwarp();   // limb table reuse by the next stage
}

// End of a unit (MMA pass 2): combine limbs / nibble positions, quad-reduce, add the
// bias, normalise and write.  Lane (r, j) writes tiles u = j, j + 4, ... (columns
// 2 (PPL r + u), +1).
template <int D>
__device__ __forceinline__ void v_finish_mma(VAccM<D>& va, const VLane<D>& vl, int lane, __half* out_bh, float& lsum,
                                             float* v_part /* nullptr: normalise + write fp16 */) {
    constexpr int G = D / 64, PPL = D / 16;
    const int r = lane >> 2, j = lane & 3;
    float b[G];
#pragma unroll
    for (int g = 0; g < G; ++g) b[g] = va.bsum[g];
    float l = va.l;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
#pragma unroll
        for (int g = 0; g < G; ++g) b[g] += __shfl_xor_sync(0xffffffffu, b[g], o);
    }
    lsum = l;
    const float w0 = vl.w0, w1 = vl.w1;
    const float bias = vl.gr == 0 ? b[0] : b[G - 1];
    const float inv_l = 1.0f / l;
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
        float ev = fmaf(va.acc[u][0], w0, va.acc[u][1] * w1);                    // column 2p
        float od = fmaf(va.acc[u][2], w0, va.acc[u][3] * w1) * 0.0625f;         // column 2p+1 (16 c)
        ev += __shfl_xor_sync(0xffffffffu, ev, 1);
        od += __shfl_xor_sync(0xffffffffu, od, 1);
        ev += __shfl_xor_sync(0xffffffffu, ev, 2);
        od += __shfl_xor_sync(0xffffffffu, od, 2);
        if ((u & 3) == j) {
            const int col = 2 * (PPL * r + (u ^ (vl.hx >> 2)));   // tile u holds pair PPL r + (u ^ 4) on odd rows (D = 128)
            ev += bias;
            od += bias;
            if (v_part) {
                v_part[col] = ev;
                v_part[col + 1] = od;
            } else {
                *reinterpret_cast<__half2*>(out_bh + col) = __floats2half2_rn(ev * inv_l, od * inv_l);
            }
        }
    }
}

// End of a unit: remove the 16^k factors, reduce (acc, l, bsum) over the token
// lanes (reduce-scatter for acc: lane keeps D/32 columns), and return the
// lane's column offset col0; v[0 .. D/32) = sum_t (p scale) c + bias (unnormalised).
template <int D>
__device__ __forceinline__ int reduce_unit(float2 (&acc)[16], float& l, float& bsum, int lane, int sg,
                                           float (&v)[32]) {
    constexpr int LPT = D / 32;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = __fmul2_rn(acc[k], inv_shift(k & 3));
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) {
        l += __shfl_xor_sync(0xffffffffu, l, o);
        bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {   // natural column order: v[col] (static register renaming)
        v[8 * (k / 4) + pair_col(k & 3, 0)] = acc[k].x;
        v[8 * (k / 4) + pair_col(k & 3, 1)] = acc[k].y;
    }
    int width = 32;   // live entries
    int base = 0;     // column offset (within the 32-column segment) of v[0]
#pragma unroll
    for (int o = 16; o >= LPT; o >>= 1) {
        const bool upper = (lane & o) != 0;
        const int half = width >> 1;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (k < half) {
                const float send = upper ? v[k] : v[k + half];
                const float keep = upper ? v[k + half] : v[k];
                v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        if (upper) base += half;
        width = half;
    }
#pragma unroll
    for (int k = 0; k < D / 32; ++k) v[k] += bsum;
    return sg * 32 + base;
}

// out[col0 .. col0 + D/32) = v / l as fp16.
template <int D>
__device__ __forceinline__ void write_out(__half* dst, const float (&v)[32], float l) {
    const float inv = 1.0f / l;
    if constexpr (D == 128) {
        __half2 h0 = __floats2half2_rn(v[0] * inv, v[1] * inv);
        __half2 h1 = __floats2half2_rn(v[2] * inv, v[3] * inv);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&h0);
        w.y = *reinterpret_cast<uint32_t*>(&h1);
        *reinterpret_cast<uint2*>(dst) = w;
    } else {
        *reinterpret_cast<__half2*>(dst) = __floats2half2_rn(v[0] * inv, v[1] * inv);
    }
}

// ---------------------------------------------------------------- fused append (NEXT-3)
// Quantize the new token's K and V rows (D fp16 each, contiguous in shared
// memory: [k_new | v_new]) with one warp: lanes 0-15 take the K row, lanes
// 16-31 the V row, EL = D / 16 consecutive elements per lane, so a 64-element
// group spans GL = 64 / EL lanes.  The result stays in registers (TokenQ) and
// is stored in the chunked cache layout by store_token (once into the cache in
// HBM, once into the stage image in shared memory, so the attention reads the
// new token without a round trip).  Same quantizer as quant.cu, operation for
// operation (readings A-D, P): a = RN(x - min), u = RN(a / r)
// via the per-group reciprocal + Markstein correction, t = RN(15 u),
// code = RNE(t); scale = f16(RN(r / 15)) with RN(r / 15) by the same Markstein
// step on the constant reciprocal RN(1/15) (tests/test_division.py checks it
// against IEEE division for every fp32 r in the operand range).  Only scalar
// round-to-nearest intrinsics are used, which ptxas never contracts, so the
// bytes match quant.cu (compiled -fmad=false) exactly.
struct TokenQ {
    uint32_t codes;   // the lane's EL nibbles, element 2k in the low nibble of byte k
    uint32_t meta;    // half2 {scale, min} of the lane's group
};
template <int D>
__device__ __forceinline__ TokenQ quantize_kv_token(const uint8_t* rows, int lane) {
    constexpr int EL = D / 16;                 // elements per lane (8 or 4)
    constexpr int GL = kGroup / EL;            // lanes per group (8 or 16)
    __half2 h[EL / 2];
    if constexpr (EL == 8) {
        const uint4 w = *reinterpret_cast<const uint4*>(rows + lane * 16);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = *reinterpret_cast<const __half2*>(&ws[i]);
    } else {
        const uint2 w = *reinterpret_cast<const uint2*>(rows + lane * 8);
        h[0] = *reinterpret_cast<const __half2*>(&w.x);
        h[1] = *reinterpret_cast<const __half2*>(&w.y);
    }
    __half2 lo = h[0], hi = h[0];
#pragma unroll
    for (int i = 1; i < EL / 2; ++i) {
        lo = __hmin2(lo, h[i]);
        hi = __hmax2(hi, h[i]);
    }
    __half2 mm = __halves2half2(__hmin(__low2half(lo), __high2half(lo)), __hmax(__low2half(hi), __high2half(hi)));
#pragma unroll
    for (int o = 1; o < GL; o <<= 1) {
        const uint32_t tu = __shfl_xor_sync(0xffffffffu, *reinterpret_cast<const uint32_t*>(&mm), o);
        const __half2 t = *reinterpret_cast<const __half2*>(&tu);
        mm = __halves2half2(__hmin(__low2half(mm), __low2half(t)), __hmax(__high2half(mm), __high2half(t)));
    }
    float mn = __low2float(mm);
    const float mx = __high2float(mm);
    mn = (mn == 0.0f) ? 0.0f : mn;             // reading P
    const float r = __fsub_rn(mx, mn);
    TokenQ t;
    t.codes = 0u;
    float sc = 0.0f;
    if (r != 0.0f) {                           // reading C
        constexpr float kInv15 = 0.0666666701436042785645f;   // RN(1/15)
        const float s0 = __fmul_rn(r, kInv15);
        sc = __fmaf_rn(__fmaf_rn(-s0, 15.0f, r), kInv15, s0);  // RN(r / 15)
        const float y = __frcp_rn(r);
#pragma unroll
        for (int e = 0; e < EL; ++e) {
            const float x = (e & 1) ? __high2float(h[e / 2]) : __low2float(h[e / 2]);
            const float a = __fsub_rn(x, mn);
            const float q0 = __fmul_rn(a, y);
            const float er = __fmaf_rn(-q0, r, a);
            const float u = __fmaf_rn(er, y, q0);
            const float b = __fadd_rn(__fmul_rn(u, 15.0f), 8388608.0f);   // 2^23 + RNE(15 u)
            t.codes |= (__float_as_uint(b) & 15u) << (4 * e);
        }
    }
    const __half2 m = __halves2half2(__float2half_rn(sc), __float2half_rn(mn));
    t.meta = *reinterpret_cast<const uint32_t*>(&m);
    return t;
}
// Store the lane's part of the quantized token at `slot` (index inside its
// 32-token chunk) of `chunk`: lanes 0-15 write into a K chunk (token-major code
// rows), lanes 16-31 into a V chunk (byte slot % 4 of the words of its quad row).
// Each lane is called with the chunk of its own half.
template <int D>
__device__ __forceinline__ void store_token(const TokenQ& t, int slot, uint8_t* chunk, int lane) {
    constexpr int EL = D / 16, GL = kGroup / EL;
    constexpr int CB = D / 2, MB = D / 16;
    const int l16 = lane & 15;
    if (lane < 16) {
        const int off = slot * CB + l16 * (EL / 2);
        if constexpr (EL == 8)
            *reinterpret_cast<uint32_t*>(chunk + off) = t.codes;
        else
            *reinterpret_cast<uint16_t*>(chunk + off) = uint16_t(t.codes);
    } else {
        uint8_t* p = chunk + ((slot >> 2) * CB + ((l16 * (EL / 2)) ^ (((slot >> 2) & 3) << 3))) * 4 + (slot & 3);
#pragma unroll
        for (int i = 0; i < EL / 2; ++i) p[4 * i] = uint8_t(t.codes >> (8 * i));
    }
    if (l16 % GL == 0) *reinterpret_cast<uint32_t*>(chunk + kChunk * CB + slot * MB + (l16 / GL) * 4) = t.meta;
}

}  // namespace
}  // namespace flexq

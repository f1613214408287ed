// attn_common.cuh -- shared pieces of the decode-attention kernels (dense and
// Top-K sparse): stage geometry of the chunked KV cache, PTX helpers (mbarrier,
// 1-D TMA bulk copy issued by an elected lane), the tensor-core K-score pass, the
// tensor-core P.V pass and the fused-append token quantizer.  See
// decode_attention.cu and DESIGN.md section 3 for the design notes.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

// One stage = NCH consecutive 32-token chunks of one cache (K or V); its smem
// image has the HBM layout: per chunk [codes 32 x D/2][meta 32 x D/16].
// Each warp also owns an "extra" area with the fp16 rows of its current work
// unit: q, and for the fused append the new token's k and v rows.
template <int D, int NCH>
struct Cfg {
    static constexpr int CH = kChunk * NCH;            // tokens per stage
    static constexpr int CB = D / 2;                   // code bytes per token
    static constexpr int MB = D / 16;                  // meta bytes per token (D/64 half2)
    static constexpr int CHB = kChunk * (CB + MB);     // chunk bytes (18 D)
    static constexpr int OFF_M = kChunk * CB;          // meta inside a chunk
    static constexpr int STG = NCH * CHB;              // stage bytes
    static constexpr int XQ = 0;                       // extra area: q
    static constexpr int XNEW = 2 * D;                 //   k_new, v_new (fused append)
    static constexpr int XTRA = 6 * D;
    static_assert(STG % 16 == 0 && CHB % 16 == 0 && XTRA % 16 == 0, "TMA bulk alignment");
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
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
// Warp-collective forms: every lane of the warp calls them with the same
// (warp-uniform) operands and elect.sync picks the one lane that issues, so the
// copy-issue code stays straight-line (no lane-0 branch around the TMA).
__device__ __forceinline__ void mbar_expect_tx_elect(uint64_t* bar, uint32_t bytes) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_addr(bar)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_elect(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                               uint64_t policy) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;\n\t}" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
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

// ---------------------------------------------------------------- pass 1 on the tensor cores
// The scores of 16 tokens at a time as integer matrix products on IMMA
// (mma.sync m16n8k32, u8 codes x s8 q digits, exact int32 accumulation):
//   A (16 x 32, u8)  = codes of 16 tokens (rows) x 32 elements (k), straight from
//                      the smem stage.  The even columns of a code word are its low
//                      nibbles (w & 0x0F0F0F0F), the odd columns its high nibbles,
//                      taken in place as w & 0xF0F0F0F0 = 16 c: the even and odd
//                      columns go to separate MMAs (Clo, Chi) and 16 Clo + Chi = 16 C
//                      is formed once per token block (no shifts in the inner loop).
//                      MMA m = 2i + h covers code words 2i, 2i+1 of the lane's
//                      16-byte slice of the row, h = 0 even / h = 1 odd columns.
//   B (32 x 8, s8)   = q as a 23-bit fixed-point integer per 64-element group
//                      (scale 2^(22 - E_g), |q| < 2^E_g), split into three signed
//                      base-256 digits; column n = (digit, group) (3 G columns used).
//   C (16 x 8, s32)  = per token, the dot products of its codes with each digit of
//                      each group's q.
// The element order along k is the same permutation on both operands (a dot
// product does not care).  Epilogue per token (each lane holds two C columns of
// two tokens; a 2-step quad reduction adds them up):
//   score = sum_g scale_g 2^(E_g - 22) qscale (C_g0 + 2^8 C_g1 + 2^16 C_g2)
//           + sum_g min_g qscale sum_{j in g} q_j                  (log2 domain).
// Column map: D = 128: n = 0..5 -> (d0,g0) (d1,g0) (d2,g0) (d2,g1) (d0,g1) (d1,g1);
// D = 64: n = 0..2 -> d0, d1, d2.  Lanes tig 0 and 2 combine their two columns in
// int32 (C_d0 + 2^8 C_d1), tig 1 holds the two d2 columns, tig 3 (zero columns)
// adds the min term.
__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int D>
struct KFrag {
    static constexpr int KS = D / 32;   // MMAs per token block
    uint32_t b[KS][2];                  // B fragment (q digits of the lane's column) per MMA
    int k256;                           // 256: combine the lane's two C columns in int32
    float wA, wB, bA, bB;               // v = fma(x0, wA, bA) hA + fma(x1, wB, bB) hB
    int offA, offB;                     // byte offsets of hA / hB in the token's meta
};

// q (fp16 [D] at qs, smem) -> the lane's KFrag.  Lane (n, j) owns the B column n
// and the k rows 4j..4j+3, 16+4j..16+4j+3 of every MMA.
template <int D>
__device__ __forceinline__ void load_q_mma(const uint8_t* qs, float qscale, int lane, KFrag<D>& kf) {
    constexpr int KS = D / 32, G = D / 64, NE = 8 * KS;   // elements per lane (its 16-B code slice)
    constexpr int JG = 4 / G;                             // quad lanes per group
    const int n = lane >> 2, j = lane & 3;
    const uint4* qv = reinterpret_cast<const uint4*>(qs) + KS * j;   // elements 8 (KS j + w) + e
    __half2 h[NE / 2];
#pragma unroll
    for (int w = 0; w < KS; ++w) {
        const uint4 u = qv[w];
        h[4 * w + 0] = *reinterpret_cast<const __half2*>(&u.x);
        h[4 * w + 1] = *reinterpret_cast<const __half2*>(&u.y);
        h[4 * w + 2] = *reinterpret_cast<const __half2*>(&u.z);
        h[4 * w + 3] = *reinterpret_cast<const __half2*>(&u.w);
    }
    __half2 am = __habs2(h[0]);
    float2 s2 = __half22float2(h[0]);
#pragma unroll
    for (int i = 1; i < NE / 2; ++i) {
        am = __hmax2(am, __habs2(h[i]));                 // exact
        const float2 f = __half22float2(h[i]);
        s2.x += f.x;
        s2.y += f.y;
    }
    float mx = fmaxf(__low2float(am), __high2float(am));
    float sum = s2.x + s2.y;
#pragma unroll
    for (int o = 1; o < JG; o <<= 1) {
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
    }
    // E = the exponent with mx < 2^E (mx = 0 -> E = -126, harmless); Q = RN(q 2^(22 - E)), |Q| < 2^22
    const int eb = int((__float_as_uint(mx) >> 23) & 0xFFu);   // mx in [2^(eb-127), 2^(eb-126))
    const int E = max(eb - 126, -100);
    const float up = __int_as_float((127 + 22 - E) << 23);      // 2^(22 - E), exact scaling
    const int gl = j / JG;                                       // the group of the lane's words
    int dig = -1, grp = -1;
    if (G == 2) {
        dig = n < 3 ? n : (n == 3 ? 2 : (n == 4 ? 0 : (n == 5 ? 1 : -1)));
        grp = n < 3 ? 0 : (n < 6 ? 1 : -1);
    } else if (n < 3) {
        dig = n;
        grp = 0;
    }
    const bool live = dig >= 0 && grp == gl;
    // Signed base-256 digits: R = Q + 0x8080 = (d0 + 128) + 2^8 (d1 + 128) + 2^16 d2, so digit
    // k < 2 is byte k of R minus 128 (= byte ^ 0x80 as s8) and d2 is byte 2 of R (|d2| <= 64).
    // RN(q up) is formed by the 1.5 2^23 magic add (exact for |q up| < 2^22; ties to even).
    const uint32_t dsel = uint32_t(dig < 0 ? 0 : dig);
    const uint32_t sel01 = dsel | ((dsel + 4u) << 4);           // PRMT: byte dsel of a, of b
    const uint32_t flip = dsel < 2u ? 0x80808080u : 0u;
#pragma unroll
    for (int m = 0; m < KS; ++m) {                 // MMA m: words 2i, 2i+1 (i = m / 2), h = m % 2
        const int i = m >> 1, hb = m & 1;
        uint32_t bw[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {              // b0: word 2i, b1: word 2i + 1
            const int w = 2 * i + r;
            uint32_t R[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {          // element 2e + hb of word w
                const __half2 hh = h[4 * w + e];
                const float qv2 = hb ? __high2float(hh) : __low2float(hh);
                R[e] = __float_as_uint(fmaf(qv2, up, 12582912.0f)) - (0x4B400000u - 0x8080u);
            }
            bw[r] = __byte_perm(__byte_perm(R[0], R[1], sel01), __byte_perm(R[2], R[3], sel01), 0x5410) ^ flip;
        }
        kf.b[m][0] = live ? bw[0] : 0u;
        kf.b[m][1] = live ? bw[1] : 0u;
    }
    // per-group weights from the quad lanes that own each group (the 1/16 of Chi folded in)
    const float w_l = qscale * __int_as_float((127 + E - 22 - 4) << 23);   // qscale 2^(E - 22) / 16
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

// Pass 1, one 16-token block `blk` of the stage at sb (tokens 16 blk + [0, 16)): scores -> sc
// (stage-relative index t0 + token), running max mx over tokens < n (per lane: the caller
// reduces it over the whole warp, xor 1 .. 16).
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
    int clo[4] = {0, 0, 0, 0}, chi[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < KS / 2; ++i) {
        mma_u8s8(clo, w0[2 * i] & 0x0F0F0F0Fu, w8[2 * i] & 0x0F0F0F0Fu, w0[2 * i + 1] & 0x0F0F0F0Fu,
                 w8[2 * i + 1] & 0x0F0F0F0Fu, kf.b[2 * i][0], kf.b[2 * i][1]);
        mma_u8s8(chi, w0[2 * i] & 0xF0F0F0F0u, w8[2 * i] & 0xF0F0F0F0u, w0[2 * i + 1] & 0xF0F0F0F0u,
                 w8[2 * i + 1] & 0xF0F0F0F0u, kf.b[2 * i + 1][0], kf.b[2 * i + 1][1]);
    }
    int c[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = clo[i] * 16 + chi[i];   // 16 C, exact (|16 C| < 2^31)
    const uint8_t* mr = ch + C::OFF_M + slot * C::MB;
    const float hA0 = __half2float(*reinterpret_cast<const __half*>(mr + kf.offA));
    const float hB0 = __half2float(*reinterpret_cast<const __half*>(mr + kf.offB));
    const float hA8 = __half2float(*reinterpret_cast<const __half*>(mr + 8 * C::MB + kf.offA));
    const float hB8 = __half2float(*reinterpret_cast<const __half*>(mr + 8 * C::MB + kf.offB));
    float v0 = fmaf(fmaf(float(c[0] + kf.k256 * c[1]), kf.wA, kf.bA), hA0, fmaf(float(c[1]), kf.wB, kf.bB) * hB0);
    float v8 = fmaf(fmaf(float(c[2] + kf.k256 * c[3]), kf.wA, kf.bA), hA8, fmaf(float(c[3]), kf.wB, kf.bB) * hB8);
    // quad sum as a reduce-scatter: after the xor-1 round even lanes hold row r's pair sum and
    // odd lanes row r + 8's, after the xor-2 round the full sums (the same additions in the same
    // order as two all-reduces, half the shuffles)
    const bool odd = j & 1;
    float v = (odd ? v8 : v0) + __shfl_xor_sync(0xffffffffu, odd ? v0 : v8, 1);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    const int mine = tok + (odd ? 8 : 0);
    if (mine < n) {
        mx = fmaxf(mx, v);
        if (j < 2) sc[t0 + mine] = v;
    }
}

// ---------------------------------------------------------------- pass 2 on the tensor cores
// P.V of each 32-token k-step as IMMA m16n8k32 (u8 x u8, exact int32):
//   A (16 x 32) = V codes: row r <-> column 2 p (low nibbles, w & 0x0F0F0F0F),
//                 row r + 8 <-> column 2 p + 1 (high nibbles, w & 0xF0F0F0F0 = 16 c),
//                 p = PPL r + u for tile u; k <-> tokens: positions 4j..4j+3 are the
//                 4 tokens of quad 8s + j (one quad-interleaved word), 16+4j.. quad 8s+4+j;
//   B (32 x 8)  = the weights a_tg = p_t scale_tg as 24-bit fixed point, split into three
//                 byte limbs (table [group][quad][limb], built per stage); column n =
//                 (limb, group) as in pass 1's map;
//   C (16 x 8)  = per column, per (limb, group) int32 sums over the whole work unit.
// The fixed-point scale of a group is a running one: 2^(23 - e_g) with 2^(e_g - kVHead)
// above the largest weight seen so far in the unit (p <= 1, the unit's exact max is known
// from pass 1).  When a stage's weights reach 2^e_g, the int32 sums of that group are first
// flushed into fp32 (exact conversion of the limb sums at the old scale, then zeroed) and
// e_g is raised; otherwise the sums simply keep accumulating in int32 (no overflow:
// <= 1088 tokens x 255 x 240).  Limbs and nibble positions are combined per lane row at
// the flush and at the end of the unit.
template <int D, int NCH>
constexpr int kLimbWords = (D / 64) * (NCH * kChunk / 4) * 4;   // [group][quad][4 words]

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
    int c[PPL][4];                       // int32 sums of C, per tile / C register
    float ev[PPL], od[PPL];              // flushed fp32 parts of the lane row's even / odd column (x 16)
    int e[D / 64];                       // running exponent per group (weights < 2^e)
    float l, bsum[D / 64];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int u = 0; u < PPL; ++u) {
#pragma unroll
            for (int i = 0; i < 4; ++i) c[u][i] = 0;
            ev[u] = 0.0f;
            od[u] = 0.0f;
        }
        l = 0.0f;
#pragma unroll
        for (int g = 0; g < D / 64; ++g) {
            bsum[g] = 0.0f;
            e[g] = -100;
        }
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

// Headroom of the running fixed-point scale: a group's scale is set 2^kVHead above the
// largest weight seen so far, so later stages rarely raise it (each raise flushes the
// group's int32 sums to fp32); weights keep >= 19 significant bits against the running bound.
constexpr int kVHead = 4;

// 2^(e - 23): the value of one unit of a limb-0 sum at running exponent e (0: no weights yet).
__device__ __forceinline__ float unit_of(int e) {
    return e < -100 ? 0.0f : __int_as_float((127 + e - 23) << 23);
}

// One stage of pass 2: weight pre-pass (lane (quad qd, group g) computes the 4 weights
// of its quad; the per-group max comes from one REDUX max on the float bits, a >= 0 so
// the bit patterns order like the values), running-scale update, limb table, MMAs.
template <int D, int NCH>
__device__ __forceinline__ void v_stage_mma(VAccM<D>& va, const VLane<D>& vl, const uint8_t* sb, const float* sc,
                                            float M, int n, int lane, uint32_t* limbs) {
    using C = Cfg<D, NCH>;
    constexpr int G = D / 64, PPL = D / 16, Q = C::CH / 4;
    static_assert(Q * G <= 32, "one (quad, group) per lane");
    {   // ---- weights of the stage's tokens -> limb table
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
        if (g == 0) va.l += ps;                   // p is counted once (lanes of group 1 repeat the quad)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) if (g == gg) va.bsum[gg] += bs;
        float up = 0.0f;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const uint32_t mb = __reduce_max_sync(0xffffffffu, (g == gg) ? __float_as_uint(amax) : 0u);
            // weights < 2^es with es = exponent field - 126 (0 -> tiny, dropped below)
            const int es = int((mb >> 23) & 0xFFu) - 126;
            if (es > va.e[gg]) {                  // warp-uniform: the running scale grows
                if (vl.gr == gg && va.e[gg] > -100) {   // flush the lane row's sums of this group (exact; none before its first weights)
                    const float f = unit_of(va.e[gg]);
                    const float w0 = vl.w0 * f, w1 = vl.w1 * f;
#pragma unroll
                    for (int u = 0; u < PPL; ++u) {
                        va.ev[u] = fmaf(float(va.c[u][0]), w0, fmaf(float(va.c[u][1]), w1, va.ev[u]));
                        va.od[u] = fmaf(float(va.c[u][2]), w0, fmaf(float(va.c[u][3]), w1, va.od[u]));
#pragma unroll
                        for (int i = 0; i < 4; ++i) va.c[u][i] = 0;
                    }
                }
                va.e[gg] = es + kVHead;
            }
            const int eg = va.e[gg];              // weights < 2^eg; fixed point 2^(23 - eg)
            const float u = eg < -100 ? 0.0f : __int_as_float((127 + 23 - eg) << 23);
            up = (g == gg) ? u : up;
        }
        if (act) {
            const uint32_t q0 = uint32_t(__float2int_rn(a[0] * up)), q1 = uint32_t(__float2int_rn(a[1] * up));
            const uint32_t q2 = uint32_t(__float2int_rn(a[2] * up)), q3 = uint32_t(__float2int_rn(a[3] * up));
            const uint32_t l01 = __byte_perm(q0, q1, 0x5140), l23 = __byte_perm(q2, q3, 0x5140);   // bytes 0, 1
            const uint32_t h01 = __byte_perm(q0, q1, 0x7362), h23 = __byte_perm(q2, q3, 0x7362);   // bytes 2, 3
            *reinterpret_cast<uint4*>(limbs + (g * Q + qd) * 4) = make_uint4(
                __byte_perm(l01, l23, 0x5410), __byte_perm(l01, l23, 0x7632), __byte_perm(h01, h23, 0x5410), 0u);
        }
        __syncwarp();
    }
    // ---- MMAs over the stage's 32-token k-steps
    const int r = lane >> 2, j = lane & 3;
    const uint32_t* lt = limbs + vl.tab;
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
            mma_u8u8(va.c[u], xa[u] & 0x0F0F0F0Fu, xa[u] & 0xF0F0F0F0u, xb[u] & 0x0F0F0F0Fu, xb[u] & 0xF0F0F0F0u, b0,
                     b1);
    }
    __syncwarp();   // limb table reuse by the next stage
}

// End of a unit (pass 2): convert the int32 sums with the running scales, combine limbs /
// nibble positions, quad-reduce, add the bias, then normalise and write fp16 (v_part ==
// nullptr) or store the unnormalised partial (v_part[D], natural column order).  Lane
// (r, j) writes tiles u = j, j + 4, ... (columns 2 (PPL r + u), +1).
template <int D>
__device__ __forceinline__ void v_finish_mma(const VAccM<D>& va, const VLane<D>& vl, int lane, __half* out_bh,
                                             float& lsum, float* v_part) {
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
    // column weights: limb weight x 2^(e_g - 23) of the lane row's group (vl.w0 / w1 are 0 for
    // columns of the other group and unused columns)
    const float f = unit_of(vl.gr == 0 ? va.e[0] : va.e[G - 1]);
    const float w0 = vl.w0 * f, w1 = vl.w1 * f;
    const float bias = vl.gr == 0 ? b[0] : b[G - 1];
    const float inv_l = 1.0f / l;
#pragma unroll
    for (int u = 0; u < PPL; ++u) {
        float ev = fmaf(float(va.c[u][0]), w0, fmaf(float(va.c[u][1]), w1, va.ev[u]));             // column 2p
        float od = fmaf(float(va.c[u][2]), w0, fmaf(float(va.c[u][3]), w1, va.od[u])) * 0.0625f;   // 2p+1 (16 c)
        ev += __shfl_xor_sync(0xffffffffu, ev, 1);
        od += __shfl_xor_sync(0xffffffffu, od, 1);
        ev += __shfl_xor_sync(0xffffffffu, ev, 2);
        od += __shfl_xor_sync(0xffffffffu, od, 2);
        if ((u & 3) == j) {
            const int col = 2 * (PPL * r + (u ^ (vl.hx >> 2)));   // tile u holds pair PPL r + (u ^ 4) on odd rows (D = 128)
            ev += bias;
            od += bias;
            if (v_part) {
                *reinterpret_cast<float2*>(v_part + col) = make_float2(ev, od);
            } else {
                *reinterpret_cast<__half2*>(out_bh + col) = __floats2half2_rn(ev * inv_l, od * inv_l);
            }
        }
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

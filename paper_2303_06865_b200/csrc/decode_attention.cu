// decode_attention.cu -- decode-step attention over the 4-bit group-wise
// compressed KV cache, dequantization fused in registers (sm_100a).
//
// Computes, per (batch, head) (readings K, M):
//   out = softmax(q . K^[0:cur_len]^T / sqrt(D)) . V^[0:cur_len],
//   K^_tj = fmaf(c_tj, scale_tg, min_tg) in fp32 (never rounded to fp16).
//
// Design:
//  * Persistent kernel, one warp = one work unit = (b, h, context split);
//    units handed out by an atomic ticket in the workspace (self-resetting).
//  * Each warp owns an S-stage shared-memory ring.  A stage is NCH consecutive
//    32-token chunks of the K cache (pass 1) or of the V cache (pass 2) --
//    codes + fp16 (scale, min), one contiguous run in HBM -- loaded by one
//    elected lane with a single 1-D TMA bulk copy (cp.async.bulk -> mbarrier
//    complete_tx); q rides with the unit's first stage.  Loads run S-1 stages
//    ahead of the math, across units.
//  * Two passes per unit, no online rescaling: pass 1 streams the unit's K
//    halves and writes every score (log2 domain) to a per-warp smem buffer,
//    pass 2 takes the exact max, streams the V halves and accumulates
//    p_t = 2^(s_t - M).  Only one of q (pass 1) or the V accumulators (pass
//    2) is live at a time, which keeps the register footprint small.
//  * Lane layout: D/32 lanes per token, 16 B of codes (32 nibbles) per lane.
//    Dequantization is factored out of the inner loop (lever a):
//      score = sum_g [ scale_g * sum_{j in g} q_j c_j + min_g * sum_{j in g} q_j ]
//      o_j   = sum_t (p_t scale_tg) c_tj + sum_t p_t min_tg
//    Nibbles become floats with one LOP3 each (2^23 magic-exponent trick; the
//    nibble keeps its bit position, so its value carries a 16^k factor that
//    is folded into q on the K side and removed once at the end on the V
//    side), one packed FADD2 per pair removes the 2^23 bias exactly, one
//    packed FFMA2 per pair accumulates.
//  * End of unit: reduce-scatter of the 32 per-lane accumulators across the
//    token lanes (28 shuffles), each lane writes D/32 outputs.  Units of a
//    split (b, h) write (acc, m, l) partials; the last split (atomic ticket)
//    merges them with the log-sum-exp rule (online-softmax combine).
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kMaxSplitUnits = 8192;   // partial slots in the workspace
constexpr int kMinSplitTokens = 64;
constexpr int kMinUnitTokens = 512;    // smallest per-warp score buffer of any variant (sizes the workspace)

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
    static constexpr int STAGE = OFF_Q + 2 * D;        // + q (fp16) for the unit's first stage
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

// Nibble e of a 32-bit code word as the float 2^23 + c_e * 16^k:
// e = 0..4 in place (bits 4e..4e+3, k = e); e = 5..7 from w >> 12 at bits
// 8..19 (k = e - 3).  The magic exponent lives in a register so that
// (w & mask) | magic is a single LOP3 (LOP3 takes one immediate).
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
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t magic, float2 (&f)[4]) {
    const uint32_t w12 = w >> 12;
    const float2 bias = make_float2(-8388608.0f, -8388608.0f);
    f[0] = __fadd2_rn(make_float2(nib<0x0000Fu>(w, magic), nib<0x000F0u>(w, magic)), bias);     // (c0, 16 c1)
    f[1] = __fadd2_rn(make_float2(nib<0x00F00u>(w, magic), nib<0x0F000u>(w, magic)), bias);     // (256 c2, 4096 c3)
    f[2] = __fadd2_rn(make_float2(nib<0xF0000u>(w, magic), nib<0x00F00u>(w12, magic)), bias);   // (65536 c4, 256 c5)
    f[3] = __fadd2_rn(make_float2(nib<0x0F000u>(w12, magic), nib<0xF0000u>(w12, magic)), bias); // (4096 c6, 65536 c7)
}
// 2^-k of the two nibbles of pair p (order of unpack8).
__device__ __forceinline__ float2 inv_shift(int pair) {
    switch (pair) {
        case 0: return make_float2(1.0f, 0.0625f);
        case 1: return make_float2(0.00390625f, 0.000244140625f);
        case 2: return make_float2(1.52587890625e-05f, 0.00390625f);
        default: return make_float2(0.000244140625f, 1.52587890625e-05f);
    }
}

struct Desc {        // per-slot descriptor (shared memory)
    int unit;        // work unit id (-1: none)
    int bh;          // (batch, head) index of the unit
    int t0;          // first token of the stage, relative to the unit
    int flags;       // kFirst | kV | kLastK | kLast, tokens in the stage << 8
};
constexpr int kFirst = 1, kV = 2, kLastK = 4, kLast = 8;

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
};

// Pass 1, one warp iteration (tokens i*TPI + [0, TPI) of the stage): scores -> smem (log2 domain).
// lc / lm: the lane's byte offsets inside a token row (codes / meta).
template <int D, int NCH, bool FULL>
__device__ __forceinline__ void k_iter(int i, const float2 (&qp)[16], float qsum, const uint8_t* sb, float* sc,
                                       int t0, int tl, int n, int lc, int lm, int sg, uint32_t magic, float& mx) {
    using C = Cfg<D, NCH>;
    const int tok = i * C::TPI + tl;
    const uint4 kw = lds128(sb + C::code_off(i) + lc);
    const float2 km = __half22float2(*reinterpret_cast<const __half2*>(sb + C::meta_off(i) + lm));
    float2 d0 = make_float2(0.0f, 0.0f), d1 = d0;
    float2 f[4];
    unpack8(kw.x, magic, f);
    d0 = __ffma2_rn(qp[0], f[0], d0); d1 = __ffma2_rn(qp[1], f[1], d1);
    d0 = __ffma2_rn(qp[2], f[2], d0); d1 = __ffma2_rn(qp[3], f[3], d1);
    unpack8(kw.y, magic, f);
    d0 = __ffma2_rn(qp[4], f[0], d0); d1 = __ffma2_rn(qp[5], f[1], d1);
    d0 = __ffma2_rn(qp[6], f[2], d0); d1 = __ffma2_rn(qp[7], f[3], d1);
    unpack8(kw.z, magic, f);
    d0 = __ffma2_rn(qp[8], f[0], d0); d1 = __ffma2_rn(qp[9], f[1], d1);
    d0 = __ffma2_rn(qp[10], f[2], d0); d1 = __ffma2_rn(qp[11], f[3], d1);
    unpack8(kw.w, magic, f);
    d0 = __ffma2_rn(qp[12], f[0], d0); d1 = __ffma2_rn(qp[13], f[1], d1);
    d0 = __ffma2_rn(qp[14], f[2], d0); d1 = __ffma2_rn(qp[15], f[3], d1);
    d0 = __fadd2_rn(d0, d1);
    float s = fmaf(km.x, d0.x + d0.y, km.y * qsum);
#pragma unroll
    for (int o = 1; o < C::LPT; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (FULL || tok < n) {
        mx = fmaxf(mx, s);
        if (sg == 0) sc[t0 + tok] = s;
    }
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

// UNR: unroll factor of the full-stage loops (code size vs. scheduling freedom:
// fully unrolled K and V bodies overflow the instruction cache).
// MAXT: per-warp score buffer (tokens); longer contexts are split into units of <= MAXT.
template <int D, int NCH, int S, int WPC, int UNR, int MAXT>
__global__ void __launch_bounds__(WPC * 32, (20 / WPC) > 0 ? (20 / WPC) : 1)
decode_attention_kernel(const Params P) {
    using C = Cfg<D, NCH>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* ring = smem + warp * (S * C::STAGE);
    float* scores = reinterpret_cast<float*>(smem + WPC * S * C::STAGE) + warp * MAXT;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WPC * (S * C::STAGE + MAXT * 4)) + warp * S;
    Desc* desc = reinterpret_cast<Desc*>(smem + WPC * (S * (C::STAGE + 8) + MAXT * 4)) + warp * S;

    const int units = P.bh_total * P.nsplit;
    const uint64_t policy = evict_first_policy();
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_proxy_async();
    }
    __syncwarp();

    // ---------------- producer (warp-uniform state; lane 0 issues the copies)
    int p_unit = -1, p_bh = 0, p_first = 0, p_end = 0, p_tok = 0;
    bool p_v = false;
    auto next_unit = [&]() {
        int t = 0;
        if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= units) {
            p_unit = -1;
            return;
        }
        p_unit = t;
        int split = 0;
        p_bh = t;
        if (P.nsplit > 1) {
            p_bh = t / P.nsplit;
            split = t - p_bh * P.nsplit;
        }
        p_tok = p_first = split * P.split_len;
        p_end = min(P.cur_len, p_tok + P.split_len);
        p_v = false;
    };
    auto issue = [&](int slot) {
        if (lane == 0) {
            Desc d;
            uint32_t bytes = 0;
            if (p_unit >= 0) {
                const bool first = !p_v && p_tok == p_first;
                const bool last_of_pass = p_tok + C::CH >= p_end;
                d.unit = p_unit;
                d.bh = p_bh;
                d.t0 = p_tok - p_first;
                const int n = min(C::CH, p_end - p_tok);
                d.flags = (first ? kFirst : 0) | (p_v ? kV : 0) | (!p_v && last_of_pass ? kLastK : 0) |
                          (p_v && last_of_pass ? kLast : 0) | (n << 8);
                bytes = uint32_t((n + kChunk - 1) / kChunk) * C::CHB + (first ? 2 * D : 0);
            } else {
                d.unit = -1; d.bh = 0; d.t0 = 0; d.flags = 0;
            }
            desc[slot] = d;
            fence_proxy_async();
            mbar_expect_tx(&bars[slot], bytes);
            if (p_unit >= 0) {
                uint8_t* sb = ring + slot * C::STAGE;
                const int64_t chunk = int64_t(p_bh) * P.chunks + (p_tok >> 5);
                const uint32_t data = bytes - ((d.flags & kFirst) ? 2 * D : 0);
                bulk_g2s(sb, (p_v ? P.vc : P.kc) + chunk * C::CHB, data, &bars[slot], policy);
                if (d.flags & kFirst) bulk_g2s(sb + C::OFF_Q, P.q + int64_t(p_bh) * D, 2 * D, &bars[slot], policy);
            }
        }
        if (p_unit >= 0) {
            p_tok += C::CH;
            if (p_tok >= p_end) {
                if (!p_v) {
                    p_v = true;
                    p_tok = p_first;
                } else {
                    next_unit();
                }
            }
        }
    };

    next_unit();
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) issue(s);

    // ---------------- consumer: per unit, pass 1 (K stages) then pass 2 (V stages)
    const int tl = lane / C::LPT;         // token slot in an iteration
    const int sg = lane % C::LPT;         // 16-byte segment of the token row
    const int lc = tl * C::CB + sg * 16;  // lane's codes offset inside an iteration's rows
    const int lm = tl * C::MB + (sg >> 1) * 4;   // lane's meta (group of the segment) offset
    const uint32_t magic = magic_reg();

    int slot = 0;
    uint32_t parity = 0;
    auto next_stage = [&](Desc& d) -> const uint8_t* {   // issue ahead, wait for the current slot
        issue(slot == 0 ? S - 1 : slot - 1);
        mbar_wait(&bars[slot], parity);
        d = desc[slot];
        return ring + slot * C::STAGE;
    };
    auto release = [&]() {
        __syncwarp();
        if (++slot == S) {
            slot = 0;
            parity ^= 1u;
        }
    };

#pragma unroll 1
    for (;;) {
        Desc d;
        const uint8_t* sb = next_stage(d);
        if (d.unit < 0) break;
        const int bh = d.bh;
        const int unit = d.unit;

        // ------------------------------------------------ pass 1: scores -> smem
        float M;
        {
            float2 qp[16];                    // q * qscale * 2^-k, pairs in unpack8 order
            float qsum = 0.0f;
            {
                const uint4 q0 = lds128(sb + C::OFF_Q + sg * 64);
                const uint4 q1 = lds128(sb + C::OFF_Q + sg * 64 + 16);
                const uint4 q2 = lds128(sb + C::OFF_Q + sg * 64 + 32);
                const uint4 q3 = lds128(sb + C::OFF_Q + sg * 64 + 48);
                const uint32_t qw[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                                         q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
#pragma unroll
                for (int k = 0; k < 16; ++k) {     // pair k = columns 2k, 2k+1 = word k/4, pair k%4
                    float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qw[k]));
                    f = __fmul2_rn(f, make_float2(P.qscale, P.qscale));
                    qsum += f.x + f.y;
                    qp[k] = __fmul2_rn(f, inv_shift(k & 3));
                }
            }
            float mx = -INFINITY;
#pragma unroll 1
            for (;;) {
                const int n = d.flags >> 8;
                if (n == C::CH) {
#pragma unroll UNR
                    for (int i = 0; i < C::ITERS; ++i)
                        k_iter<D, NCH, true>(i, qp, qsum, sb, scores, d.t0, tl, n, lc, lm, sg, magic, mx);
                } else {
#pragma unroll 1
                    for (int i = 0; i < C::ITERS; ++i)
                        if (i * C::TPI < n)
                            k_iter<D, NCH, false>(i, qp, qsum, sb, scores, d.t0, tl, n, lc, lm, sg, magic, mx);
                }
                const bool last = d.flags & kLastK;
                release();
                if (last) break;
                sb = next_stage(d);
            }
#pragma unroll
            for (int o = C::LPT; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            M = mx;
        }

        // ------------------------------------------------ pass 2: P.V with p = 2^(s - M)
        float2 acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = make_float2(0.0f, 0.0f);
        float l = 0.0f, bsum = 0.0f;
#pragma unroll 1
        for (;;) {
            sb = next_stage(d);
            const int n = d.flags >> 8;
            if (n == C::CH) {
#pragma unroll UNR
                for (int i = 0; i < C::ITERS; ++i)
                    v_iter<D, NCH, true>(i, acc, l, bsum, sb, scores, M, d.t0, tl, n, lc, lm, magic);
            } else {
#pragma unroll 1
                for (int i = 0; i < C::ITERS; ++i)
                    if (i * C::TPI < n)
                        v_iter<D, NCH, false>(i, acc, l, bsum, sb, scores, M, d.t0, tl, n, lc, lm, magic);
            }
            const bool last = d.flags & kLast;
            release();
            if (last) break;
        }

        // ------------------------------------------------ end of unit: reduce over token lanes, write
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = __fmul2_rn(acc[k], inv_shift(k & 3));
#pragma unroll
        for (int o = C::LPT; o < 32; o <<= 1) {
            l += __shfl_xor_sync(0xffffffffu, l, o);
            bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
        }
        float v[32];
#pragma unroll
        for (int k = 0; k < 16; ++k) { v[2 * k] = acc[k].x; v[2 * k + 1] = acc[k].y; }
        int width = 32;   // live entries
        int base = 0;     // column offset (within the 32-column segment) of v[0]
#pragma unroll
        for (int o = 16; o >= C::LPT; o >>= 1) {
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
        // lane now holds columns [32 sg + base, + D/32)
        const int col0 = sg * 32 + base;
        if (P.nsplit == 1) {
            const float inv = 1.0f / l;
            __half* dst = P.out + int64_t(bh) * D + col0;
            if constexpr (D == 128) {
                __half2 h0 = __floats2half2_rn((v[0] + bsum) * inv, (v[1] + bsum) * inv);
                __half2 h1 = __floats2half2_rn((v[2] + bsum) * inv, (v[3] + bsum) * inv);
                uint2 w;
                w.x = *reinterpret_cast<uint32_t*>(&h0);
                w.y = *reinterpret_cast<uint32_t*>(&h1);
                *reinterpret_cast<uint2*>(dst) = w;
            } else {
                *reinterpret_cast<__half2*>(dst) = __floats2half2_rn((v[0] + bsum) * inv, (v[1] + bsum) * inv);
            }
        } else {
            float* dst = P.part + int64_t(unit) * D + col0;
#pragma unroll
            for (int k = 0; k < D / 32; ++k) dst[k] = v[k] + bsum;
            if (lane == 0) P.ml[unit] = make_float2(M, l);
            __threadfence();
            __syncwarp();
            uint32_t done = 0;
            if (lane == 0) done = atomicAdd(&P.tickets[bh], 1u);
            done = __shfl_sync(0xffffffffu, done, 0);
            if (done == uint32_t(P.nsplit - 1)) {   // last split of this (b, h): merge
                __threadfence();
                float Mx = -INFINITY;
                for (int s2 = 0; s2 < P.nsplit; ++s2) Mx = fmaxf(Mx, __ldcg(&P.ml[bh * P.nsplit + s2].x));
                for (int c = lane; c < D; c += 32) {
                    float num = 0.0f, den = 0.0f;
                    for (int s2 = 0; s2 < P.nsplit; ++s2) {
                        const int u = bh * P.nsplit + s2;
                        const float2 mlv = __ldcg(&P.ml[u]);
                        const float w = ex2(mlv.x - Mx);
                        num = fmaf(w, __ldcg(&P.part[int64_t(u) * D + c]), num);
                        den = fmaf(w, mlv.y, den);
                    }
                    P.out[int64_t(bh) * D + c] = __float2half_rn(num / den);
                }
                if (lane == 0) P.tickets[bh] = 0u;   // leave the workspace zeroed
            }
        }
    }

    // retire: the last warp out resets the ticket counter for the next call
    if (lane == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * WPC;
        if (atomicAdd(P.ctrl + 1, 1u) == total - 1) {
            P.ctrl[0] = 0u;
            P.ctrl[1] = 0u;
            __threadfence();
        }
    }
}

template <int D, int NCH, int S, int WPC, int MAXT>
constexpr size_t smem_bytes() {
    return size_t(WPC) * (S * (Cfg<D, NCH>::STAGE + 8 + sizeof(Desc)) + MAXT * 4);
}

int sm_count() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int D, int NCH, int S, int WPC, int UNR, int MAXT>
int ctas_per_sm() {
    static int occ = -1;
    if (occ < 0) {
        auto k = decode_attention_kernel<D, NCH, S, WPC, UNR, MAXT>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_bytes<D, NCH, S, WPC, MAXT>()));
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, WPC * 32, smem_bytes<D, NCH, S, WPC, MAXT>());
        occ = o > 0 ? o : 1;
    }
    return occ;
}

struct WsLayout {
    size_t ctrl, tickets, part, ml, total;
};
// Split-K partial slots: kMaxSplitUnits for occupancy splits, plus one per
// (b, h) and unit-long piece when the capacity exceeds the smallest unit.
int64_t split_slots(int bh, int t_cap) {
    const int64_t pieces = (t_cap + kMinUnitTokens - 1) / kMinUnitTokens;
    return pieces > 1 ? std::max<int64_t>(kMaxSplitUnits, int64_t(bh) * pieces) : kMaxSplitUnits;
}
WsLayout ws_layout(int bh, int d, int t_cap) {
    WsLayout w;
    const int64_t slots = split_slots(bh, t_cap);
    w.ctrl = 0;
    w.tickets = 256;
    w.part = (w.tickets + size_t(bh) * 4 + 255) / 256 * 256;
    w.ml = w.part + size_t(slots) * d * 4;
    w.total = w.ml + size_t(slots) * 8;
    return w;
}

template <int D, int NCH, int S, int WPC, int UNR, int MAXT>
cudaError_t launch(const AttnArgs& a, cudaStream_t stream) {
    const int bh = a.batch * a.heads;
    const int occ = ctas_per_sm<D, NCH, S, WPC, UNR, MAXT>();
    const int ctas_resident = sm_count() * occ;
    const int warps_resident = ctas_resident * WPC;
    // context split: only when (b, h) units cannot fill the resident warps
    // context split: forced when a unit would exceed the score buffer, else only
    // when (b, h) units cannot fill the resident warps
    const int min_split = (a.cur_len + MAXT - 1) / MAXT;
    int nsplit = min_split;
    if (int64_t(bh) * nsplit < warps_resident) {
        nsplit = (warps_resident + bh - 1) / bh;
        const int max_by_len = (a.cur_len + kMinSplitTokens - 1) / kMinSplitTokens;
        nsplit = min(nsplit, max_by_len);
        nsplit = int(std::min<int64_t>(nsplit, split_slots(bh, a.t_cap) / bh));
        nsplit = max(nsplit, min_split);
    }
    int split_len = (a.cur_len + nsplit - 1) / nsplit;
    split_len = (split_len + Cfg<D, NCH>::CH - 1) / Cfg<D, NCH>::CH * Cfg<D, NCH>::CH;
    nsplit = (a.cur_len + split_len - 1) / split_len;
    const int units = bh * nsplit;
    const int ctas = min(ctas_resident, (units + WPC - 1) / WPC);

    const WsLayout w = ws_layout(bh, D, a.t_cap);
    uint8_t* ws = static_cast<uint8_t*>(a.workspace);
    Params P;
    P.q = static_cast<const __half*>(a.q);
    P.kc = static_cast<const uint8_t*>(a.k_cache);
    P.vc = static_cast<const uint8_t*>(a.v_cache);
    P.out = static_cast<__half*>(a.out);
    P.ctrl = reinterpret_cast<uint32_t*>(ws + w.ctrl);
    P.tickets = reinterpret_cast<uint32_t*>(ws + w.tickets);
    P.part = reinterpret_cast<float*>(ws + w.part);
    P.ml = reinterpret_cast<float2*>(ws + w.ml);
    P.bh_total = bh;
    P.chunks = a.chunks;
    P.cur_len = a.cur_len;
    P.nsplit = nsplit;
    P.split_len = split_len;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    decode_attention_kernel<D, NCH, S, WPC, UNR, MAXT><<<ctas, WPC * 32, smem_bytes<D, NCH, S, WPC, MAXT>(), stream>>>(P);
    return cudaGetLastError();
}

// Stage geometry (tokens per stage CH, ring depth S, warps per CTA).  The
// defaults come from the B200 sweep recorded in DESIGN.md; the environment
// variable FLEXQ_ATTN_CFG="<CH>,<S>,<WPC>" selects another compiled variant
// (tuning only).
int64_t tune_variant() {
    static int64_t v = -2;
    if (v == -2) {
        v = -1;
        const char* e = getenv("FLEXQ_ATTN_CFG");
        int ch = 0, st = 0, wpc = 0, unr = 4, mt = 1024;
        if (e && sscanf(e, "%d,%d,%d,%d,%d", &ch, &st, &wpc, &unr, &mt) >= 3)
            v = ((((int64_t(ch) * 16 + st) * 16 + wpc) * 16 + unr) * 4096) + mt;
    }
    return v;
}

#define FLEXQ_V(ch, s, w, u, mt) (((((int64_t(ch) * 16 + (s)) * 16 + (w)) * 16 + (u)) * 4096) + (mt))

}  // namespace

size_t attention_workspace_bytes(int batch, int heads, int head_dim, int t_cap) {
    return ws_layout(batch * heads, head_dim, t_cap).total;
}

// FLEXQ_ATTN_CFG="<stage tokens>,<S>,<WPC>,<unroll>,<score tokens>" (tuning only).
cudaError_t launch_decode_attention(const AttnArgs& a, cudaStream_t stream) {
    const int64_t v = tune_variant();
    if (a.head_dim == 128) {
        switch (v) {
            case FLEXQ_V(64, 2, 4, 4, 1024): return launch<128, 2, 2, 4, 4, 1024>(a, stream);
            case FLEXQ_V(64, 2, 4, 8, 1024): return launch<128, 2, 2, 4, 8, 1024>(a, stream);
            case FLEXQ_V(64, 2, 2, 4, 576): return launch<128, 2, 2, 2, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 1, 4, 576): return launch<128, 2, 2, 1, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 4, 4, 576): return launch<128, 2, 2, 4, 4, 576>(a, stream);
            case FLEXQ_V(32, 2, 4, 4, 576): return launch<128, 1, 2, 4, 4, 576>(a, stream);
            case FLEXQ_V(32, 3, 2, 4, 576): return launch<128, 1, 3, 2, 4, 576>(a, stream);
            default: return launch<128, 2, 2, 4, 4, 1024>(a, stream);
        }
    }
    switch (v) {
        case FLEXQ_V(64, 2, 2, 4, 576): return launch<64, 2, 2, 2, 4, 576>(a, stream);
        default: return launch<64, 2, 2, 4, 4, 1024>(a, stream);
    }
}

}  // namespace flexq

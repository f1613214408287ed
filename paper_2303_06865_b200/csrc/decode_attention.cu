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
//  * Each warp owns an S-stage shared-memory ring.  One stage = CH tokens of
//    K codes + V codes (TMA 1-D bulk copies, cp.async.bulk -> mbarrier
//    complete_tx) and K/V fp16 (scale, min) pairs (cp.async 8/4-byte copies,
//    arrive.noinc on the same mbarrier); the first stage of a unit also
//    carries q.  Loads run S-1 stages ahead of the math, across units.
//  * Lane layout: D/32 lanes per token, 16 B of codes (32 nibbles) per lane.
//    Dequantization is factored out of the inner loop (lever a):
//      score = sum_g [ scale_g * sum_{j in g} q_j c_j + min_g * sum_{j in g} q_j ]
//      o_j   = sum_t (p_t scale_tg) c_tj + sum_t p_t min_tg
//    Nibbles become floats with one LOP3 each (2^23 magic-exponent trick; the
//    nibble keeps its bit position, so its value carries a 16^k factor that
//    is folded into q on the K side and removed once at the end on the V
//    side), one packed FADD2 per pair removes the 2^23 bias exactly, one
//    packed FFMA2 per pair accumulates.
//  * Online softmax in the exp2 domain with a warp-uniform running max that
//    is only raised when a score exceeds it by > 8 (so p <= 2^8, no
//    overflow); the final result divides by the sum taken against the same
//    max, so it is exact math, not an approximation.
//  * End of unit: reduce-scatter of the 32 per-lane accumulators across the
//    token lanes (28 shuffles), each lane writes 4 outputs.  Split units
//    write (acc, m, l) partials; the last split of a (b, h) (atomic ticket)
//    merges them with the log-sum-exp rule.
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kWarpsPerCta = 4;
constexpr int kMaxSplitUnits = 8192;   // partial slots in the workspace
constexpr int kMinSplitTokens = 64;
constexpr float kRescaleThresh = 8.0f; // log2 units: p <= 2^8 between rescales

template <int D, int CH_>
struct Cfg {
    static constexpr int LPT = D / 32;                 // lanes per token
    static constexpr int TPI = 32 / LPT;               // tokens per warp iteration
    static constexpr int CH = CH_;                     // tokens per stage
    static constexpr int CB = D / 2;                   // code bytes per token
    static constexpr int MB = D / 16;                  // meta bytes per token (D/64 half2)
    static constexpr int ITERS = CH / TPI;
    static constexpr int OFF_VC = CH * CB;
    static constexpr int OFF_KM = 2 * CH * CB;
    static constexpr int OFF_VM = 2 * CH * CB + CH * MB;
    static constexpr int OFF_Q = 2 * CH * (CB + MB);
    static constexpr int STAGE = OFF_Q + 2 * D;        // + q (fp16) for the unit's first stage
    static_assert(STAGE % 16 == 0, "stage alignment");
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
template <int N>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(dst)), "l"(src), "n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar)) : "memory");
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

// Nibble e of word w as a float carrying 2^kShift[e]:
// e = 0..4 in place (bits 4e..4e+3); e = 5..7 from w >> 12 at bits 8..19.
constexpr uint32_t kMagic = 0x4B000000u;  // 2^23
// The magic exponent must live in a register: LOP3 takes one immediate, so
// (w & mask) | magic is a single LOP3 only when magic is not an immediate.
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
    float2 u0 = make_float2(nib<0x0000Fu>(w, magic), nib<0x000F0u>(w, magic));
    float2 u1 = make_float2(nib<0x00F00u>(w, magic), nib<0x0F000u>(w, magic));
    float2 u2 = make_float2(nib<0xF0000u>(w, magic), nib<0x00F00u>(w12, magic));
    float2 u3 = make_float2(nib<0x0F000u>(w12, magic), nib<0xF0000u>(w12, magic));
    const float2 bias = make_float2(-8388608.0f, -8388608.0f);
    f[0] = __fadd2_rn(u0, bias);   // exact: (c0, 16 c1)
    f[1] = __fadd2_rn(u1, bias);   // (256 c2, 4096 c3)
    f[2] = __fadd2_rn(u2, bias);   // (65536 c4, 256 c5)
    f[3] = __fadd2_rn(u3, bias);   // (4096 c6, 65536 c7)
}
// 2^-shift of nibble e (pairs as in unpack8).
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
    int t0;          // first token of this stage
    int n;           // tokens in this stage
    int flags;       // bit0 first stage of unit, bit1 last stage of unit
};

struct Params {
    const __half* q;
    const uint8_t* kc;
    const uint8_t* km;
    const uint8_t* vc;
    const uint8_t* vm;
    __half* out;
    uint32_t* ctrl;      // [0] next ticket, [1] finished warps
    uint32_t* tickets;   // per (b, h): finished splits
    float* part;         // [unit][D] partial numerators
    float2* ml;          // [unit] (m, l)
    int bh_total, t_cap, cur_len, nsplit, split_len;
    float qscale;        // log2(e) / sqrt(D)
};

template <int D, int CH, int kStages>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
decode_attention_kernel(const Params P) {
    using C = Cfg<D, CH>;
    static_assert(CH % C::TPI == 0 && CH <= 64, "stage size");
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* ring = smem + warp * (kStages * C::STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kWarpsPerCta * kStages * C::STAGE) + warp * kStages;
    Desc* desc = reinterpret_cast<Desc*>(smem + kWarpsPerCta * kStages * (C::STAGE + 8)) + warp * kStages;

    const int units = P.bh_total * P.nsplit;
    const uint64_t policy = evict_first_policy();
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 33);
        fence_proxy_async();
    }
    __syncwarp();

    // ---------------- producer state (warp-collective) ----------------
    int p_unit = -1, p_tok = 0, p_end = 0;   // current unit, next token to load, unit end
    auto next_unit = [&]() {
        int t = 0;
        if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= units) { p_unit = -1; return; }
        p_unit = t;
        const int split = t % P.nsplit;
        p_tok = split * P.split_len;
        p_end = min(P.cur_len, p_tok + P.split_len);
    };
    auto issue = [&](int slot) {      // load the next stage into `slot`; returns via desc
        Desc d;
        if (p_unit < 0) {
            d.unit = -1; d.t0 = 0; d.n = 0; d.flags = 0;
        } else {
            const int bh = p_unit / P.nsplit;
            const int split = p_unit % P.nsplit;
            const int n = min(C::CH, p_end - p_tok);
            d.unit = p_unit; d.t0 = p_tok; d.n = n;
            d.flags = (p_tok == split * P.split_len ? 1 : 0) | (p_tok + n >= p_end ? 2 : 0);
            uint8_t* sb = ring + slot * C::STAGE;
            const int64_t row = int64_t(bh) * P.t_cap + p_tok;
            if (lane == 0) {
                fence_proxy_async();
                const uint32_t cbytes = uint32_t(n) * C::CB;
                const uint32_t qbytes = (d.flags & 1) ? 2u * D : 0u;
                mbar_expect_tx(&bars[slot], 2 * cbytes + qbytes);
                bulk_g2s(sb, P.kc + row * C::CB, cbytes, &bars[slot], policy);
                bulk_g2s(sb + C::OFF_VC, P.vc + row * C::CB, cbytes, &bars[slot], policy);
                if (qbytes) bulk_g2s(sb + C::OFF_Q, P.q + int64_t(bh) * D, qbytes, &bars[slot], policy);
            }
            for (int i = lane; i < n; i += 32) {
                cp_async<C::MB>(sb + C::OFF_KM + i * C::MB, P.km + (row + i) * C::MB);
                cp_async<C::MB>(sb + C::OFF_VM + i * C::MB, P.vm + (row + i) * C::MB);
            }
            p_tok += n;
            if (p_tok >= p_end) next_unit();
        }
        if (lane == 0) desc[slot] = d;
        cp_async_arrive_noinc(&bars[slot]);
        if (d.unit < 0 && lane == 0) {
            // keep the barrier phase count consistent: expect nothing, arrive once
            mbar_expect_tx(&bars[slot], 0);
        }
        __syncwarp();   // desc[slot] visible to every lane before it is waited on
    };

    next_unit();
    for (int s = 0; s < kStages - 1; ++s) issue(s);

    // ---------------- consumer state ----------------
    const int tl = lane / C::LPT;         // token slot in an iteration
    const int sg = lane % C::LPT;         // 16-byte segment of the token row
    const int grp = sg >> 1;              // quantization group of the segment (64 = 2 x 32)
    float2 qp[16];                        // q * qscale * 2^-shift, pairs per unpack8 order
    float qsum = 0.0f;                    // sum of q * qscale over the lane's 32 columns
    float2 acc[16];
    float m = -INFINITY, l = 0.0f, bsum = 0.0f;
    const uint32_t magic = magic_reg();

    for (int it = 0;; ++it) {
        const int slot = it % kStages;
        const uint32_t parity = (it / kStages) & 1;
        issue((it + kStages - 1) % kStages);
        mbar_wait(&bars[slot], parity);
        const Desc d = desc[slot];
        if (d.unit < 0) break;
        const uint8_t* sb = ring + slot * C::STAGE;

        if (d.flags & 1) {   // first stage of a unit: load q, reset state
            const uint4 q0 = lds128(sb + C::OFF_Q + sg * 64);
            const uint4 q1 = lds128(sb + C::OFF_Q + sg * 64 + 16);
            const uint4 q2 = lds128(sb + C::OFF_Q + sg * 64 + 32);
            const uint4 q3 = lds128(sb + C::OFF_Q + sg * 64 + 48);
            const uint32_t qw[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                                     q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
            qsum = 0.0f;
#pragma unroll
            for (int k = 0; k < 16; ++k) {     // pair k = columns 2k, 2k+1 = word k/4, pair k%4
                float2 f = __half22float2(*reinterpret_cast<const __half2*>(&qw[k]));
                f.x *= P.qscale;
                f.y *= P.qscale;
                qsum += f.x + f.y;
                const float2 s = inv_shift(k & 3);
                qp[k] = make_float2(f.x * s.x, f.y * s.y);
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) acc[k] = make_float2(0.0f, 0.0f);
            m = -INFINITY;
            l = 0.0f;
            bsum = 0.0f;
        }

#pragma unroll
        for (int i = 0; i < C::ITERS; ++i) {
            const int tok = i * C::TPI + tl;
            const bool valid = tok < d.n;
            // ---- K: partial dot over 32 columns, then the group affine terms
            const uint4 kw = lds128(sb + tok * C::CB + sg * 16);
            const __half2 kmh = *reinterpret_cast<const __half2*>(sb + C::OFF_KM + tok * C::MB + grp * 4);
            float2 d0 = make_float2(0.0f, 0.0f), d1 = d0;
            {
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
            }
            const float2 km = __half22float2(kmh);
            float s = fmaf(km.x, (d0.x + d0.y) + (d1.x + d1.y), km.y * qsum);
#pragma unroll
            for (int o = 1; o < C::LPT; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            s = valid ? s : -INFINITY;

            // ---- online softmax (log2 domain), warp-uniform max
            if (__any_sync(0xffffffffu, s > m + kRescaleThresh)) {
                float mx = s;
#pragma unroll
                for (int o = C::LPT; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float mnew = fmaxf(m, mx);
                const float sc = ex2(m - mnew);     // m = -inf -> 0
#pragma unroll
                for (int k = 0; k < 16; ++k) acc[k] = make_float2(acc[k].x * sc, acc[k].y * sc);
                l *= sc;
                bsum *= sc;
                m = mnew;
            }
            const float p = valid ? ex2(s - m) : 0.0f;
            l += p;

            // ---- V: acc_j += (p * scale) * c_j ; bias += p * min
            const uint4 vw = lds128(sb + C::OFF_VC + tok * C::CB + sg * 16);
            const __half2 vmh = *reinterpret_cast<const __half2*>(sb + C::OFF_VM + tok * C::MB + grp * 4);
            float2 vm = __half22float2(vmh);
            vm.x = valid ? vm.x : 0.0f;
            vm.y = valid ? vm.y : 0.0f;
            const float a = p * vm.x;
            bsum = fmaf(p, vm.y, bsum);
            const float2 a2 = make_float2(a, a);
            {
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
        }
        __syncwarp();

        if (d.flags & 2) {   // last stage of the unit: reduce and write
            // remove the 16^k nibble-position factors
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const float2 s = inv_shift(k & 3);
                acc[k] = make_float2(acc[k].x * s.x, acc[k].y * s.y);
            }
            // l and bias: full reduction over token lanes
#pragma unroll
            for (int o = C::LPT; o < 32; o <<= 1) {
                l += __shfl_xor_sync(0xffffffffu, l, o);
                bsum += __shfl_xor_sync(0xffffffffu, bsum, o);
            }
            // reduce-scatter of the 32 accumulators (16 float2) over token lanes
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
            // lane now holds columns [32 sg + base, + width)
            const int col0 = sg * 32 + base;
            const int bh = d.unit / P.nsplit;
            if (P.nsplit == 1) {
                const float inv = 1.0f / l;
                __half* dst = P.out + int64_t(bh) * D + col0;
                if constexpr (D == 128) {   // width 4
                    __half2 h0 = __floats2half2_rn((v[0] + bsum) * inv, (v[1] + bsum) * inv);
                    __half2 h1 = __floats2half2_rn((v[2] + bsum) * inv, (v[3] + bsum) * inv);
                    uint2 w;
                    w.x = *reinterpret_cast<uint32_t*>(&h0);
                    w.y = *reinterpret_cast<uint32_t*>(&h1);
                    *reinterpret_cast<uint2*>(dst) = w;
                } else {                    // width 2
                    *reinterpret_cast<__half2*>(dst) = __floats2half2_rn((v[0] + bsum) * inv, (v[1] + bsum) * inv);
                }
            } else {
                float* dst = P.part + int64_t(d.unit) * D + col0;
#pragma unroll
                for (int k = 0; k < D / 32; ++k) dst[k] = v[k] + bsum;   // width == D / 32
                if (lane == 0) P.ml[d.unit] = make_float2(m, l);
                __threadfence();
                __syncwarp();
                uint32_t done = 0;
                if (lane == 0) done = atomicAdd(&P.tickets[bh], 1u);
                done = __shfl_sync(0xffffffffu, done, 0);
                if (done == uint32_t(P.nsplit - 1)) {   // last split of this (b, h): merge
                    __threadfence();
                    float M = -INFINITY;
                    for (int s2 = 0; s2 < P.nsplit; ++s2) M = fmaxf(M, __ldcg(&P.ml[bh * P.nsplit + s2].x));
                    for (int c = lane; c < D; c += 32) {
                        float num = 0.0f, den = 0.0f;
                        for (int s2 = 0; s2 < P.nsplit; ++s2) {
                            const int u = bh * P.nsplit + s2;
                            const float2 mlv = __ldcg(&P.ml[u]);
                            const float w = ex2(mlv.x - M);
                            num = fmaf(w, __ldcg(&P.part[int64_t(u) * D + c]), num);
                            den = fmaf(w, mlv.y, den);
                        }
                        P.out[int64_t(bh) * D + c] = __float2half_rn(num / den);
                    }
                    if (lane == 0) P.tickets[bh] = 0u;   // leave the workspace zeroed
                }
            }
        }
    }

    // retire: the last warp out resets the ticket counter for the next call
    if (lane == 0) {
        __threadfence();
        const uint32_t total = gridDim.x * kWarpsPerCta;
        if (atomicAdd(P.ctrl + 1, 1u) == total - 1) {
            P.ctrl[0] = 0u;
            P.ctrl[1] = 0u;
            __threadfence();
        }
    }
}

template <int D, int CH, int S>
constexpr size_t smem_bytes() {
    return size_t(kWarpsPerCta) * S * (Cfg<D, CH>::STAGE + 8 + sizeof(Desc));
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

template <int D, int CH, int S>
int ctas_per_sm() {
    static int occ = -1;
    if (occ < 0) {
        cudaFuncSetAttribute(decode_attention_kernel<D, CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem_bytes<D, CH, S>()));
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, decode_attention_kernel<D, CH, S>, kWarpsPerCta * 32,
                                                      smem_bytes<D, CH, S>());
        occ = o > 0 ? o : 1;
    }
    return occ;
}

struct WsLayout {
    size_t ctrl, tickets, part, ml, total;
};
WsLayout ws_layout(int bh, int d) {
    WsLayout w;
    w.ctrl = 0;
    w.tickets = 256;
    w.part = (w.tickets + size_t(bh) * 4 + 255) / 256 * 256;
    w.ml = w.part + size_t(kMaxSplitUnits) * d * 4;
    w.total = w.ml + size_t(kMaxSplitUnits) * 8;
    return w;
}

template <int D, int CH, int S>
cudaError_t launch(const AttnArgs& a, cudaStream_t stream) {
    const int bh = a.batch * a.heads;
    const int occ = ctas_per_sm<D, CH, S>();
    const int ctas_resident = sm_count() * occ;
    const int warps_resident = ctas_resident * kWarpsPerCta;
    // context split: only when (b, h) units cannot fill the resident warps
    int nsplit = 1;
    if (bh < warps_resident) {
        nsplit = (warps_resident + bh - 1) / bh;
        const int max_by_len = (a.cur_len + kMinSplitTokens - 1) / kMinSplitTokens;
        nsplit = min(nsplit, max_by_len);
        nsplit = min(nsplit, kMaxSplitUnits / bh);
        if (nsplit < 1) nsplit = 1;
    }
    int split_len = (a.cur_len + nsplit - 1) / nsplit;
    split_len = (split_len + CH - 1) / CH * CH;
    nsplit = (a.cur_len + split_len - 1) / split_len;
    const int units = bh * nsplit;
    const int ctas = min(ctas_resident, (units + kWarpsPerCta - 1) / kWarpsPerCta);

    const WsLayout w = ws_layout(bh, D);
    uint8_t* ws = static_cast<uint8_t*>(a.workspace);
    Params P;
    P.q = static_cast<const __half*>(a.q);
    P.kc = static_cast<const uint8_t*>(a.k_codes);
    P.km = static_cast<const uint8_t*>(a.k_meta);
    P.vc = static_cast<const uint8_t*>(a.v_codes);
    P.vm = static_cast<const uint8_t*>(a.v_meta);
    P.out = static_cast<__half*>(a.out);
    P.ctrl = reinterpret_cast<uint32_t*>(ws + w.ctrl);
    P.tickets = reinterpret_cast<uint32_t*>(ws + w.tickets);
    P.part = reinterpret_cast<float*>(ws + w.part);
    P.ml = reinterpret_cast<float2*>(ws + w.ml);
    P.bh_total = bh;
    P.t_cap = a.t_cap;
    P.cur_len = a.cur_len;
    P.nsplit = nsplit;
    P.split_len = split_len;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    decode_attention_kernel<D, CH, S><<<ctas, kWarpsPerCta * 32, smem_bytes<D, CH, S>(), stream>>>(P);
    return cudaGetLastError();
}

}  // namespace

size_t attention_workspace_bytes(int batch, int heads, int head_dim, int /*t_cap*/) {
    return ws_layout(batch * heads, head_dim).total;
}

// Stage geometry (tokens per stage CH, ring depth S).  The defaults come from
// the B200 sweep recorded in DESIGN.md; FLEXQ_ATTN_CFG="<CH>,<S>" selects
// another compiled variant (tuning only).
static int tune_variant() {
    static int v = -2;
    if (v == -2) {
        v = -1;
        const char* e = getenv("FLEXQ_ATTN_CFG");
        if (e) {
            int ch = 0, st = 0;
            if (sscanf(e, "%d,%d", &ch, &st) == 2) v = ch * 16 + st;
        }
    }
    return v;
}

cudaError_t launch_decode_attention(const AttnArgs& a, cudaStream_t stream) {
    const int v = tune_variant();
    if (a.head_dim == 128) {
        switch (v) {
            case 32 * 16 + 2: return launch<128, 32, 2>(a, stream);
            case 32 * 16 + 3: return launch<128, 32, 3>(a, stream);
            case 32 * 16 + 4: return launch<128, 32, 4>(a, stream);
            case 16 * 16 + 3: return launch<128, 16, 3>(a, stream);
            case 16 * 16 + 4: return launch<128, 16, 4>(a, stream);
            case 16 * 16 + 5: return launch<128, 16, 5>(a, stream);
            case 64 * 16 + 2: return launch<128, 64, 2>(a, stream);
            default: return launch<128, 32, 4>(a, stream);
        }
    }
    switch (v) {
        case 32 * 16 + 4: return launch<64, 32, 4>(a, stream);
        case 64 * 16 + 2: return launch<64, 64, 2>(a, stream);
        default: return launch<64, 64, 3>(a, stream);
    }
}

}  // namespace flexq

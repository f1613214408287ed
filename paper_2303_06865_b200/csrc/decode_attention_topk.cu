// decode_attention_topk.cu -- Top-K sparse decode attention over the 4-bit
// compressed KV cache (FlexGen Sec. 4 "Sparse Attention", PAPER.md P:853-857,
// SPEC S:496-504).
//
//   s_t = q . K^_t / sqrt(D) for every cached token (full K stream);
//   keep the `keep` largest s_t (equal scores: lower token index first);
//   out = sum_{t kept} p_t V^_t with p renormalised over the kept set.
//
// Only the kept V rows are loaded ("only load a subset of the V cache",
// P:856): at keep = 10% the step reads K (0.5625 B/elem) + 10% of V instead of
// all of V, ~55% of the dense bytes.
//
// Two launches:
//  * topk_select_kernel -- persistent warps, one warp = one (b, h) (no context split; the
//    per-warp score buffer holds kTopkMaxTokens).  The K pass is the dense kernel's TMA-bulk-
//    staged tensor-core pass (attn_common.cuh).  Selection is an exact bitwise select on
//    order-preserving 32-bit keys of the fp32 scores held in registers (one warp-wide REDUX
//    count per bit below the bits all keys share, stopping once exactly `keep` keys lie above
//    the candidate); ties at the threshold key go to the lowest token indices (ballot prefix
//    counts), so the kept set is the definition's.  The head's kept list (index, unnormalised
//    weight p_t) goes to the workspace.  With the V gather out of this kernel the warp's K
//    stream only pauses for the select.
//  * topk_gather_kernel -- one warp per (b, h) reads the kept V rows and accumulates
//    sum p_t V^_t / sum p_t in fp32; groups of rows are loaded before any is used, so the gathers of a
//    head are in flight together.  In the token-major layout (FLEXQ_KV_TOKEN_MAJOR) a kept
//    token is one contiguous 64-byte row (D = 128); in the dense layout it is spread over its
//    256-byte quad row (the price of the dense kernel's operand order).
// The gather is launched with programmatic dependent launch, so its grid is scheduled while
// the select grid drains.
#include <cuda_fp16.h>
#include <stdint.h>

#include <stdlib.h>

#include <mutex>

#include "attn_common.cuh"
#include "flexq_internal.h"

#ifndef FLEXQ_TOPK_MINB
#define FLEXQ_TOPK_MINB 4   // select kernel: CTAs per SM the register budget is sized for
#endif
#ifndef FLEXQ_TOPK_WPC
#define FLEXQ_TOPK_WPC 4    // select kernel: warps (= (b, h) units in flight) per CTA
#endif

namespace flexq {
namespace {

// ---------------------------------------------------------------- V-row gather helpers
// Nibble -> float conversion of one 32-bit code word (8 codes, columns e = 0..7):
// (w & 0xF<<4e) | 0x4B000000 = 2^23 + c_e 16^e (one LOP3 per code, e = 5..7 from
// w >> 12), one FADD2 removes 2^23 per pair.  Pairs: f[0] = (c0, 16 c1),
// f[1] = (256 c2, 4096 c3), f[2] = (65536 c4, 256 c5), f[3] = (4096 c6, 65536 c7).
// The value is exact; the power-of-two factor is removed once per unit
// (inv_shift).  The magic constant lives in a register so that (w & mask) | magic
// is a single LOP3.
__device__ __forceinline__ uint32_t magic_reg() {
    uint32_t m;
    asm volatile("mov.b32 %0, 0x4B000000;" : "=r"(m));
    return m;
}
template <uint32_t M>
__device__ __forceinline__ uint32_t lop_and_or(uint32_t w, uint32_t magic) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "n"(M), "r"(magic));  // (a & b) | c
    return r;
}
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t magic, float2 (&f)[4]) {
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
}
// 2^-k of the two codes of pair p (order of unpack8).
__device__ __forceinline__ float2 inv_shift(int pair) {
    switch (pair) {
        case 0: return make_float2(1.0f, 0.0625f);
        case 1: return make_float2(0.00390625f, 0.000244140625f);
        case 2: return make_float2(1.52587890625e-05f, 0.00390625f);
        default: return make_float2(0.000244140625f, 1.52587890625e-05f);
    }
}
// acc_j += (p scale) c_j over the lane's 32 columns, bias += p min, l += p.
__device__ __forceinline__ void v_accum(float2 (&acc)[16], float& l, float& bsum, uint4 vw, float2 vm, float p,
                                        uint32_t magic) {
    l += p;
    const float a = p * vm.x;
    bsum = fmaf(p, vm.y, bsum);
    const float2 a2 = make_float2(a, a);
    const uint32_t wv[4] = {vw.x, vw.y, vw.z, vw.w};
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        float2 f[4];
        unpack8(wv[w], magic, f);
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[4 * w + k] = __ffma2_rn(a2, f[k], acc[4 * w + k]);
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
        v[8 * (k / 4) + 2 * (k & 3)] = acc[k].x;
        v[8 * (k / 4) + 2 * (k & 3) + 1] = acc[k].y;
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

// The gather's row loads carry the 64-byte L2 fetch hint (SASS LDG...LTC64B): a kept token's code
// row is one aligned 64-byte run and its (scale, min) pair 8 bytes, so a larger line fill only
// drags in neighbours that are mostly not kept (FLEXQ_TOPK_L2HINT=0: no hint, A/B builds).
#ifndef FLEXQ_TOPK_L2HINT
#define FLEXQ_TOPK_L2HINT 1
#endif
#if FLEXQ_TOPK_L2HINT
#define FLEXQ_LDG_ROW "ld.global.nc.L1::no_allocate.L2::64B"
#else
#define FLEXQ_LDG_ROW "ld.global.nc.L1::no_allocate"
#endif
__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
    uint4 r;
    asm volatile(FLEXQ_LDG_ROW ".v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_nc32(const void* p) {
    uint32_t r;
    asm volatile(FLEXQ_LDG_ROW ".u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

struct SelectParams {
    const __half* q;
    const uint8_t* kc;
    int32_t* sel;        // optional [bh][keep] kept token indices (ascending)
    int32_t* kidx;       // [bh][keep] kept token indices (workspace)
    float* kw;           // [bh][keep] their unnormalised softmax weights 2^(s_t - M) (the gather renormalises)
    uint32_t* ctrl;      // [0] next ticket, [1] finished warps (workspace)
    int bh_total, chunks, cur_len, keep;
    float qscale;
};

// c += (a >= b), unsigned, as a compare and a predicated add (the ternary form compiled to a
// compare, an add and a predicated move per key: the select's count rounds are its hot loop)
__device__ __forceinline__ void count_ge(int& c, uint32_t a, uint32_t b) {
    asm("{\n\t.reg .pred p;\n\tsetp.ge.u32 p, %1, %2;\n\t@p add.s32 %0, %0, 1;\n\t}" : "+r"(c) : "r"(a), "r"(b));
}
__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);   // larger float <=> larger key
}

// Kernel 1: scores of every cached token (the dense kernel's tensor-core K pass over a TMA-bulk
// ring), the exact top-`keep` selection, and the kept list with its weights.
template <int D, int NCH, int S, int WPC, int MAXT>
__global__ void __launch_bounds__(WPC * 32, FLEXQ_TOPK_MINB)
topk_select_kernel(const SelectParams P) {
    using C = Cfg<D, NCH>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // q is refilled at a unit's first stage, issued S - 1 stages ahead -- before the previous unit
    // has read its own q when units are a single stage (cur_len <= 64) -- so two q areas alternate,
    // each on its own barrier: unit u + 2's q is issued after unit u has read its q for
    // S - 1 <= 2 nst - 1 (the launcher keeps S = 2 for single-stage units)
    constexpr int NQ = 2;
    constexpr int PW = S * C::STG + NQ * 2 * D + MAXT * 4;   // per warp: ring, q, scores
    uint8_t* ring = smem + warp * PW;
    uint8_t* qsm0 = ring + S * C::STG;
    float* scores = reinterpret_cast<float*>(qsm0 + NQ * 2 * D);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WPC * PW) + warp * (S + NQ);   // + the q barriers

    const uint64_t policy = evict_first_policy();
    if (lane == 0) {
        for (int s = 0; s < S + NQ; ++s) mbar_init(&bars[s], 1);
        fence_proxy_async();
    }
    __syncwarp();
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // ---------------- producer: the K stages of whole (b, h) units (no split)
    const int nst = (P.cur_len + C::CH - 1) / C::CH;
    int p_bh = -1, p_stage = 0, p_units = 0;
    const uint8_t* p_k = nullptr;
    int fq0 = -1, fq1 = -1, fq2 = -1, fq3 = -1, fcount = 0;
    auto next_unit = [&]() {
        int t = 0;
        if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
        t = __shfl_sync(0xffffffffu, t, 0);
        p_bh = t < P.bh_total ? t : -1;
        p_stage = 0;
        if (p_bh >= 0) p_k = P.kc + int64_t(p_bh) * P.chunks * C::CHB;
        if (fcount == 0) fq0 = p_bh; else if (fcount == 1) fq1 = p_bh; else if (fcount == 2) fq2 = p_bh; else fq3 = p_bh;
        ++fcount;
    };
    auto issue = [&](int slot) {   // warp-collective (elect.sync issues)
        if (p_bh < 0) {
            mbar_expect_tx_elect(&bars[slot], 0);
            return;
        }
        const int n = min(C::CH, P.cur_len - p_stage * C::CH);
        const uint32_t bytes = uint32_t((n + kChunk - 1) / kChunk) * C::CHB;
        mbar_expect_tx_elect(&bars[slot], bytes);
        bulk_g2s_elect(ring + slot * C::STG, p_k + int64_t(p_stage) * C::STG, bytes, &bars[slot], policy);
        if (p_stage == 0) {   // the unit's q, on its own barrier (one phase per unit)
            fence_proxy_async();
            const int qb = p_units & 1;
            ++p_units;
            mbar_expect_tx_elect(&bars[S + qb], 2 * D);
            bulk_g2s_elect(qsm0 + qb * 2 * D, P.q + int64_t(p_bh) * D, 2 * D, &bars[S + qb], policy);
        }
        if (++p_stage == nst) next_unit();
    };
    next_unit();
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) issue(s);

    const unsigned lt_mask = (1u << lane) - 1u;
    const int n_tok = P.cur_len;
    const int keep = P.keep;

    int slot = 0;
    uint32_t parity = 0, qparity = 0;   // qparity: bit b = phase of q area b
    int c_units = 0;
    auto acquire = [&]() -> const uint8_t* {
        issue(slot == 0 ? S - 1 : slot - 1);
        mbar_wait(&bars[slot], parity);
        return ring + slot * C::STG;
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
        const int bh = fq0;
        fq0 = fq1;
        fq1 = fq2;
        fq2 = fq3;
        --fcount;
        if (bh < 0) break;

        // ------------------------------------------------ all scores -> smem
        float M;
        {
            const uint8_t* sb = acquire();
            const int qb = c_units & 1;
            ++c_units;
            mbar_wait(&bars[S + qb], (qparity >> qb) & 1u);
            qparity ^= 1u << qb;
            const uint8_t* qsm = qsm0 + qb * 2 * D;
            KFrag<D> kf;                      // the lane's q digits + epilogue weights
            load_q_mma<D>(qsm, P.qscale, lane, kf);
            float mx = -INFINITY;
#pragma unroll 1
            for (int st = 0;;) {
                const int t0 = st * C::CH;
                const int n = min(C::CH, n_tok - t0);
                if (n == C::CH) {
#pragma unroll
                    for (int b = 0; b < C::CH / 16; ++b) k_block_mma<D, NCH>(b, kf, sb, scores, t0, C::CH, lane, mx);
                } else {
#pragma unroll
                    for (int b = 0; b < C::CH / 16; ++b)
                        if (b * 16 < n) k_block_mma<D, NCH>(b, kf, sb, scores, t0, n, lane, mx);
                }
                release();
                if (++st == nst) break;
                sb = acquire();
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            M = mx;   // the largest score is always kept, so M is the kept set's max
        }

        // ------------------------------------------------ select (exact: keep largest, ties -> lowest index)
        // The key T of rank `keep` is built bit by bit over the order-preserving 32-bit keys of
        // the scores, held in registers (token j * 32 + lane; padding 0, below every candidate):
        // a bit is set when at least `keep` keys are >= the candidate, and the search stops as
        // soon as exactly `keep` are.  It starts below the bits every key shares (the highest bit
        // where the largest and smallest key differ): the sign and exponent bits are common to
        // most heads' scores, so ~9 of the 32 count rounds were spent confirming them.  Kept:
        // key > T, or key == T among the first krem by index.  (A shared-atomic histogram of
        // score bins with a rank among the threshold bin's candidates issued ~25 % fewer
        // instructions but ran slower inside the bench's decode step: DESIGN.md section 3.)
        constexpr int KPL = MAXT / 32;
        uint32_t key[KPL];
        uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int t = j * 32 + lane;
            key[j] = t < n_tok ? order_key(scores[t]) : 0u;
            if (t < n_tok) kmin = min(kmin, key[j]);
        }
        kmin = __reduce_min_sync(0xffffffffu, kmin);
        const uint32_t kmax = order_key(M);
        uint32_t T = kmax;
        int krem = keep;                     // every key equal: the lowest `keep` indices
        if (kmin != kmax) {
            const int hb = 31 - __clz(kmax ^ kmin);
            T = kmax & ~((2u << hb) - 1u);   // the shared prefix: every key is >= it
            bool exact = false;
#pragma unroll 1
            for (int bit = hb; bit >= 0; --bit) {
                const uint32_t cand = T | (1u << bit);
                int c = 0;
#pragma unroll
                for (int j = 0; j < KPL; ++j) count_ge(c, key[j], cand);
                c = int(__reduce_add_sync(0xffffffffu, uint32_t(c)));
                if (c >= keep) {
                    T = cand;
                    if (c == keep) {         // exactly `keep` keys >= T: all of them (no tie to break)
                        exact = true;
                        break;
                    }
                }
            }
            if (!exact) {
                int gt = 0;
#pragma unroll
                for (int j = 0; j < KPL; ++j) gt += key[j] > T ? 1 : 0;
                krem = keep - int(__reduce_add_sync(0xffffffffu, uint32_t(gt)));
            }
        }
        // the kept list, straight to the workspace in ascending token order, with the unnormalised
        // weights p_t = 2^(s_t - M) (the gather renormalises over the kept set): two ballots
        // and predicated stores per 32 tokens; the optional `sel` output is the same list
        {
            const int64_t lo = int64_t(bh) * keep;
            int32_t* const hk = P.kidx + lo;
            float* const hw = P.kw + lo;
            int base = 0, ties = 0;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                const int t = j * 32 + lane;
                const bool eq = key[j] == T && t < n_tok;
                const unsigned beq = __ballot_sync(0xffffffffu, eq);
                const bool kc = key[j] > T || (eq && ties + __popc(beq & lt_mask) < krem);
                const unsigned bk = __ballot_sync(0xffffffffu, kc);
                if (kc) {
                    const int o = base + __popc(bk & lt_mask);
                    hk[o] = t;
                    hw[o] = ex2(scores[t] - M);
                    if (P.sel != nullptr) P.sel[lo + o] = t;
                }
                base += __popc(bk);
                ties += __popc(beq);
            }
        }
        __syncwarp();   // scores / kept are rewritten by the next unit
    }

    // let the gather kernel's grid launch (its griddepcontrol.wait still waits for this grid)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
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

struct GatherParams {
    const uint8_t* vc;
    const int32_t* kidx;
    const float* kw;
    __half* out;
    int bh_total, chunks, keep;
};

// Kernel 2: out = sum over the kept tokens of w_t V^_t, one warp per (b, h).  LPT = D / 32 lanes
// per token, lane sg of a token owns its columns 32 sg .. 32 sg + 31 (16 code bytes, one group's
// half).  Token-major V (VTM): the 16 bytes are one load of the token's row; quad-interleaved V:
// four 16-byte loads of the token's quad row and a byte gather (PRMT).  GB groups of TPI tokens
// are loaded before any is accumulated (the loads are independent gathers).
template <int D, bool VTM>
#ifndef FLEXQ_TOPK_GATHER_MINB
#define FLEXQ_TOPK_GATHER_MINB 3   // gather CTAs (of 8 warps) per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(256, FLEXQ_TOPK_GATHER_MINB) topk_gather_kernel(const GatherParams P) {
    constexpr int CB = D / 2, MB = D / 16, CHB = kChunk * (CB + MB);
    constexpr int LPT = D / 32, TPI = 32 / LPT, GB = VTM ? 8 : 4;   // row groups loaded before use
    const int lane = threadIdx.x & 31;
    const int bh = int(blockIdx.x) * (blockDim.x >> 5) + int(threadIdx.x >> 5);
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the kept lists of the select kernel
    if (bh >= P.bh_total) return;
    const int tl = lane / LPT, sg = lane % LPT;
    const uint32_t magic = magic_reg();
    const uint8_t* vbase = P.vc + int64_t(bh) * P.chunks * CHB;
    const int32_t* idx = P.kidx + int64_t(bh) * P.keep;
    const float* wts = P.kw + int64_t(bh) * P.keep;
    float2 acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = make_float2(0.0f, 0.0f);
    float l = 0.0f, bsum = 0.0f;
#pragma unroll 1
    for (int j0 = 0; j0 < P.keep; j0 += GB * TPI) {
        uint4 raw[GB][VTM ? 1 : 4];
        uint32_t meta[GB];
        float w[GB];
        int tk[GB];
#pragma unroll
        for (int g = 0; g < GB; ++g) {
            const int j = j0 + g * TPI + tl;
            const bool v = j < P.keep;
            const int t = v ? __ldg(idx + j) : 0;
            tk[g] = t;
            w[g] = v ? __ldg(wts + j) : 0.0f;
            const uint8_t* cb = vbase + (t >> 5) * CHB;
            meta[g] = ldg_nc32(cb + kChunk * CB + (t & 31) * MB + (sg >> 1) * 4);
            if constexpr (VTM) {
                raw[g][0] = ldg_nc128(cb + (t & 31) * CB + 16 * sg);
            } else {
                // quad row of the token; 8-pair block b of it sits at block b ^ (quad & 3)
                const int quad = (t & 31) >> 2;
                const uint8_t* qr = cb + quad * CB * 4;
                const uint8_t* b0 = qr + ((2 * sg) ^ (quad & 3)) * 32;
                const uint8_t* b1 = qr + ((2 * sg + 1) ^ (quad & 3)) * 32;
                raw[g][0] = ldg_nc128(b0);
                raw[g][1] = ldg_nc128(b0 + 16);
                raw[g][2] = ldg_nc128(b1);
                raw[g][3] = ldg_nc128(b1 + 16);
            }
        }
#pragma unroll
        for (int g = 0; g < GB; ++g) {
            uint4 row;
            if constexpr (VTM) {
                row = raw[g][0];
            } else {   // byte t % 4 of each word: the token's 16 bytes of the segment
                const uint32_t k = uint32_t(tk[g] & 3);
                const uint32_t selb = k | ((k + 4) << 4);
                uint32_t o[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t a = __byte_perm(raw[g][q].x, raw[g][q].y, selb);
                    const uint32_t b = __byte_perm(raw[g][q].z, raw[g][q].w, selb);
                    o[q] = __byte_perm(a, b, 0x5410);
                }
                row = make_uint4(o[0], o[1], o[2], o[3]);
            }
            const float2 vm = __half22float2(*reinterpret_cast<const __half2*>(&meta[g]));
            v_accum(acc, l, bsum, row, vm, w[g], magic);   // w = 0 for padding slots
        }
    }
    float v[32];
    const int col0 = reduce_unit<D>(acc, l, bsum, lane, sg, v);
    write_out<D>(P.out + int64_t(bh) * D + col0, v, l);   // renormalise over the kept set
}

template <int D, int NCH, int S, int WPC, int MAXT>
constexpr size_t select_smem_bytes() {
    constexpr int NQ = 2;
    return size_t(WPC) * (S * Cfg<D, NCH>::STG + NQ * 2 * D + MAXT * 4 + (S + NQ) * 8);
}

constexpr size_t kTopkCtrlBytes = 2048;

template <int D, int NCH, int S, int WPC, int MAXT>
cudaError_t launch_topk(const TopkArgs& a, cudaStream_t stream) {
    auto k = topk_select_kernel<D, NCH, S, WPC, MAXT>;
    const size_t smem = select_smem_bytes<D, NCH, S, WPC, MAXT>();
    // per-device launch facts, computed once per device under a lock
    constexpr int kMaxDev = 64;
    static int occs[kMaxDev], smss[kMaxDev];
    static std::once_flag once[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    std::call_once(once[dev], [&] {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int o = 0, n = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, WPC * 32, smem);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        occs[dev] = o > 0 ? o : 1;
        smss[dev] = n > 0 ? n : 148;
    });
    const int occ = occs[dev], sms = smss[dev];
    const int bh = a.batch * a.heads;
    const int ctas = min(sms * occ, (bh + WPC - 1) / WPC);
    uint8_t* ws = static_cast<uint8_t*>(a.workspace);
    const size_t list = size_t(bh) * size_t(a.keep);
    SelectParams P;
    P.q = static_cast<const __half*>(a.q);
    P.kc = static_cast<const uint8_t*>(a.k_cache);
    P.sel = static_cast<int32_t*>(a.sel);
    P.ctrl = reinterpret_cast<uint32_t*>(ws);
    P.kidx = reinterpret_cast<int32_t*>(ws + kTopkCtrlBytes);
    P.kw = reinterpret_cast<float*>(ws + kTopkCtrlBytes + list * 4);
    P.bh_total = bh;
    P.chunks = a.chunks;
    P.cur_len = a.cur_len;
    P.keep = a.keep;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    k<<<ctas, WPC * 32, smem, stream>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    GatherParams G;
    G.vc = static_cast<const uint8_t*>(a.v_cache);
    G.kidx = P.kidx;
    G.kw = P.kw;
    G.out = static_cast<__half*>(a.out);
    G.bh_total = bh;
    G.chunks = a.chunks;
    G.keep = a.keep;
    // programmatic dependent launch: the gather grid is scheduled as the select grid drains
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((bh + 7) / 8));
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (a.v_tm) return cudaLaunchKernelEx(&cfg, topk_gather_kernel<D, true>, G);
    return cudaLaunchKernelEx(&cfg, topk_gather_kernel<D, false>, G);
}

}  // namespace

size_t topk_workspace_bytes(int batch, int heads, int t_cap) {
    // the kept lists: int32 index + fp32 weight per (b, h, kept token), keep <= t_cap
    return kTopkCtrlBytes + size_t(batch) * size_t(heads) * size_t(t_cap) * 8;
}

template <int S>
cudaError_t launch_topk_s(const TopkArgs& a, cudaStream_t stream) {
    constexpr int W = FLEXQ_TOPK_WPC;
    if (a.head_dim == 128)
        return a.cur_len <= 576 ? launch_topk<128, 2, S, W, 576>(a, stream)
                                : launch_topk<128, 2, S, W, kTopkMaxTokens>(a, stream);
    return a.cur_len <= 576 ? launch_topk<64, 2, S, W, 576>(a, stream)
                            : launch_topk<64, 2, S, W, kTopkMaxTokens>(a, stream);
}

cudaError_t launch_decode_attention_topk(const TopkArgs& a, cudaStream_t stream) {
    // select kernel ring depth (tuning: FLEXQ_TOPK_RING=2|3|4): more stages in flight while a head's
    // keys are selected, but fewer resident warps; 16 warps x 2 stages measured fastest
    static const int ring = [] {
        const char* e = getenv("FLEXQ_TOPK_RING");
        const int r = e ? atoi(e) : 2;   // B200: 2 stages 143 us, 3 stages 156 us, 4 stages 192 us (OPT-175B)
        return r >= 2 && r <= 4 ? r : 2;
    }();
    // two alternating q areas are safe for S - 1 <= 2 nst - 1 stages ahead (nst: stages per
    // unit); single-stage units (cur_len <= 64) keep the 2-stage ring
    if (ring == 2 || a.cur_len <= 64) return launch_topk_s<2>(a, stream);
    if (ring == 4) return launch_topk_s<4>(a, stream);
    return launch_topk_s<3>(a, stream);
}

}  // namespace flexq

// decode_attention_topk.cu -- Top-K sparse decode attention over the 4-bit
// compressed KV cache (FlexGen Sec. 4 "Sparse Attention", PAPER.md P:853-857,
// SPEC S:496-504).
//
//   s_t = q . K^_t / sqrt(D) for every cached token (pass 1, full K stream);
//   keep the `keep` largest s_t (equal scores: lower token index first);
//   out = sum_{t kept} p_t V^_t with p renormalised over the kept set.
//
// Only the kept V rows are loaded ("only load a subset of the V cache",
// P:856): at keep = 10% the step reads K (0.5625 B/elem) + 10% of V instead of
// all of V, ~55% of the dense bytes.
//
// Design: persistent warps, one warp = one (b, h) (no context split; the
// per-warp score buffer holds kTopkMaxTokens).  Pass 1 is the dense kernel's
// TMA-bulk-staged K pass (attn_common.cuh).  Selection is an exact bitwise
// select on order-preserving 32-bit keys of the fp32 scores held in registers
// (one warp-wide REDUX count per bit, stopping once exactly `keep` keys lie
// above the candidate); ties at the threshold key go to the lowest token
// indices (ballot prefix counts), so the kept set is the definition's.
// Pass 2 gathers the kept V rows straight from HBM (the token's quad row of
// the quad-interleaved V chunk, 64 B per lane in 128-bit loads, its byte
// extracted with PRMT, three groups of rows in flight) into
// fp32 register accumulators.
#include <cuda_fp16.h>
#include <stdint.h>

#include <mutex>

#include "attn_common.cuh"
#include "flexq_internal.h"

#ifndef FLEXQ_TOPK_MINB
#define FLEXQ_TOPK_MINB 4   // CTAs per SM the register budget is sized for
#endif
#ifndef FLEXQ_TOPK_WPC
#define FLEXQ_TOPK_WPC 3    // warps (= (b, h) units in flight) per CTA
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

struct TopkParams {
    const __half* q;
    const uint8_t* kc;
    const uint8_t* vc;
    __half* out;
    int32_t* sel;        // optional [bh][keep] kept token indices (ascending)
    uint32_t* ctrl;      // [0] next ticket, [1] finished warps (workspace)
    int bh_total, chunks, cur_len, keep;
    float qscale;
};

__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);   // larger float <=> larger key
}

__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_nc32(const void* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

template <int D, int NCH, int S, int WPC, int MAXT>
__global__ void __launch_bounds__(WPC * 32, FLEXQ_TOPK_MINB)
decode_attention_topk_kernel(const TopkParams P) {
    using C = Cfg<D, NCH>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    constexpr int PW = S * C::STG + 2 * D + MAXT * 6;   // per warp: ring, q, scores, kept list
    uint8_t* ring = smem + warp * PW;
    uint8_t* qsm = ring + S * C::STG;
    float* scores = reinterpret_cast<float*>(qsm + 2 * D);
    uint16_t* kept = reinterpret_cast<uint16_t*>(qsm + 2 * D + MAXT * 4);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WPC * PW) + warp * S;

    const uint64_t policy = evict_first_policy();
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_proxy_async();
    }
    __syncwarp();

    // ---------------- producer: the K stages of whole (b, h) units (no split)
    const int nst = (P.cur_len + C::CH - 1) / C::CH;
    int p_bh = -1, p_stage = 0;
    const uint8_t* p_k = nullptr;
    int fq0 = -1, fq1 = -1, fq2 = -1, fcount = 0;
    auto next_unit = [&]() {
        int t = 0;
        if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
        t = __shfl_sync(0xffffffffu, t, 0);
        p_bh = t < P.bh_total ? t : -1;
        p_stage = 0;
        if (p_bh >= 0) p_k = P.kc + int64_t(p_bh) * P.chunks * C::CHB;
        if (fcount == 0) fq0 = p_bh; else if (fcount == 1) fq1 = p_bh; else fq2 = p_bh;
        ++fcount;
    };
    auto issue = [&](int slot) {   // warp-collective (elect.sync issues)
        if (p_bh < 0) {
            mbar_expect_tx_elect(&bars[slot], 0);
            return;
        }
        const int n = min(C::CH, P.cur_len - p_stage * C::CH);
        const uint32_t bytes = uint32_t((n + kChunk - 1) / kChunk) * C::CHB;
        const bool first = p_stage == 0;
        uint8_t* sb = ring + slot * C::STG;
        mbar_expect_tx_elect(&bars[slot], bytes + (first ? 2 * D : 0));
        bulk_g2s_elect(sb, p_k + int64_t(p_stage) * C::STG, bytes, &bars[slot], policy);
        // q of the unit (read at its first stage, before the next unit's q is issued: S = 2)
        if (first) bulk_g2s_elect(qsm, P.q + int64_t(p_bh) * D, 2 * D, &bars[slot], policy);
        if (++p_stage == nst) next_unit();
    };
    next_unit();
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) issue(s);

    constexpr int LPT = D / 32;   // V gather: lanes per token
    constexpr int TPI = 32 / LPT; //   tokens per warp iteration
    const int tl = lane / LPT;
    const int sg = lane % LPT;
    const uint32_t magic = magic_reg();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int n_tok = P.cur_len;
    const int keep = P.keep;

    int slot = 0;
    uint32_t parity = 0;
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
        --fcount;
        if (bh < 0) break;

        // ------------------------------------------------ pass 1: all scores -> smem
        float M;
        {
            const uint8_t* sb = acquire();
            KFrag<D> kf;                      // the lane's q digits + epilogue weights for pass 1
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
            for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            M = mx;   // the largest score is always kept, so M is the kept set's max
        }

        // ------------------------------------------------ select: key T of rank `keep`
        // Keys live in registers (token j * 32 + lane); T is built bit by bit from the
        // top: a bit is set when at least `keep` keys are >= the candidate.  The search
        // stops as soon as exactly `keep` keys are >= the candidate (then every kept
        // key is >= T and no tie needs breaking); otherwise T ends as the exact key of
        // rank `keep`.  Padding slots hold key 0, below every candidate.
        constexpr int KPL = MAXT / 32;
        uint32_t key[KPL];
#pragma unroll
        for (int j = 0; j < KPL; ++j) {
            const int t = j * 32 + lane;
            key[j] = t < n_tok ? order_key(scores[t]) : 0u;
        }
        uint32_t T = 0u;
        bool exact = false;
#pragma unroll 1
        for (int bit = 31; bit >= 0; --bit) {
            const uint32_t cand = T | (1u << bit);
            int c = 0;
#pragma unroll
            for (int j = 0; j < KPL; ++j) c += key[j] >= cand ? 1 : 0;
            c = int(__reduce_add_sync(0xffffffffu, uint32_t(c)));
            if (c >= keep) {
                T = cand;
                if (c == keep) {
                    exact = true;
                    break;
                }
            }
        }
        // kept: key > T, or key == T among the first krem such tokens by index
        {
            int krem = keep;
            if (!exact) {
                int gt = 0;
#pragma unroll
                for (int j = 0; j < KPL; ++j) gt += key[j] > T ? 1 : 0;
                krem = keep - int(__reduce_add_sync(0xffffffffu, uint32_t(gt)));
            }
            int base = 0, ties = 0;
#pragma unroll
            for (int j = 0; j < KPL; ++j) {
                if (j * 32 >= n_tok) break;
                const bool gt = key[j] > T;
                const bool eq = key[j] == T;
                const unsigned beq = __ballot_sync(0xffffffffu, eq);
                const bool keepit = gt || (eq && ties + __popc(beq & lt_mask) < krem);
                const unsigned bk = __ballot_sync(0xffffffffu, keepit);
                if (keepit) kept[base + __popc(bk & lt_mask)] = uint16_t(j * 32 + lane);
                base += __popc(bk);
                ties += __popc(beq);
            }
            __syncwarp();
            if (P.sel)
                for (int j = lane; j < keep; j += 32) P.sel[int64_t(bh) * keep + j] = kept[j];
        }

        // ------------------------------------------------ pass 2: gather the kept V rows
        float2 acc[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = make_float2(0.0f, 0.0f);
        float l = 0.0f, bsum = 0.0f;
        const uint8_t* vbase = P.vc + int64_t(bh) * P.chunks * C::CHB;
        // V codes are quad-interleaved (include/flexq.h): token t's 16 B segment sg
        // (column pairs 16 sg .. 16 sg + 15) is byte t % 4 of 16 words of its quad
        // row (two swizzled 8-pair blocks); load the 64 B and gather that byte with PRMT.
        auto load_row = [&](int t, uint4 (&raw)[4], uint32_t& meta) {
            const uint8_t* cb = vbase + (t >> 5) * C::CHB;
            const int quad = (t & 31) >> 2;
            const uint8_t* q = cb + quad * C::CB * 4;
            // swizzled layout: 8-pair block b of the quad row sits at block b ^ (quad & 3)
            const uint8_t* b0 = q + ((2 * sg) ^ (quad & 3)) * 32;
            const uint8_t* b1 = q + ((2 * sg + 1) ^ (quad & 3)) * 32;
            raw[0] = ldg_nc128(b0);
            raw[1] = ldg_nc128(b0 + 16);
            raw[2] = ldg_nc128(b1);
            raw[3] = ldg_nc128(b1 + 16);
            meta = ldg_nc32(cb + C::OFF_M + (t & 31) * C::MB + (sg >> 1) * 4);
        };
        auto row_bytes = [&](int t, const uint4 (&raw)[4]) -> uint4 {
            const uint32_t k = uint32_t(t & 3);
            const uint32_t sel = k | ((k + 4) << 4);
            uint32_t o[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t a = __byte_perm(raw[j].x, raw[j].y, sel);   // bytes k of words 4j, 4j+1
                const uint32_t b = __byte_perm(raw[j].z, raw[j].w, sel);   // words 4j+2, 4j+3
                o[j] = __byte_perm(a, b, 0x5410);
            }
            return make_uint4(o[0], o[1], o[2], o[3]);
        };
        auto row_of = [&](int j, int& t) -> bool {
            t = j < keep ? int(kept[j]) : 0;
            return j < keep;
        };
        // three groups of rows in flight (the gather is latency-bound); the loop is
        // unrolled over the three register slots so no slot is copied while its
        // loads are outstanding
        int ta, tb, tc;
        bool va = row_of(tl, ta), vb = row_of(TPI + tl, tb), vc = row_of(2 * TPI + tl, tc);
        uint4 ra[4] = {}, rb[4] = {}, rc[4] = {};
        uint32_t ma = 0u, mb = 0u, mc = 0u;
        if (va) load_row(ta, ra, ma);
        if (vb) load_row(tb, rb, mb);
        if (vc) load_row(tc, rc, mc);
        auto step = [&](int g, int& t, bool& v, uint4 (&r)[4], uint32_t& m) {
            float2 vm = __half22float2(*reinterpret_cast<const __half2*>(&m));
            float p = ex2(scores[t] - M);
            if (!v) {
                p = 0.0f;
                vm = make_float2(0.0f, 0.0f);
            }
            v_accum(acc, l, bsum, row_bytes(t, r), vm, p, magic);
            v = row_of((g + 3) * TPI + tl, t);   // refill the slot with group g + 3
            m = 0u;
            if (v) load_row(t, r, m);
        };
#pragma unroll 1
        for (int g = 0;; g += 3) {
            step(g, ta, va, ra, ma);
            if ((g + 1) * TPI >= keep) break;
            step(g + 1, tb, vb, rb, mb);
            if ((g + 2) * TPI >= keep) break;
            step(g + 2, tc, vc, rc, mc);
            if ((g + 3) * TPI >= keep) break;
        }
        float v[32];
        const int col0 = reduce_unit<D>(acc, l, bsum, lane, sg, v);
        write_out<D>(P.out + int64_t(bh) * D + col0, v, l);
        __syncwarp();
    }

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
constexpr size_t topk_smem_bytes() {
    return size_t(WPC) * (S * (Cfg<D, NCH>::STG + 8) + 2 * D + MAXT * 6);
}

template <int D, int NCH, int S, int WPC, int MAXT>
cudaError_t launch_topk(const TopkArgs& a, cudaStream_t stream) {
    auto k = decode_attention_topk_kernel<D, NCH, S, WPC, MAXT>;
    const size_t smem = topk_smem_bytes<D, NCH, S, WPC, MAXT>();
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
    TopkParams P;
    P.q = static_cast<const __half*>(a.q);
    P.kc = static_cast<const uint8_t*>(a.k_cache);
    P.vc = static_cast<const uint8_t*>(a.v_cache);
    P.out = static_cast<__half*>(a.out);
    P.sel = static_cast<int32_t*>(a.sel);
    P.ctrl = static_cast<uint32_t*>(a.workspace);
    P.bh_total = bh;
    P.chunks = a.chunks;
    P.cur_len = a.cur_len;
    P.keep = a.keep;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    k<<<ctas, WPC * 32, smem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode_attention_topk(const TopkArgs& a, cudaStream_t stream) {
    constexpr int W = FLEXQ_TOPK_WPC;
    if (a.head_dim == 128)
        return a.cur_len <= 576 ? launch_topk<128, 2, 2, W, 576>(a, stream)
                                : launch_topk<128, 2, 2, W, kTopkMaxTokens>(a, stream);
    return a.cur_len <= 576 ? launch_topk<64, 2, 2, W, 576>(a, stream)
                            : launch_topk<64, 2, 2, W, kTopkMaxTokens>(a, stream);
}

}  // namespace flexq

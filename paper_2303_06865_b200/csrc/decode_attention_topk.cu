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
    uint8_t* ring = smem + warp * (S * C::STAGE);
    uint8_t* wsm = smem + WPC * S * C::STAGE + warp * (MAXT * 6);
    float* scores = reinterpret_cast<float*>(wsm);
    uint16_t* kept = reinterpret_cast<uint16_t*>(wsm + MAXT * 4);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WPC * (S * C::STAGE + MAXT * 6)) + warp * S;

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
    auto issue = [&](int slot) {
        if (p_bh < 0) {
            if (lane == 0) mbar_expect_tx(&bars[slot], 0);
            return;
        }
        if (lane == 0) {
            const int n = min(C::CH, P.cur_len - p_stage * C::CH);
            const uint32_t bytes = uint32_t((n + kChunk - 1) / kChunk) * C::CHB;
            const bool first = p_stage == 0;
            uint8_t* sb = ring + slot * C::STAGE;
            mbar_expect_tx(&bars[slot], bytes + (first ? 2 * D : 0));
            bulk_g2s(sb, p_k + int64_t(p_stage) * (NCH * C::CHB), bytes, &bars[slot], policy);
            if (first) bulk_g2s(sb + C::OFF_Q, P.q + int64_t(p_bh) * D, 2 * D, &bars[slot], policy);
        }
        if (++p_stage == nst) next_unit();
    };
    next_unit();
#pragma unroll 1
    for (int s = 0; s < S - 1; ++s) issue(s);

    const int tl = lane / C::LPT;
    const int sg = lane % C::LPT;
    const int lc = tl * C::CB + sg * 16;
    const int lm = tl * C::MB + (sg >> 1) * 4;
    const uint32_t magic = magic_reg();
    const unsigned lt_mask = (1u << lane) - 1u;
    const int n_tok = P.cur_len;
    const int keep = P.keep;

    int slot = 0;
    uint32_t parity = 0;
    auto acquire = [&]() -> const uint8_t* {
        issue(slot == 0 ? S - 1 : slot - 1);
        mbar_wait(&bars[slot], parity);
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
        const int bh = fq0;
        fq0 = fq1;
        fq1 = fq2;
        --fcount;
        if (bh < 0) break;

        // ------------------------------------------------ pass 1: all scores -> smem
        float M;
        {
            const uint8_t* sb = acquire();
#if FLEXQ_K_MMA
            KFrag<D> kf;                      // the lane's q digits + epilogue weights for pass 1
            load_q_mma<D>(sb + C::OFF_Q, P.qscale, lane, kf);
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
#else
            KQuery kq;
            load_q(sb + C::OFF_Q + sg * 64, P.qscale, kq);
            float mx = -INFINITY;
#pragma unroll 1
            for (int st = 0;;) {
                const int t0 = st * C::CH;
                const int n = min(C::CH, n_tok - t0);
                if (n == C::CH) {
#pragma unroll 4
                    for (int i = 0; i < C::ITERS; ++i)
                        k_iter<D, NCH, true>(i, kq, sb, scores, t0, tl, n, lc, lm, sg, magic, mx);
                } else {
#pragma unroll 4
                    for (int i = 0; i < C::ITERS; ++i)
                        if (i * C::TPI < n)
                            k_iter<D, NCH, false>(i, kq, sb, scores, t0, tl, n, lc, lm, sg, magic, mx);
                }
                release();
                if (++st == nst) break;
                sb = acquire();
            }
#endif
#pragma unroll
            for (int o = C::LPT; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
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
        bool va = row_of(tl, ta), vb = row_of(C::TPI + tl, tb), vc = row_of(2 * C::TPI + tl, tc);
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
            v = row_of((g + 3) * C::TPI + tl, t);   // refill the slot with group g + 3
            m = 0u;
            if (v) load_row(t, r, m);
        };
#pragma unroll 1
        for (int g = 0;; g += 3) {
            step(g, ta, va, ra, ma);
            if ((g + 1) * C::TPI >= keep) break;
            step(g + 1, tb, vb, rb, mb);
            if ((g + 2) * C::TPI >= keep) break;
            step(g + 2, tc, vc, rc, mc);
            if ((g + 3) * C::TPI >= keep) break;
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
    return size_t(WPC) * (S * (Cfg<D, NCH>::STAGE + 8) + MAXT * 6);
}

template <int D, int NCH, int S, int WPC, int MAXT>
cudaError_t launch_topk(const TopkArgs& a, cudaStream_t stream) {
    static int occ = -1;
    auto k = decode_attention_topk_kernel<D, NCH, S, WPC, MAXT>;
    const size_t smem = topk_smem_bytes<D, NCH, S, WPC, MAXT>();
    if (occ < 0) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, WPC * 32, smem);
        occ = o > 0 ? o : 1;
    }
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
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

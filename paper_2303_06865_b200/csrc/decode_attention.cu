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

#include "attn_common.cuh"

#ifndef FLEXQ_AB_FENCE
#define FLEXQ_AB_FENCE 1
#endif
#ifndef FLEXQ_AB_GSTORE
#define FLEXQ_AB_GSTORE 2   // fused append write-back: 2 lane stores (default), 1 TMA bulk store, 0 none (A/B)
#endif
#ifndef FLEXQ_AB_STPOL
#define FLEXQ_AB_STPOL 0    // write-back cache policy (A/B): 0 default, 1 L2 evict-last, 2 streaming
#endif
#ifndef FLEXQ_AB_QUANT
#define FLEXQ_AB_QUANT 1
#endif
#ifndef FLEXQ_AB_NEWCOPY
#define FLEXQ_AB_NEWCOPY 1
#endif
#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kMaxSplitUnits = 8192;   // partial slots in the workspace
constexpr int kMinSplitTokens = 128;  // smallest context split (two 64-token stages)
constexpr int kUnitsPerWarp = 0;       // occupancy splits off by default (B200 sweep):
                                       // split only where a context exceeds the score buffer
constexpr int kMinUnitTokens = 512;    // smallest per-warp score buffer of any variant (sizes the workspace)

// UNR: unroll factor of the full-stage loops (code size vs. scheduling freedom:
// fully unrolled K and V bodies overflow the instruction cache).
// MAXT: per-warp score buffer (tokens); longer contexts are split into units of <= MAXT.
template <int D, int NCH, int S, int WPC, int UNR, int MAXT>
__global__ void __launch_bounds__(WPC * 32, (16 / WPC) > 0 ? (16 / WPC) : 1)
decode_attention_kernel(const Params P) {
    using C = Cfg<D, NCH>;
    static_assert(S >= 2 && S <= 4, "ring depth");
    extern __shared__ __align__(128) uint8_t smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    uint8_t* ring = smem + warp * (S * C::STAGE);
    float* scores = reinterpret_cast<float*>(smem + WPC * S * C::STAGE) + warp * MAXT;
    uint32_t* limbs = reinterpret_cast<uint32_t*>(smem + WPC * (S * C::STAGE + MAXT * 4)) + warp * (kLimbWords<D, NCH>);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WPC * (S * C::STAGE + MAXT * 4 + kLimbWords<D, NCH> * 4)) +
                     warp * S;

    const int units = P.bh_total * P.nsplit;
    const uint64_t policy = evict_first_policy();
    // Programmatic dependent launch (NEXT-3 multi-layer decode): let the next layer's launch be
    // scheduled now (its CTAs become resident as this grid's retire) and, before touching any
    // global memory, wait for the previous grid in the stream to complete (a no-op when the
    // launch carried no programmatic dependency).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_proxy_async();
    }
    __syncwarp();
    asm volatile("griddepcontrol.wait;" ::: "memory");

    // Unit geometry: unit u = (b, h, split); tokens [first, first + len), nst stages per pass.
    auto geo = [&](int u, int& bh, int& first, int& len) {
        int split = 0;
        bh = u;
        if (P.nsplit > 1) {
            bh = u / P.nsplit;
            split = u - bh * P.nsplit;
        }
        first = split * P.split_len;
        len = min(P.cur_len - first, P.split_len);
    };

    // ---------------- producer (warp-uniform state; lane 0 issues the copies).
    // Stage sequence per unit: nst K stages, then nst V stages.  Unit ids go
    // through a 3-entry register FIFO to the consumer, which lags by <= S-1 stages.
    int p_unit = -1, p_stage = 0, p_nst = 0;
    const uint8_t* p_k = nullptr;   // first K chunk of the unit
    const uint8_t* p_v = nullptr;   // first V chunk
    const __half* p_q = nullptr;
    int p_len = 0;
    bool p_new = false;             // fused append: this unit holds token cur_len - 1
    int fq0 = -1, fq1 = -1, fq2 = -1, fcount = 0;
    auto next_unit = [&]() {
        int t = 0;
        if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
        t = __shfl_sync(0xffffffffu, t, 0);
        p_unit = t < units ? t : -1;
        p_stage = 0;
        if (p_unit >= 0) {
            int bh, first;
            geo(p_unit, bh, first, p_len);
            p_nst = (p_len + C::CH - 1) / C::CH;
            const int64_t c0 = int64_t(bh) * P.chunks + (first >> 5);
            p_k = P.kc + c0 * C::CHB;
            p_v = P.vc + c0 * C::CHB;
            p_q = P.q + int64_t(bh) * D;
            p_new = P.k_new != nullptr && first + p_len == P.cur_len;
        }
        if (fcount == 0) fq0 = p_unit; else if (fcount == 1) fq1 = p_unit; else fq2 = p_unit;
        ++fcount;
    };
    bool store_pending = false;     // a fused-append TMA store may still be reading a stage slot
    auto issue = [&](int slot) {
        if (lane == 0 && store_pending) {
            // the patched slot is refilled only after the bulk store has read it; waiting here
            // (one stage of math after the store was issued) instead of right after issuing it
            // takes the wait off the critical path
            bulk_wait_read0();
            store_pending = false;
        }
        if (p_unit < 0) {
            if (lane == 0) mbar_expect_tx(&bars[slot], 0);   // keeps the phase sequence; nothing to load
            return;
        }
        const bool vpass = p_stage >= p_nst;
        const int si = vpass ? p_stage - p_nst : p_stage;
        const int n = min(C::CH, p_len - si * C::CH);
        if (lane == 0) {
            const uint32_t bytes = uint32_t((n + kChunk - 1) / kChunk) * C::CHB;
            const bool first = p_stage == 0;
            uint8_t* sb = ring + slot * C::STAGE;
            const bool with_new = FLEXQ_AB_NEWCOPY && first && p_new;
            mbar_expect_tx(&bars[slot], bytes + (first ? 2 * D : 0) + (with_new ? 4 * D : 0));
            bulk_g2s(sb, (vpass ? p_v : p_k) + int64_t(si) * (NCH * C::CHB), bytes, &bars[slot], policy);
            if (first) bulk_g2s(sb + C::OFF_Q, p_q, 2 * D, &bars[slot], policy);
            if (with_new) {
                const int64_t row = (p_q - P.q);   // (b, h) * D
                bulk_g2s(sb + C::OFF_NEW, P.k_new + row, 2 * D, &bars[slot], policy);
                bulk_g2s(sb + C::OFF_NEW + 2 * D, P.v_new + row, 2 * D, &bars[slot], policy);
            }
        }
        if (++p_stage == 2 * p_nst) next_unit();
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
#if FLEXQ_V_MMA
    const VLane<D> vlane = v_lane<D, NCH>(lane);
#endif

    int slot = 0;
    uint32_t parity = 0;
    auto acquire = [&]() -> const uint8_t* {   // issue ahead, then wait for the current slot
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
        const int unit = fq0;              // pop the consumer's next unit
        fq0 = fq1;
        fq1 = fq2;
        --fcount;
        if (unit < 0) break;
        int bh, first, len;
        geo(unit, bh, first, len);
        const int nst = (len + C::CH - 1) / C::CH;

        // fused append: the unit holding token cur_len - 1 quantizes k_new / v_new (they
        // arrive with its first stage), stores them to the cache at once, and patches
        // the stage images of its last K and V stages before the math reads them
        const bool owns_new = P.k_new != nullptr && first + len == P.cur_len;
        const int new_idx = (P.cur_len - 1) - first - (nst - 1) * C::CH;   // inside the last stage
        const int new_slot = (P.cur_len - 1) & (kChunk - 1);
        TokenQ tq{};                       // lanes 0-15: the K row, 16-31: the V row
        // Patch the stage image, then write the patched bytes to the cache as whole
        // 16-B pieces: the token's K code row (or, for V, the whole 4-token quad row
        // the swizzled layout spreads it over) and the 32-B sector of the quad's
        // metadata.  Rewriting neighbours' unchanged bytes is harmless (no other
        // writer), and full-sector stores avoid partial-sector read-modify-writes.
        auto patch = [&](const uint8_t* sb, bool vpass) {
            uint8_t* s_chunk = const_cast<uint8_t*>(sb) + (new_idx >> 5) * C::CHB;
            if (vpass == (lane >= 16)) store_token<D>(tq, new_slot, s_chunk, lane);
            __syncwarp();
#if FLEXQ_AB_GSTORE == 2
            {   // lanes copy the patched 16-byte pieces to the cache with plain stores
                uint8_t* g_chunk = (vpass ? P.vc_w : P.kc_w) +
                                   (int64_t(bh) * P.chunks + ((P.cur_len - 1) >> 5)) * C::CHB;
                const int rows = vpass ? (new_slot >> 2) * 4 * C::CB : new_slot * C::CB;   // byte offset
                const int moff = C::OFF_M + (new_slot & ~3) * C::MB;                     // quad's meta
                const int nrow = (vpass ? 4 * C::CB : C::CB) / 16, nmeta = (4 * C::MB) / 16;
                uint8_t* gdst = nullptr;
                const uint8_t* ssrc = nullptr;
                if (lane < nrow) {
                    gdst = g_chunk + rows + 16 * lane;
                    ssrc = s_chunk + rows + 16 * lane;
                } else if (lane < nrow + nmeta) {
                    gdst = g_chunk + moff + 16 * (lane - nrow);
                    ssrc = s_chunk + moff + 16 * (lane - nrow);
                }
                if (gdst) {
                    const uint4 d = *reinterpret_cast<const uint4*>(ssrc);
#if FLEXQ_AB_STPOL == 1
                    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(gdst), "r"(d.x),
                                 "r"(d.y), "r"(d.z), "r"(d.w), "l"(evict_last_policy())
                                 : "memory");
#elif FLEXQ_AB_STPOL == 2
                    __stcs(reinterpret_cast<uint4*>(gdst), d);
#else
                    *reinterpret_cast<uint4*>(gdst) = d;
#endif
                }
            }
#elif FLEXQ_AB_GSTORE
            fence_proxy_async();   // the patch (generic writes) before the TMA store reads it
            __syncwarp();
            if (lane == 0) {
                uint8_t* g_chunk = (vpass ? P.vc_w : P.kc_w) +
                                   (int64_t(bh) * P.chunks + ((P.cur_len - 1) >> 5)) * C::CHB;
                const int rows = vpass ? (new_slot >> 2) * 4 * C::CB : new_slot * C::CB;   // byte offset
                const int moff = C::OFF_M + (new_slot & ~3) * C::MB;                     // quad's meta
                bulk_s2g(g_chunk + rows, s_chunk + rows, vpass ? 4 * C::CB : C::CB);
                bulk_s2g(g_chunk + moff, s_chunk + moff, 4 * C::MB);
                bulk_commit();
                store_pending = true;   // waited for before the slot's next bulk copy (issue)
            }
#endif
#if FLEXQ_AB_FENCE
            fence_proxy_async();   // generic smem writes before the slot's next bulk copy
#endif
            __syncwarp();
        };

        // ------------------------------------------------ pass 1: scores -> smem
        float M;
        {
            const uint8_t* sb = acquire();
            if (owns_new) {
#if FLEXQ_AB_QUANT
                tq = quantize_kv_token<D>(sb + C::OFF_NEW, lane);
#endif
                if (nst == 1) patch(sb, false);
            }
#if FLEXQ_K_MMA
            KFrag<D> kf;                      // the lane's q digits + epilogue weights for pass 1
            load_q_mma<D>(sb + C::OFF_Q, P.qscale, lane, kf);
            float mx = -INFINITY;
#pragma unroll 1
            for (int st = 0;;) {
                const int t0 = st * C::CH;
                const int n = min(C::CH, len - t0);
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
                if (owns_new && st == nst - 1) patch(sb, false);
            }
#else
            KQuery kq;                        // the lane's q for pass 1
            load_q(sb + C::OFF_Q + sg * 64, P.qscale, kq);
            float mx = -INFINITY;
#pragma unroll 1
            for (int st = 0;;) {
                const int t0 = st * C::CH;
                const int n = min(C::CH, len - t0);
                if (n == C::CH) {
#pragma unroll UNR
                    for (int i = 0; i < C::ITERS; ++i)
                        k_iter<D, NCH, true>(i, kq, sb, scores, t0, tl, n, lc, lm, sg, magic, mx);
                } else {
#pragma unroll UNR
                    for (int i = 0; i < C::ITERS; ++i)
                        if (i * C::TPI < n)
                            k_iter<D, NCH, false>(i, kq, sb, scores, t0, tl, n, lc, lm, sg, magic, mx);
                }
                release();
                if (++st == nst) break;
                sb = acquire();
                if (owns_new && st == nst - 1) patch(sb, false);
            }
#endif
#pragma unroll
            for (int o = C::LPT; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            M = mx;
        }

        // ------------------------------------------------ pass 2: P.V with p = 2^(s - M)
        // V codes are quad-interleaved (include/flexq.h): lanes own columns, IDP.4A over
        // 4 tokens at a time against per-stage fixed-point weights a_t = p_t scale_tg.
#if FLEXQ_V_MMA
        VAccM<D> va;
        va.init();
#pragma unroll 1
        for (int st = 0; st < nst; ++st) {
            const uint8_t* sb = acquire();
            if (owns_new && st == nst - 1) patch(sb, true);
            const int t0 = st * C::CH;
            const int n = min(C::CH, len - t0);
            v_stage_mma<D, NCH>(va, vlane, sb, scores + t0, M, n, lane, limbs);
            release();
        }

        // ------------------------------------------------ end of unit: combine, reduce, write
        float l;
        if (P.nsplit == 1) {
            v_finish_mma<D>(va, vlane, lane, P.out + int64_t(bh) * D, l, nullptr);
        } else {
            v_finish_mma<D>(va, vlane, lane, nullptr, l, P.part + int64_t(unit) * D);
#else
        VAcc<D> va;
        va.init();
#pragma unroll 1
        for (int st = 0; st < nst; ++st) {
            const uint8_t* sb = acquire();
            if (owns_new && st == nst - 1) patch(sb, true);
            const int t0 = st * C::CH;
            const int n = min(C::CH, len - t0);
            v_stage<D, NCH>(va, sb, scores + t0, M, n, lane, limbs);
            release();
        }

        // ------------------------------------------------ end of unit: reduce l / bias, write
        float v[32], l;
        const int col0 = va.finish(lane, v, l);
        if (P.nsplit == 1) {
            write_out<D>(P.out + int64_t(bh) * D + col0, v, l);
        } else {
            float* dst = P.part + int64_t(unit) * D + col0;
#pragma unroll
            for (int k = 0; k < D / 32; ++k) dst[k] = v[k];
#endif
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
        if (store_pending) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // before smem goes away
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
    return size_t(WPC) * (S * (Cfg<D, NCH>::STAGE + 8) + MAXT * 4 + kLimbWords<D, NCH> * 4);
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

// Split target in units per resident warp (FLEXQ_UNITS_PER_WARP overrides, tuning only).
int units_per_warp() {
    static int u = -1;
    if (u < 0) {
        const char* e = getenv("FLEXQ_UNITS_PER_WARP");
        u = e ? atoi(e) : kUnitsPerWarp;
        if (u < 0) u = 0;   // 0: split only where the score buffer forces it
    }
    return u;
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
    // context split: forced when a unit would exceed the score buffer; otherwise
    // (FLEXQ_UNITS_PER_WARP = u > 0, tuning) when there are fewer than u (b, h)
    // units per resident warp, keeping >= kMinSplitTokens tokens per split.  The
    // B200 sweep found occupancy splits slower at every BASELINE shape (the
    // partial write + merge costs more than the idle warps), so u = 0.
    const int min_split = (a.cur_len + MAXT - 1) / MAXT;
    int nsplit = min_split;
    const int64_t target = int64_t(units_per_warp()) * warps_resident;
    if (target > 0 && int64_t(bh) * nsplit < target) {
        nsplit = int((target + bh - 1) / bh);
        const int max_by_len = (a.cur_len + kMinSplitTokens - 1) / kMinSplitTokens;
        nsplit = min(nsplit, max_by_len);
        nsplit = int(std::min<int64_t>(nsplit, split_slots(bh, a.t_cap) / bh));
        nsplit = max(nsplit, min_split);
    } else if (target == 0 && int64_t(bh) * nsplit * 8 <= warps_resident) {
        // a small problem (>= 8 resident warps per unit, e.g. the tiny config's 48 heads) is
        // latency-bound on each warp's serial context walk: split the context down to one stage
        // per split (tiny: 14.95 -> 9.95 us at two stages per split).  Problems near one unit per warp
        // (OPT-6.7B's 2048 heads) stay unsplit: the partial write + merge costs more there.
        const int max_by_len = (a.cur_len + Cfg<D, NCH>::CH - 1) / Cfg<D, NCH>::CH;   // one stage per split
        nsplit = int(std::min<int64_t>({int64_t(max_by_len), split_slots(bh, a.t_cap) / bh,
                                        int64_t(warps_resident) / bh}));
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
    P.k_new = static_cast<const __half*>(a.k_new);
    P.v_new = static_cast<const __half*>(a.v_new);
    P.kc_w = static_cast<uint8_t*>(const_cast<void*>(a.k_cache));
    P.vc_w = static_cast<uint8_t*>(const_cast<void*>(a.v_cache));
    static const bool pdl = [] {
        const char* e = getenv("FLEXQ_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(ctas));
    cfg.blockDim = dim3(WPC * 32);
    cfg.dynamicSmemBytes = smem_bytes<D, NCH, S, WPC, MAXT>();
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, decode_attention_kernel<D, NCH, S, WPC, UNR, MAXT>, P);
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
            case FLEXQ_V(64, 2, 1, 4, 576): return launch<128, 2, 2, 1, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 3, 4, 576): return launch<128, 2, 2, 3, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 2, 8, 576): return launch<128, 2, 2, 2, 8, 576>(a, stream);
            case FLEXQ_V(64, 2, 2, 4, 1024): return launch<128, 2, 2, 2, 4, 1024>(a, stream);
            case FLEXQ_V(32, 3, 3, 4, 576): return launch<128, 1, 3, 3, 4, 576>(a, stream);
            case FLEXQ_V(32, 3, 1, 4, 576): return launch<128, 1, 3, 1, 4, 576>(a, stream);
            case FLEXQ_V(32, 2, 3, 4, 576): return launch<128, 1, 2, 3, 4, 576>(a, stream);
            case FLEXQ_V(32, 4, 2, 4, 576): return launch<128, 1, 4, 2, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 2, 4, 576): return launch<128, 2, 2, 2, 4, 576>(a, stream);
            case FLEXQ_V(64, 2, 3, 4, 1088): return launch<128, 2, 2, 3, 4, 1088>(a, stream);
            case FLEXQ_V(64, 2, 2, 4, 1088): return launch<128, 2, 2, 2, 4, 1088>(a, stream);
            default:   // B200 sweep: 2 warps / CTA; score buffer sized to the context
                return a.cur_len <= 576 ? launch<128, 2, 2, 2, 4, 576>(a, stream)
                                        : launch<128, 2, 2, 2, 4, 1088>(a, stream);
        }
    }
    switch (v) {
        case FLEXQ_V(64, 2, 4, 4, 1024): return launch<64, 2, 2, 4, 4, 1024>(a, stream);
        case FLEXQ_V(32, 3, 3, 4, 576): return launch<64, 1, 3, 3, 4, 576>(a, stream);
        case FLEXQ_V(64, 2, 2, 4, 576): return launch<64, 2, 2, 2, 4, 576>(a, stream);
        default: return launch<64, 2, 2, 3, 4, 576>(a, stream);
    }
}

}  // namespace flexq

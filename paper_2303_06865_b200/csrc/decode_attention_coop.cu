// decode_attention_coop.cu -- decode-step attention for launches with few heads (the small
// regime: OPT-6.7B, the N = 4 / N = 8 shards of OPT-175B), same method and arithmetic as
// decode_attention.cu (readings K, M; the fused append of NEXT-3).
//
// Why a second schedule: the one-warp-per-head kernel keeps at most two 64-token stages in flight
// per warp, so a launch with about one head per resident warp walks each head's ~17 stages at the
// memory latency and reaches ~4 TB/s.  Here a CTA streams ONE head at a time
// through a deep shared ring and splits its stages over several consumer warps:
//   * warp NC (the producer) takes heads by atomic tickets and issues, per head, its K stages then
//     its V stages into a kRing-stage ring (one cp.async.bulk per 64-token stage, a 16-byte
//     descriptor per slot: head, pass, stage, tokens); q (and, for the fused append, the new
//     token's K and V rows) go to the head's slot of two alternating head slots, on that slot's
//     own barrier;
//   * consumer warp w takes ring stages w, w + NC, ... of the CTA's stage stream.  K stages:
//     the tensor-core K pass (k_block_mma) into the head slot's shared score buffer and the slot's
//     max (shared atomicMax on order-preserving keys), then the slot's K counter.  V stages wait
//     until the head's K stages are all counted (the exact max is then known), run v_stage_mma into
//     the warp's own accumulators, and at the warp's last V stage of the head write an
//     unnormalised partial to the slot; the last of the head's V consumers sums the partials (all
//     share M, so no rescaling) and writes out, then frees the head slot for the producer;
//   * the fused append: the consumer of the head's last K stage quantizes the new token
//     (quantize_kv_token), patches that stage image and writes the K row back, and leaves the
//     quantized token in the slot for the consumer of the last V stage.
// Contexts must fit one score buffer (cur_len <= MAXT); the launcher falls back otherwise.
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "attn_common.cuh"
#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kNchC = 2;      // chunks per stage (64 tokens)
constexpr int kNC = 4;        // consumer warps per CTA
constexpr int kRing = 12;     // ring stages per CTA
constexpr int kThreadsC = (kNC + 1) * 32;

struct CoopParams {
    const __half* q;
    const uint8_t* kc;
    const uint8_t* vc;
    __half* out;
    uint32_t* ctrl;        // [0] head ticket, [1] retired CTAs (self-resetting)
    int bh_total, nck, nst, cur_len;
    int64_t chunks;
    float qscale;
    const __half* k_new;   // fused append of token cur_len - 1, or nullptr
    const __half* v_new;
    uint8_t* kc_w;
    uint8_t* vc_w;
};

// Stage descriptor, written by the producer into the ring slot's descriptor before the copy is
// issued (visible to the consumer through the slot's barrier).  bh < 0: end of the stream.
struct Desc {
    int bh;        // head (b * H + h)
    int info;      // bits 0-1 head slot, bit 2 V pass, bits 3-15 stage index, bits 16-30 head sequence
    int n;         // tokens in the stage
    int j0mod;     // (global index of the head's first V stage) mod kNC
};

template <int D, int MAXT>
struct CoopSmem {
    using C = Cfg<D, kNchC>;
    static constexpr int RING = 0;
    static constexpr int DESC = RING + kRing * C::STG;
    static constexpr int SLOT = DESC + kRing * 16;                  // two head slots
    // head slot layout
    static constexpr int S_X = 0;                                  // q | k_new | v_new (6 D bytes)
    static constexpr int S_SC = S_X + C::XTRA;                     // scores [MAXT]
    static constexpr int S_PART = S_SC + MAXT * 4;                 // partials [kNC][D] floats
    static constexpr int S_L = S_PART + kNC * D * 4;               // l per consumer [kNC]
    static constexpr int S_TQ = S_L + kNC * 4;                     // quantized new token [32] x 8 B
    static constexpr int S_CNT = S_TQ + 32 * 8;                    // max key, K count, V count
    static constexpr int SLOT_BYTES = (S_CNT + 16 + 127) / 128 * 128;
    static constexpr int LIMBS = SLOT + 2 * SLOT_BYTES;            // per consumer limb tables
    static constexpr int BARS = LIMBS + kNC * kLimbWords<D, kNchC> * 4;
    // barriers: full[kRing], empty[kRing], xbar[2], hfree[2]
    static constexpr int TOTAL = BARS + (2 * kRing + 4) * 8;
};

__device__ __forceinline__ uint32_t fkey(float f) {   // order-preserving unsigned key of a float
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ __forceinline__ void mbar_arrive_one(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

template <int D, int MAXT>
__global__ void __launch_bounds__(kThreadsC, 3) decode_attention_coop_kernel(const CoopParams P) {
    using C = Cfg<D, kNchC>;
    using L = CoopSmem<D, MAXT>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem + L::RING;
    Desc* desc = reinterpret_cast<Desc*>(smem + L::DESC);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BARS);
    uint64_t* full = bars;
    uint64_t* empty = bars + kRing;
    uint64_t* xbar = bars + 2 * kRing;
    uint64_t* hfree = bars + 2 * kRing + 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto slot_base = [&](int s) { return smem + L::SLOT + s * L::SLOT_BYTES; };

    if (threadIdx.x == 0) {
        for (int i = 0; i < kRing; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(xbar + s, 1);
            mbar_init(hfree + s, 1);
        }
        fence_proxy_async();
    }
    __syncthreads();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == kNC) {
        // ---------------- producer (the whole warp; elect.sync picks the issuing lane)
        const uint64_t policy = evict_first_policy();
        int j = 0;            // global stage index
        int hseq = 0;         // heads issued by this CTA
        for (;;) {
            int t = 0;
            if (lane == 0) t = int(atomicAdd(P.ctrl, 1u));
            t = __shfl_sync(0xffffffffu, t, 0);
            const int bh = t < P.bh_total ? t : -1;
            if (bh < 0) break;
            const int hs = hseq & 1;
            // the slot's previous head (hseq - 2) must be finished by the consumers
            if (hseq >= 2) mbar_wait(hfree + hs, uint32_t(((hseq >> 1) - 1) & 1));
            uint8_t* sl = slot_base(hs);
            if (lane == 0) {
                uint32_t* cnt = reinterpret_cast<uint32_t*>(sl + L::S_CNT);
                cnt[0] = 0u;     // max key (0 is below every key)
                cnt[1] = 0u;     // K stages done
                cnt[2] = 0u;     // V partials done
            }
            __syncwarp();
            const bool fused = P.k_new != nullptr;
            const int64_t row = int64_t(bh) * D;
            fence_proxy_async();
            mbar_expect_tx_elect(xbar + hs, fused ? 6 * D : 2 * D);
            bulk_g2s_elect(sl + L::S_X + C::XQ, P.q + row, 2 * D, xbar + hs, policy);
            if (fused) {
                bulk_g2s_elect(sl + L::S_X + C::XNEW, P.k_new + row, 2 * D, xbar + hs, policy);
                bulk_g2s_elect(sl + L::S_X + C::XNEW + 2 * D, P.v_new + row, 2 * D, xbar + hs, policy);
            }
            const uint8_t* kb = P.kc + int64_t(bh) * P.chunks * C::CHB;
            const uint8_t* vb = P.vc + int64_t(bh) * P.chunks * C::CHB;
            const int jv0 = j + P.nst;     // global index of the head's first V stage
            for (int pass = 0; pass < 2; ++pass) {
                for (int si = 0; si < P.nst; ++si, ++j) {
                    const int rs = j % kRing;
                    if (j >= kRing) mbar_wait(empty + rs, uint32_t(((j / kRing) - 1) & 1));
                    const int n = min(C::CH, P.cur_len - si * C::CH);
                    const int nchunks = (n + kChunk - 1) / kChunk;
                    if (lane == 0)
                        desc[rs] = Desc{bh, hs | (pass << 2) | (si << 3) | ((hseq & 0x7FFF) << 16), n, jv0 % kNC};
                    __syncwarp();
                    const uint32_t bytes = uint32_t(nchunks * C::CHB);
                    mbar_expect_tx_elect(full + rs, bytes);
                    bulk_g2s_elect(ring + rs * C::STG, (pass ? vb : kb) + int64_t(si) * C::STG, bytes, full + rs,
                                   policy);
                }
            }
            ++hseq;
        }
        // end of stream: one end descriptor per consumer
        for (int k = 0; k < kNC; ++k, ++j) {
            const int rs = j % kRing;
            if (j >= kRing) mbar_wait(empty + rs, uint32_t(((j / kRing) - 1) & 1));
            if (lane == 0) desc[rs] = Desc{-1, 0, 0, 0};
            __syncwarp();
            mbar_expect_tx_elect(full + rs, 0);   // an arrival, nothing to load
        }
    } else {
        // ---------------- consumers
        const int w = warp;
        const VLane<D> vlane = v_lane<D, kNchC>(lane);
        uint32_t* limbs = reinterpret_cast<uint32_t*>(smem + L::LIMBS) + w * kLimbWords<D, kNchC>;
        KFrag<D> kf;
        VAccM<D> va;
        int cur_head = -1;       // head sequence number whose q digits kf holds
        for (int j = w;; j += kNC) {
            const int rs = j % kRing;
            mbar_wait(full + rs, uint32_t((j / kRing) & 1));
            const Desc d = desc[rs];
            if (d.bh < 0) break;
            const int hs = d.info & 3, vpass = (d.info >> 2) & 1, si = (d.info >> 3) & 0x1FFF;
            const int hseq = (d.info >> 16) & 0x7FFF;
            uint8_t* sl = slot_base(hs);
            float* scores = reinterpret_cast<float*>(sl + L::S_SC);
            uint32_t* cnt = reinterpret_cast<uint32_t*>(sl + L::S_CNT);
            const uint8_t* sb = ring + rs * C::STG;
            const int t0 = si * C::CH;
            const bool last = si == P.nst - 1;
            const bool owns_new = P.k_new != nullptr && last;
            const int new_idx = (P.cur_len - 1) - t0;             // inside the last stage
            const int new_slot = (P.cur_len - 1) & (kChunk - 1);
            auto patch = [&](bool vp, const TokenQ& tq) {         // stage image + write-back (as decode_attention.cu)
                uint8_t* s_chunk = const_cast<uint8_t*>(sb) + (new_idx >> 5) * C::CHB;
                if (vp == (lane >= 16)) store_token<D>(tq, new_slot, s_chunk, lane);
                __syncwarp();
                uint8_t* g_chunk = (vp ? P.vc_w : P.kc_w) + (int64_t(d.bh) * P.chunks + ((P.cur_len - 1) >> 5)) * C::CHB;
                const int rows = vp ? (new_slot >> 2) * 4 * C::CB : new_slot * C::CB;
                const int moff = C::OFF_M + (new_slot & ~3) * C::MB;
                const int nrow = (vp ? 4 * C::CB : C::CB) / 16, nmeta = (4 * C::MB) / 16;
                int off = -1;
                if (lane < nrow) off = rows + 16 * lane;
                else if (lane < nrow + nmeta) off = moff + 16 * (lane - nrow);
                if (off >= 0) *reinterpret_cast<uint4*>(g_chunk + off) = *reinterpret_cast<const uint4*>(s_chunk + off);
                fence_proxy_async();   // generic smem writes before the slot's next bulk copy
                __syncwarp();
            };
            if (!vpass) {
                // ---- K stage: scores of its tokens, the slot max, the K count
                if (cur_head != hseq) {
                    // slot hs serves heads hs, hs + 2, ...: head hseq is its (hseq >> 1)-th use
                    mbar_wait(xbar + hs, uint32_t((hseq >> 1) & 1));
                    load_q_mma<D>(sl + L::S_X + C::XQ, P.qscale, lane, kf);
                    cur_head = hseq;
                }
                if (owns_new) {
                    const TokenQ tq = quantize_kv_token<D>(sl + L::S_X + C::XNEW, lane);
                    reinterpret_cast<TokenQ*>(sl + L::S_TQ)[lane] = tq;   // for the last V stage's consumer
                    patch(false, tq);
                }
                float mx = -INFINITY;
                if (d.n == C::CH) {
#pragma unroll
                    for (int b = 0; b < C::CH / 16; ++b) k_block_mma<D, kNchC>(b, kf, sb, scores, t0, C::CH, lane, mx);
                } else {
#pragma unroll
                    for (int b = 0; b < C::CH / 16; ++b)
                        if (b * 16 < d.n) k_block_mma<D, kNchC>(b, kf, sb, scores, t0, d.n, lane, mx);
                }
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();                      // scores (and the token) before the count
                    atomicMax(cnt + 0, fkey(mx));
                    __threadfence_block();
                    atomicAdd(cnt + 1, 1u);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive_one(empty + rs);
            } else {
                // ---- V stage: wait for the head's K stages, then P.V into this warp's accumulators
                if (lane == 0)
                    while (ld_volatile_u32(cnt + 1) < uint32_t(P.nst)) __nanosleep(64);
                __syncwarp();
                __threadfence_block();
                const float M = fkey_inv(ld_volatile_u32(cnt + 0));
                if (si < kNC) va.init();                        // this warp's first V stage of the head
                if (owns_new) patch(true, reinterpret_cast<const TokenQ*>(sl + L::S_TQ)[lane]);
                v_stage_mma<D, kNchC>(va, vlane, sb, scores + t0, M, d.n, lane, limbs);
                __syncwarp();
                if (lane == 0) mbar_arrive_one(empty + rs);
                if (si + kNC >= P.nst) {                        // this warp's last V stage of the head
                    float* part = reinterpret_cast<float*>(sl + L::S_PART) + w * D;
                    float l;
                    v_finish_mma<D>(va, vlane, lane, nullptr, l, part);
                    if (lane == 0) reinterpret_cast<float*>(sl + L::S_L)[w] = l;
                    __syncwarp();
                    uint32_t done = 0;
                    if (lane == 0) {
                        __threadfence_block();
                        done = atomicAdd(cnt + 2, 1u) + 1u;
                        __threadfence_block();
                    }
                    done = __shfl_sync(0xffffffffu, done, 0);
                    const uint32_t nv = uint32_t(min(P.nst, kNC));   // warps holding a partial
                    if (done == nv) {
                        // sum the partials (one per participating warp, all with the same M); the
                        // participating warps are those of V stages 0 .. nv - 1
                        constexpr int CPL = D / 32;
                        const float* parts = reinterpret_cast<const float*>(sl + L::S_PART);
                        const float* ls = reinterpret_cast<const float*>(sl + L::S_L);
                        float num[CPL];
#pragma unroll
                        for (int c = 0; c < CPL; ++c) num[c] = 0.0f;
                        float den = 0.0f;
                        for (int k = 0; k < int(nv); ++k) {    // stage order: deterministic
                            const int ww = (d.j0mod + k) % kNC;
                            den += ls[ww];
#pragma unroll
                            for (int c = 0; c < CPL; ++c) num[c] += parts[ww * D + CPL * lane + c];
                        }
                        const float inv = 1.0f / den;
                        __half* o = P.out + int64_t(d.bh) * D + CPL * lane;
                        if constexpr (CPL == 4) {
                            const __half2 h0 = __floats2half2_rn(num[0] * inv, num[1] * inv);
                            const __half2 h1 = __floats2half2_rn(num[2] * inv, num[3] * inv);
                            uint2 u;
                            u.x = *reinterpret_cast<const uint32_t*>(&h0);
                            u.y = *reinterpret_cast<const uint32_t*>(&h1);
                            *reinterpret_cast<uint2*>(o) = u;
                        } else {
                            *reinterpret_cast<__half2*>(o) = __floats2half2_rn(num[0] * inv, num[1] * inv);
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive_one(hfree + hs);   // the slot may take the next head
                    }
                }
            }
        }
        // the fused append's K write-back used generic stores to the cache; the V stores likewise:
        // nothing further (no cross-CTA reads of them in this launch)
    }

    // retire: the last CTA out resets the head ticket
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(P.ctrl + 1, 1u) == gridDim.x - 1) {
            P.ctrl[0] = 0u;
            P.ctrl[1] = 0u;
            __threadfence();
        }
    }
}

template <int D, int MAXT>
cudaError_t launch_coop(const AttnArgs& a, cudaStream_t stream) {
    using L = CoopSmem<D, MAXT>;
    auto k = decode_attention_coop_kernel<D, MAXT>;
    static int occs[kMaxDevices];
    static std::once_flag once[kMaxDevices];
    const int dev = current_device();
    std::call_once(once[dev], [&] {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::TOTAL));
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, kThreadsC, L::TOTAL);
        occs[dev] = o > 0 ? o : 1;
    });
    const int bh = a.batch * a.heads;
    CoopParams P;
    P.q = static_cast<const __half*>(a.q);
    P.kc = static_cast<const uint8_t*>(a.k_cache);
    P.vc = static_cast<const uint8_t*>(a.v_cache);
    P.out = static_cast<__half*>(a.out);
    P.ctrl = static_cast<uint32_t*>(a.workspace);
    P.bh_total = bh;
    P.nck = (a.cur_len + kChunk - 1) / kChunk;
    P.nst = (P.nck + kNchC - 1) / kNchC;
    P.cur_len = a.cur_len;
    P.chunks = a.chunks;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    P.k_new = static_cast<const __half*>(a.k_new);
    P.v_new = static_cast<const __half*>(a.v_new);
    P.kc_w = static_cast<uint8_t*>(const_cast<void*>(a.k_cache));
    P.vc_w = static_cast<uint8_t*>(const_cast<void*>(a.v_cache));
    const int grid = std::max(1, std::min(bh, device_sm_count() * occs[dev]));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(kThreadsC);
    cfg.dynamicSmemBytes = L::TOTAL;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, P);
}

}  // namespace

bool coop_attention_fits(int head_dim, int cur_len) { return cur_len <= (head_dim == 128 ? 576 : 576); }

cudaError_t launch_decode_attention_coop(const AttnArgs& a, cudaStream_t stream) {
    if (a.head_dim == 128) return launch_coop<128, 576>(a, stream);
    return launch_coop<64, 576>(a, stream);
}

}  // namespace flexq

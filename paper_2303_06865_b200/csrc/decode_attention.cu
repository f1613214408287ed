// decode_attention.cu -- decode-step attention over the 4-bit group-wise
// compressed KV cache, dequantization fused in registers (sm_100a).
//
// Computes, per (batch, head) (readings K, M):
//   out = softmax(q . K^[0:cur_len]^T / sqrt(D)) . V^[0:cur_len],
//   K^_tj = fmaf(c_tj, scale_tg, min_tg) in fp32 (never rounded to fp16).
//
// Design ("decode_attention_kernel"):
//  * Persistent kernel, one warp per CTA, every warp resident.  Work items are
//    handed out by an atomic ticket (fetched one item ahead, so its latency hides
//    behind the current item): first whole (b, h) heads, then -- for the last
//    heads, about one per warp -- pieces of a head (a contiguous run of its
//    32-token chunks).  Fast SMs take more items, and the end of the launch is cut
//    into small pieces, so no SM idles while another finishes a whole head (the
//    per-SM streaming rate differs by up to ~6-15 % on B200).
//  * A piece writes (acc, m, l) partials; the last piece of its head to finish (a
//    per-head ticket) merges them in piece order with the log-sum-exp rule
//    (online-softmax combine) and resets the ticket: results are deterministic.
//    Contexts longer than the score buffer (MAXT tokens) are split the same way.
//  * Each warp owns a 2-stage shared-memory ring.  A stage is 2 consecutive
//    32-token chunks of the K cache (pass 1) or of the V cache (pass 2) -- codes
//    + fp16 (scale, min), one contiguous run in HBM -- loaded with a single 1-D
//    TMA bulk copy (cp.async.bulk -> mbarrier complete_tx); q (and, for the fused
//    append, the new token's k and v rows) rides with an item's first stage into
//    the warp's extra area.  Loads run one stage ahead of the math, across items;
//    elect.sync picks the lane that issues.
//  * Two passes per item, no online rescaling: pass 1 streams the K stages and
//    writes every score (log2 domain) to the warp's smem score buffer; pass 2
//    takes the exact max, streams the V stages and accumulates p_t = 2^(s_t - M).
//    Both passes run on the tensor cores as exact integer MMAs (attn_common.cuh).
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "attn_common.cuh"
#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kNch = 2;             // chunks per stage (64 tokens)
constexpr int kMaxWarps = 4096;     // grid cap
constexpr int kMaxPieces = 32;      // pieces per head (partial slots per head)
constexpr int kMinPieceChunks = 2;  // smallest piece
constexpr int kCtasPerSm = 16;      // one-warp CTAs resident per SM (register / smem budget)
constexpr int kPfWholeHeadsPerWarp = 3;   // from this many items per warp the L2 prefetch takes the whole first K pass
constexpr int kMaxCtrs = 16;        // ticket counters, 64 B apart in the 1 KB control block
constexpr int kRetire = 16 * kMaxCtrs;

#ifndef FLEXQ_ATTN_L2PF
#define FLEXQ_ATTN_L2PF 2            // K stages of the first item prefetched to L2 before griddepcontrol.wait (0: off)
#endif
#ifndef FLEXQ_ATTN_TRACE
#define FLEXQ_ATTN_TRACE 0           // 1: per-warp %globaltimer stamps of the last launch (tuning build)
#endif
#if FLEXQ_ATTN_TRACE
__device__ unsigned long long g_attn_trace[kMaxWarps][4];   // resident, after wait, end, pieces
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

struct Params {
    const __half* q;
    const uint8_t* kc;     // chunked K cache
    const uint8_t* vc;     // chunked V cache
    __half* out;
    uint32_t* ctrl;        // [0, nctr) ticket counters, [63] retired warps (self-resetting)
    uint32_t* tickets;     // per (b, h): finished pieces (self-resetting)
    float* part;           // [bh][kMaxPieces][D] unnormalised partial outputs
    float2* ml;            // [bh][kMaxPieces] (m, l) of each partial
    int nck;               // chunks per head
    // Two phases: a static stream-K prefix over heads [0, hs), then ticket items over heads [hs, bh)
    // ("Schedule").  Either may be empty.
    int total;             // static: hs nck chunks, warp w owns [w total / W, (w+1) total / W)
    int wq, wr;            // static: total = wq W + wr
    int maxch;             // static: most chunks per piece (score buffer)
    int hs;                // first ticket head
    int na, ka;            // tickets, part A: heads [hs, hs + na), ka pieces each (ka > 1 only past the score buffer)
    int kb;                // tickets, part B: heads [hs + na, bh), kb pieces each
    int items;             // na ka + (bh - hs - na) kb
    int nctr;              // ticket counters: warp w draws items c, c + nctr, ... from counter c = w % nctr
                           // (spreads the same-address atomics of a launch over nctr L2 lines)
    int64_t chunks;        // chunk stride per (b, h) in the cache
    int cur_len;
    float qscale;          // log2(e) / sqrt(D)
    const __half* k_new;   // fused append (NEXT-3): token cur_len - 1 of every (b, h), [B H][D];
    const __half* v_new;   //   nullptr = the cache already holds it
    uint8_t* kc_w;         // writable aliases of kc / vc for the fused append
    uint8_t* vc_w;
    int pf_chunks;         // K chunks of the first item prefetched to L2 before griddepcontrol.wait
};

// Work item t: piece k of np of head bh = chunks [o, o + nch) (np = 1: the whole head).
struct Piece {
    int bh, o, nch, k, np;
};
__device__ __forceinline__ bool decode_item(const Params& P, int t, Piece& p) {
    if (t >= P.items) return false;
    const int ta = P.na * P.ka;
    const bool in_a = t < ta;
    const int np = in_a ? P.ka : P.kb;
    const int tt = in_a ? t : t - ta;
    const int h = np == 1 ? tt : tt / np;   // whole heads (np = 1: every BASELINE launch but tiny) skip the divisions
    p.np = np;
    p.k = tt - h * np;
    p.bh = P.hs + (in_a ? 0 : P.na) + h;
    p.o = np == 1 ? 0 : p.k * P.nck / np;
    p.nch = np == 1 ? P.nck : (p.k + 1) * P.nck / np - p.o;
    return true;
}

// Static mode: first chunk of warp w's range, floor(w total / W) without 64-bit arithmetic.
__device__ __forceinline__ int range_start(const Params& P, int w, int W) {
    return w * P.wq + (w * P.wr) / W;
}
// Static mode: the piece starting at global chunk c of a warp whose range ends at r1 --
// cut at the head's end and every maxch chunks.
__device__ __forceinline__ void static_piece(const Params& P, int c, int r1, Piece& p) {
    p.bh = c / P.nck;
    p.o = c - p.bh * P.nck;
    p.nch = min(min(r1, (p.bh + 1) * P.nck), c + P.maxch) - c;
    p.k = 0;
    p.np = (p.o == 0 && p.nch == P.nck) ? 1 : 0;   // 0: a piece; index / count by head_pieces
}
// Static mode: index of the piece of head bh that starts at chunk offset o, and the head's
// piece count -- the warp segments of the head, each cut every maxch chunks from its start
// (the cuts static_piece makes).  A pure function of the launch: the merge order is fixed.
__device__ int head_pieces(const Params& P, int W, int bh, int o, int& count) {
    const int h0 = bh * P.nck, h1 = h0 + P.nck;
    int w = int((int64_t(h0 + 1) * W - 1) / P.total);   // the warp owning chunk h0
    int idx = 0, found = -1;
    for (;;) {
        const int s = max(range_start(P, w, W), h0), e = min(range_start(P, w + 1, W), h1);
        if (e > s) {
            if (found < 0 && h0 + o >= s && h0 + o < e) found = idx + (h0 + o - s) / P.maxch;
            idx += (e - s + P.maxch - 1) / P.maxch;
        }
        if (e >= h1) break;
        ++w;
    }
    count = idx;
    return found;
}

// S: ring depth (stages in flight ahead of the math: S - 1).  The extra area (q, k_new, v_new)
// is refilled at the next item's first stage; with S = 2 that issue comes after the previous item
// has read its rows (every item has >= 2 stages), deeper rings use two extra areas, alternating.
template <int S>
constexpr int kXtraBufs = S > 2 ? 2 : 1;

template <int D, int MAXT, int S, int NCH>
__global__ void __launch_bounds__(32, kCtasPerSm) decode_attention_kernel(const Params P) {
    using C = Cfg<D, NCH>;
    constexpr int NX = kXtraBufs<S>;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x;
    uint8_t* ring = smem;
    uint8_t* xtra0 = smem + S * C::STG;   // NX extra areas
    float* scores = reinterpret_cast<float*>(xtra0 + NX * C::XTRA);
    uint32_t* limbs = reinterpret_cast<uint32_t*>(scores + MAXT);
    uint64_t* bars = reinterpret_cast<uint64_t*>(limbs + kLimbWords<D, NCH>);   // S stages, then NX extra

    const uint64_t policy = evict_first_policy();
    // Programmatic dependent launch (NEXT-3 multi-layer decode): let the next layer's launch be
    // scheduled now (its CTAs become resident as this grid's retire) and, before touching any
    // global memory, wait for the previous grid in the stream to complete (a no-op when the
    // launch carried no programmatic dependency).
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#if FLEXQ_ATTN_TRACE
    const unsigned long long t_res = gtime();
#endif
    if (lane == 0) {
        for (int s = 0; s < S + NX; ++s) mbar_init(&bars[s], 1);   // S stage barriers + the extra areas'
        fence_proxy_async();
    }
    __syncwarp();
#if FLEXQ_ATTN_L2PF
    // Before waiting for the previous grid, pull the warp's first item's first K stages into L2 (a
    // prefetch is safe whatever that grid writes: L2 is the point of coherence), so the launch's
    // ramp starts from L2: batch 18 26.6 -> 25.9 us, OPT-6.7B 30.8 -> 30.1 us, batch 144 unchanged
    // (r3g; in round 1, before the residency cap, the same prefetch lost)
    if (P.total == 0 && P.items > 0 && lane == 0) {
        Piece f;
        if (decode_item(P, int(blockIdx.x), f)) {
            const uint8_t* src = P.kc + (int64_t(f.bh) * P.chunks + f.o) * C::CHB;
            const uint32_t bytes = uint32_t(min(f.nch, P.pf_chunks)) * C::CHB;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
        }
    }
#endif
    asm volatile("griddepcontrol.wait;" ::: "memory");
#if FLEXQ_ATTN_TRACE
    const unsigned long long t_go = gtime();
    int n_pieces = 0;
#endif

    // ---------------- producer (warp-uniform): per item nst K stages, then nst V stages.
    // The next ticket is fetched one item ahead (lane 0 holds the raw atomic result
    // until it is needed); item ids go through a 3-entry FIFO to the consumer, which
    // lags by at most one stage.
    // Item ids: a static piece is its first chunk c < P.total; ticket t is P.total + t.  The
    // first ticket is fetched when the warp hands out its last static piece (or at the start,
    // if its static range is empty), then always one item ahead.
    const int W = gridDim.x;
    const int r0 = range_start(P, blockIdx.x, W);
    const int r1 = range_start(P, blockIdx.x + 1, W);
    int p_cur = r0;                        // the producer's next static chunk
    uint32_t tk_raw = 0;
    const int ctr = int(blockIdx.x) % P.nctr;
    // Pure ticket launches (no static prefix; grid <= items): warp w's first item is ticket w, the
    // counters deal tickets grid, grid + 1, ... from then on.  (When every warp drew its first
    // ticket from the counters too, the prefetch of a fast warp's second ticket could take a slow
    // warp's first: with about one head per warp that warp idled while another walked two heads.)
    bool tk_static = P.total == 0 && P.items > 0;
    const int tk_base = P.total == 0 ? int(gridDim.x) : 0;
    if (!tk_static && r0 >= r1 && P.items > 0 && lane == 0) tk_raw = atomicAdd(P.ctrl + 16 * ctr, 1u);
    Piece pp{0, 0, 0, 0, 1};
    bool p_valid = false, p_new = false;
    int p_stage = 0, p_nst = 0, p_last = 0;
    const uint8_t* p_k = nullptr;
    const uint8_t* p_v = nullptr;
    int fq0 = -1, fq1 = -1, fq2 = -1, fq3 = -1, fcount = 0;
    int p_items = 0;                       // valid items issued (selects the extra area)
    auto p_next = [&]() {
        int t;
        if (p_cur < r1) {
            t = p_cur;
            static_piece(P, p_cur, r1, pp);
            p_cur += pp.nch;
            p_valid = true;
            if (p_cur >= r1 && P.items > 0 && lane == 0) tk_raw = atomicAdd(P.ctrl + 16 * ctr, 1u);
        } else {
            const int tk = tk_static ? int(blockIdx.x) : int(__shfl_sync(0xffffffffu, tk_raw, 0)) * P.nctr + ctr + tk_base;
            tk_static = false;
            p_valid = P.items > 0 && decode_item(P, tk, pp);
            if (lane == 0 && p_valid) tk_raw = atomicAdd(P.ctrl + 16 * ctr, 1u);   // prefetch the following ticket
            t = P.total + tk;
        }
        p_stage = 0;
        if (p_valid) {
            p_nst = (pp.nch + NCH - 1) / NCH;
            p_last = pp.nch - NCH * (p_nst - 1);
            const int64_t c0 = int64_t(pp.bh) * P.chunks + pp.o;
            p_k = P.kc + c0 * C::CHB;
            p_v = P.vc + c0 * C::CHB;
            p_new = P.k_new != nullptr && pp.o + pp.nch == P.nck;
        }
        const int id = p_valid ? t : -1;
        if (fcount == 0) fq0 = id; else if (fcount == 1) fq1 = id; else if (fcount == 2) fq2 = id; else fq3 = id;
        ++fcount;
    };
    auto issue = [&](int slot) {
        if (!p_valid) {
            mbar_expect_tx_elect(&bars[slot], 0);   // keeps the phase sequence; nothing to load
            return;
        }
        const bool vpass = p_stage >= p_nst;
        const int si = vpass ? p_stage - p_nst : p_stage;
        const uint32_t bytes = uint32_t(si == p_nst - 1 ? p_last : NCH) * C::CHB;
        const bool first = p_stage == 0;
        // the extra area (q, k_new, v_new) is rewritten by the async proxy for the next item: order
        mbar_expect_tx_elect(&bars[slot], bytes);
        bulk_g2s_elect(ring + slot * C::STG, (vpass ? p_v : p_k) + int64_t(si) * C::STG, bytes, &bars[slot], policy);
        if (first) {
            // the item's rows (q; k_new, v_new for the fused append) complete on the extra area's own
            // barrier, one phase per item: the previous item read them before this item's first
            // stage is issued (one stage ahead), and both the writes and the reads of every item are
            // ordered through the same barrier's phases
            const int64_t row = int64_t(pp.bh) * D;
            const int xb = NX == 1 ? 0 : (p_items & 1);
            uint8_t* xt = xtra0 + xb * C::XTRA;
            uint64_t* xbar = &bars[S + xb];
            ++p_items;
            fence_proxy_async();
            mbar_expect_tx_elect(xbar, p_new ? 6 * D : 2 * D);
            bulk_g2s_elect(xt + C::XQ, P.q + row, 2 * D, xbar, policy);
            if (p_new) {
                bulk_g2s_elect(xt + C::XNEW, P.k_new + row, 2 * D, xbar, policy);
                bulk_g2s_elect(xt + C::XNEW + 2 * D, P.v_new + row, 2 * D, xbar, policy);
            }
        }
        if (++p_stage == 2 * p_nst) p_next();
    };
    p_next();
#pragma unroll
    for (int s = 0; s < S - 1; ++s) issue(s);

    // ---------------- consumer: the same item sequence, one stage behind
    const VLane<D> vlane = v_lane<D, NCH>(lane);
    int slot = 0, c_items = 0;
    uint32_t parity = 0, xparity = 0;      // xparity: bit b = phase of extra area b
    auto acquire = [&]() -> const uint8_t* {   // issue S - 1 stages ahead, then wait for the current slot
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

    Piece pc;
#pragma unroll 1
    for (;;) {
        const int item = fq0;              // pop the consumer's next item
        fq0 = fq1;
        fq1 = fq2;
        fq2 = fq3;
        --fcount;
        if (item < 0) break;
        if (item >= P.total) decode_item(P, item - P.total, pc);
        else static_piece(P, item, r1, pc);
#if FLEXQ_ATTN_TRACE
        ++n_pieces;
#endif
        const int bh = pc.bh;
        const int first = pc.o * kChunk;
        const int len = min(P.cur_len - first, pc.nch * kChunk);
        const int nst = (pc.nch + NCH - 1) / NCH;

        // fused append: the piece holding token cur_len - 1 quantizes k_new / v_new (they
        // arrive with its first stage), and patches the stage images of its last K and V
        // stages before the math reads them, writing the patched pieces to the cache
        const bool owns_new = P.k_new != nullptr && pc.o + pc.nch == P.nck;
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
            uint8_t* g_chunk = (vpass ? P.vc_w : P.kc_w) + (int64_t(bh) * P.chunks + ((P.cur_len - 1) >> 5)) * C::CHB;
            const int rows = vpass ? (new_slot >> 2) * 4 * C::CB : new_slot * C::CB;   // byte offset
            const int moff = C::OFF_M + (new_slot & ~3) * C::MB;                     // quad's meta
            const int nrow = (vpass ? 4 * C::CB : C::CB) / 16, nmeta = (4 * C::MB) / 16;
            int off = -1;
            if (lane < nrow) off = rows + 16 * lane;
            else if (lane < nrow + nmeta) off = moff + 16 * (lane - nrow);
            if (off >= 0) *reinterpret_cast<uint4*>(g_chunk + off) = *reinterpret_cast<const uint4*>(s_chunk + off);
            fence_proxy_async();   // generic smem writes before the slot's next bulk copy
            __syncwarp();
        };

        // ------------------------------------------------ pass 1: scores -> smem
        float M;
        {
            const uint8_t* sb = acquire();
            const int xb = NX == 1 ? 0 : (c_items & 1);   // the item's q (and new token's rows)
            const uint8_t* xt = xtra0 + xb * C::XTRA;
            ++c_items;
            mbar_wait(&bars[S + xb], (xparity >> xb) & 1u);
            xparity ^= 1u << xb;
            if (owns_new) {
                tq = quantize_kv_token<D>(xt + C::XNEW, lane);
                if (nst == 1) patch(sb, false);
            }
            KFrag<D> kf;                      // the lane's q digits + epilogue weights for pass 1
            load_q_mma<D>(xt + C::XQ, P.qscale, lane, kf);
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
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            M = mx;
        }

        // ------------------------------------------------ pass 2: P.V with p = 2^(s - M)
        VAccM<D> va;
        va.init();
#pragma unroll 1
        for (int st = 0; st < nst; ++st) {
            const uint8_t* sb = acquire();
            if (owns_new && st == nst - 1) patch(sb, true);
            const int t0 = st * C::CH;
            v_stage_mma<D, NCH>(va, vlane, sb, scores + t0, M, min(C::CH, len - t0), lane, limbs);
            release();
        }

        // ------------------------------------------------ end of item
        float l;
        if (pc.np == 1) {
            v_finish_mma<D>(va, vlane, lane, P.out + int64_t(bh) * D, l, nullptr);
            continue;
        }
        // a piece: store the partial, then count its tokens on the head's ticket (release: the
        // partial stores of every lane happen before the increment, through the warp barrier);
        // the piece that completes the count merges all of them in piece order (deterministic)
        int np = pc.np, k = pc.k;
        if (np == 0) k = head_pieces(P, W, bh, pc.o, np);
        const int64_t slot0 = int64_t(bh) * kMaxPieces;
        v_finish_mma<D>(va, vlane, lane, nullptr, l, P.part + (slot0 + k) * D);
        if (lane == 0) P.ml[slot0 + k] = make_float2(M, l);
        __syncwarp();
        uint32_t done = 0;
        if (lane == 0) {
            // release-add (MEMBAR, no L1 invalidation: a full fence.acq_rel here was the largest
            // single stall of the small-batch launches, ncu); only the merging piece acquires
            uint32_t old;
            asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(&P.tickets[bh]), "r"(uint32_t(len))
                         : "memory");
            done = old + uint32_t(len);
            if (done == uint32_t(P.cur_len)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        done = __shfl_sync(0xffffffffu, done, 0);
        if (done == uint32_t(P.cur_len)) {   // every piece of this (b, h) is in: merge
            // all loads are independent (no serial round trips): lane i < np holds piece i's
            // (m, l); lane c owns columns 4c .. 4c + 3 (D = 128) or 2c, 2c + 1 (D = 64)
            constexpr int CPL = D / 32;
            const float2 mli = lane < np ? __ldcg(&P.ml[slot0 + lane]) : make_float2(-INFINITY, 0.0f);
            float Mx = mli.x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) Mx = fmaxf(Mx, __shfl_xor_sync(0xffffffffu, Mx, o));
            const float wi = lane < np ? ex2(mli.x - Mx) : 0.0f;
            float den = wi * mli.y;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
            float num[CPL];
#pragma unroll
            for (int c = 0; c < CPL; ++c) num[c] = 0.0f;
#pragma unroll 4
            for (int i = 0; i < np; ++i) {
                const float w = __shfl_sync(0xffffffffu, wi, i);
                const float* pr = P.part + (slot0 + i) * D + CPL * lane;
                if constexpr (CPL == 4) {
                    const float4 v = __ldcg(reinterpret_cast<const float4*>(pr));
                    num[0] = fmaf(w, v.x, num[0]);
                    num[1] = fmaf(w, v.y, num[1]);
                    num[2] = fmaf(w, v.z, num[2]);
                    num[3] = fmaf(w, v.w, num[3]);
                } else {
                    const float2 v = __ldcg(reinterpret_cast<const float2*>(pr));
                    num[0] = fmaf(w, v.x, num[0]);
                    num[1] = fmaf(w, v.y, num[1]);
                }
            }
            const float inv = 1.0f / den;
            __half* o = P.out + int64_t(bh) * D + CPL * lane;
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
            if (lane == 0) P.tickets[bh] = 0u;   // leave the workspace zeroed
        }
    }

    // retire: the last warp out resets the item ticket for the next call
    if (P.items > 0 && lane == 0) {
        __threadfence();
        if (atomicAdd(P.ctrl + kRetire, 1u) == gridDim.x - 1) {
            for (int c = 0; c < P.nctr; ++c) P.ctrl[16 * c] = 0u;
            P.ctrl[kRetire] = 0u;
            __threadfence();
        }
    }
#if FLEXQ_ATTN_TRACE
    if (lane == 0 && blockIdx.x < kMaxWarps) {
        g_attn_trace[blockIdx.x][0] = t_res;
        g_attn_trace[blockIdx.x][1] = t_go;
        g_attn_trace[blockIdx.x][2] = gtime();
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        g_attn_trace[blockIdx.x][3] = (unsigned long long)n_pieces | ((unsigned long long)smid << 32);
    }
#endif
}

template <int D, int MAXT, int S, int NCH>
constexpr size_t smem_bytes() {
    return size_t(S) * Cfg<D, NCH>::STG + kXtraBufs<S> * Cfg<D, NCH>::XTRA + MAXT * 4 + kLimbWords<D, NCH> * 4 +
           (S + kXtraBufs<S>) * 8;
}

// Per-device launch facts (the SM count and the kernel's occupancy), computed once per
// device under a lock: the library keeps no other state.
struct DevInfo {
    int sms = 0;
    int occ = 0;
    int cap_smem[kCtasPerSm + 1] = {};   // [r]: dynamic smem that leaves at most r CTAs resident per SM
};
template <int D, int MAXT, int S, int NCH>
const DevInfo& dev_info() {
    constexpr int kMaxDev = 64;
    static DevInfo info[kMaxDev];
    static std::once_flag once[kMaxDev];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev) dev = 0;
    std::call_once(once[dev], [dev] {
        auto k = decode_attention_kernel<D, MAXT, S, NCH>;
        constexpr int need = int(smem_bytes<D, MAXT, S, NCH>());
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        optin = std::max(optin, need);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
        int sms = 0, o = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, 32, need);
        DevInfo& d = info[dev];
        d.sms = sms > 0 ? sms : 148;
        d.occ = o > 0 ? o : 1;
        // the smallest dynamic smem (a multiple of 128 B) at which at most r CTAs fit on an SM
        for (int r = 1; r <= kCtasPerSm; ++r) {
            int lo = need, hi = optin;
            int best = need;
            while (lo <= hi) {
                const int mid = (lo + hi) / 2 / 128 * 128;
                int om = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&om, k, 32, std::max(mid, need));
                if (om > r) {
                    lo = mid + 128;
                } else {
                    best = std::max(mid, need);
                    hi = mid - 128;
                }
            }
            d.cap_smem[r] = best;
        }
        cudaGetLastError();
    });
    return info[dev];
}

struct WsLayout {
    size_t ctrl, tickets, part, ml, total;
};
WsLayout ws_layout(int bh, int d) {
    WsLayout w;
    w.ctrl = 0;
    w.tickets = 2048;   // after the 2 KB control block (ticket counters 64 B apart, the retire count)
    w.part = (w.tickets + size_t(bh) * 4 + 255) / 256 * 256;
    w.ml = w.part + size_t(bh) * kMaxPieces * d * 4;
    w.total = w.ml + size_t(bh) * kMaxPieces * 8;
    return w;
}

// Scheduler tuning (environment, A/B sweeps only):
//   FLEXQ_ATTN_SPLIT="<min heads per warp x 100 for all-ticket mode>,<tail heads per warp x 100>,<pieces per tail head>"
//   FLEXQ_ATTN_HYBRID="<static share of the heads, %>,<chunks per ticket piece>"
//   FLEXQ_ATTN_CTRS=<ticket counters, 1..16>
constexpr int kDynHeadsPerWarpX100 = 50;    // B200 sweep: whole-head tickets win from ~0.5 heads per warp
                                            // (batch 18 / 36 shards of OPT-175B: 33 / 55 us vs 37.7 / 59.7 static)
constexpr int kHybridStaticPct = 100;       // below that: static stream-K (the static-prefix + ticket-piece
                                            // hybrid measured slower at every share; tuning only)
constexpr int kHybridPieceChunks = 3;
void tune_split(int& dyn_min_x100, int& nb_per_warp_x100, int& kb, int& hyb_pct, int& hyb_q) {
    static int v[5] = {-1, -1, -1, -1, -1};
    static std::once_flag once;
    std::call_once(once, [] {
        if (const char* e = getenv("FLEXQ_ATTN_SPLIT")) sscanf(e, "%d,%d,%d", &v[0], &v[1], &v[2]);
        if (const char* e = getenv("FLEXQ_ATTN_HYBRID")) sscanf(e, "%d,%d", &v[3], &v[4]);
    });
    if (v[0] >= 0) dyn_min_x100 = v[0];
    if (v[1] >= 0) nb_per_warp_x100 = v[1];
    if (v[2] > 0) kb = v[2];
    if (v[3] >= 0) hyb_pct = v[3];
    if (v[4] > 0) hyb_q = v[4];
}

template <int D, int MAXT, int S, int NCH>
cudaError_t launch(const AttnArgs& a, cudaStream_t stream) {
    const int bh = a.batch * a.heads;
    const DevInfo di = dev_info<D, MAXT, S, NCH>();
    const int Wres = std::min(di.sms * di.occ, kMaxWarps);
    const int nck = (a.cur_len + kChunk - 1) / kChunk;
    const int maxch = MAXT / kChunk;
    const int ka = (nck + maxch - 1) / maxch;
    if (ka > kMaxPieces / 2) return cudaErrorInvalidValue;   // context beyond 16 score buffers
    // Scheduler (B200 sweeps, DESIGN.md section 3 "Schedule"):
    //  * many heads per warp: tickets over whole heads (the last ones in pieces) balance the
    //    per-SM streaming rates and leave a short tail;
    //  * fewer, with the GPU full: a static stream-K prefix over the first hyb_pct % of the heads
    //    (every warp streams from the start), then tickets over small pieces of the rest, so the
    //    SMs that stream faster take more of the end;
    //  * small problems: static stream-K ranges only.
    int dyn_min_x100 = kDynHeadsPerWarpX100, nb_x100 = 0, kb = 0, hyb_pct = kHybridStaticPct,
        hyb_q = kHybridPieceChunks;
    tune_split(dyn_min_x100, nb_x100, kb, hyb_pct, hyb_q);
    const bool dynamic = int64_t(bh) * 100 >= int64_t(dyn_min_x100) * Wres;
    int W, hs, na = 0, nb = 0;
    if (dynamic) {
        W = Wres;
        hs = 0;
        nb = int(std::min<int64_t>(bh, (int64_t(W) * nb_x100 + 99) / 100));
        if (kb <= 0) kb = 2;
        kb = std::max(ka, std::min({kb, std::max(1, nck / kMinPieceChunks), kMaxPieces}));
        if (kb <= 1) nb = 0;
        na = bh - nb;
    } else {
        // >= kMinPieceChunks chunks per warp and <= 15 warps per head keep a head's pieces
        // within kMaxPieces (head_pieces <= 1 + ceil(W / heads) + ceil(nck / maxch))
        W = std::max(1, std::min({Wres, bh * nck / kMinPieceChunks, bh * 15}));
        hs = bh;
        if (W == Wres && hyb_pct < 100) {
            hs = int(int64_t(bh) * hyb_pct / 100);
            if (hs > 0 && int64_t(hs) * 15 < W) hs = std::min(bh, (W + 14) / 15);
            nb = bh - hs;
            kb = std::max(ka, std::min({(nck + hyb_q - 1) / hyb_q, kMaxPieces}));
        }
    }
    const WsLayout w = ws_layout(bh, D);
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
    P.nck = nck;
    P.hs = hs;
    P.na = na;
    P.ka = ka;
    P.kb = std::max(kb, 1);
    P.items = na * ka + nb * P.kb;
    P.total = hs * nck;
    static const int nctr_env = [] {
        const char* e = getenv("FLEXQ_ATTN_CTRS");
        return e ? atoi(e) : 0;
    }();
    const int grid = dynamic ? std::max(1, std::min(W, P.items)) : W;
    P.nctr = std::max(1, std::min({nctr_env > 0 ? nctr_env : kMaxCtrs, kMaxCtrs, grid}));   // every counter has warps
    P.wq = P.total / W;
    P.wr = P.total % W;
    P.maxch = maxch;
    P.chunks = a.chunks;
    P.cur_len = a.cur_len;
    P.qscale = 1.4426950408889634f / sqrtf(float(D));
    P.k_new = static_cast<const __half*>(a.k_new);
    P.v_new = static_cast<const __half*>(a.v_new);
    P.kc_w = static_cast<uint8_t*>(const_cast<void*>(a.k_cache));
    P.vc_w = static_cast<uint8_t*>(const_cast<void*>(a.v_cache));
    // L2 prefetch depth (r3g, r3u): with about one head per warp the first two K stages (batch 18:
    // 26.6 -> 25.9 us; the whole first head's K: 27.9 us); with many heads per warp the whole
    // first head's K pass, fetched while the previous grid drains (batch 144: 169.8 -> 165.7 us)
    P.pf_chunks = P.items >= kPfWholeHeadsPerWarp * grid ? nck : FLEXQ_ATTN_L2PF * NCH;
    static const bool pdl = [] {
        const char* e = getenv("FLEXQ_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid));   // dynamic: no more warps than items
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem_bytes<D, MAXT, S, NCH>();
    // At most one item per warp: cap the CTAs resident per SM at ceil(items / SMs) by asking for
    // more (unused) shared memory.  With programmatic dependent launch the CTAs land on the SMs in
    // the order the previous grid frees them; uncapped, the early SMs took 16 heads and late ones
    // as few as 4, and the launch lasted as long as the 16-head SMs (B200 trace, batch 18).
    static const bool cap_env = [] {
        const char* e = getenv("FLEXQ_ATTN_CAP");
        return !(e && e[0] == '0');
    }();
    if (cap_env && dynamic && P.items <= grid) {
        const int r = (P.items + di.sms - 1) / di.sms;
        if (r < di.occ) cfg.dynamicSmemBytes = size_t(di.cap_smem[r]);
    }
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, decode_attention_kernel<D, MAXT, S, NCH>, P);
}

// Ring depth (tuning: FLEXQ_ATTN_RING=2|3).  Measured and dropped: 4 stages of 64 tokens (9 warps
// per SM) and 4 stages of 32 tokens (15 warps per SM) -- slower at every BASELINE shape.
template <int D, int MAXT>
cudaError_t launch_ring(const AttnArgs& a, cudaStream_t stream) {
    static const int ring_env = [] {
        const char* e = getenv("FLEXQ_ATTN_RING");
        return e ? atoi(e) : 0;
    }();
    // default: S = 2 (16 warps per SM); S = 3 (11 warps per SM, two stages in flight) when the launch
    // holds 1.2 - 2 heads per S = 2 warp -- the batch-36 shard of OPT-175B: 48 us vs 55 us (B200 sweep)
    int S = 2;
    if (ring_env == 2 || ring_env == 3) {
        S = ring_env;
    } else {
        const int bh = a.batch * a.heads;
        const int w2 = dev_info<D, MAXT, 2, kNch>().sms * dev_info<D, MAXT, 2, kNch>().occ;
        if (int64_t(bh) * 10 >= int64_t(w2) * 12 && int64_t(bh) * 10 <= int64_t(w2) * 20 &&
            (a.cur_len + kChunk - 1) / kChunk >= 4)
            S = 3;
    }
    if (S == 3) return launch<D, MAXT, 3, kNch>(a, stream);
    return launch<D, MAXT, 2, kNch>(a, stream);
}

}  // namespace

size_t attention_workspace_bytes(int batch, int heads, int head_dim, int t_cap) {
    (void)t_cap;
    return ws_layout(batch * heads, head_dim).total;
}

// Score buffer sized to the context: 576 tokens covers every prompt-512 step in one piece
// per head, 1088 the prompt-1024 steps; longer contexts are cut into 1088-token pieces.
cudaError_t launch_decode_attention(const AttnArgs& a, cudaStream_t stream) {
    if (a.head_dim == 128)
        return a.cur_len <= 576 ? launch_ring<128, 576>(a, stream) : launch_ring<128, 1088>(a, stream);
    return a.cur_len <= 576 ? launch_ring<64, 576>(a, stream) : launch_ring<64, 1088>(a, stream);
}

}  // namespace flexq

#if FLEXQ_ATTN_TRACE
// Tuning build only (not in include/flexq.h): copy the last dense-attention launch's
// per-warp stamps [warp][resident, after wait, end, pieces] to host memory.
extern "C" int flexq_debug_attn_trace(void* host_dst, int warps) {
    return int(cudaMemcpyFromSymbol(host_dst, flexq::g_attn_trace, size_t(warps) * 4 * 8));
}
#endif

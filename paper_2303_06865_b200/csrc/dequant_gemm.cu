// dequant_gemm.cu -- decode-step linear layer over a group-wise 4-bit weight.
//
//   y[m][n] = sum_k x[m][k] * w^[k][n]          (t . w)
// with the weight quantized by flexq_quantize -- codes u4 [K][N/2] and half2 {scale, min}
// [K][N/64], groups of 64 "along the output channel dimension" (reading J) -- and
// "converted back to FP16 before computation" inside the kernel:
//   w^[k][n] = min(RN16(c * scale + min), 65504)   (one fp16 FMA; reading G2 in DESIGN.md)
//
// The decode batch (M = 144 at OPT-175B) is small against the weight (K x N = 12288 x
// 49152), so the MMA is "swapped": the tensor core's M dimension runs over 128 weight
// columns n, its N dimension over the batch rows m (<= 160), K over k:
//
//     D[n][m] (TMEM fp32) += A[n][k] (TMEM f16) * B[m][k] (smem f16, K-major, TMA SW128)
//
//   * A never touches shared memory.  flexq_pack_weight re-lays the quantized weight once
//     into 9 KB "panels" (256 columns x 64 k: codes column-major along k + the (scale, min)
//     pairs of those k), one contiguous bulk copy each.  Dequant warps own one TMEM lane
//     (= one weight column n) each: two 16-byte shared loads give the lane's 64 codes, four
//     LOP3/HADD2/HFMA2/HMNMX2 steps per 8 codes give 8 fp16 values already paired along k,
//     and tcgen05.st writes them straight into the A operand columns.  (In the first,
//     shared-memory-A version the dequant stores plus the MMA's A and B reads needed more
//     than the 128 B/clk of shared-memory bandwidth.)
//   * One elected thread issues tcgen05.mma (kind::f16, A from TMEM, M = 128, N = Mpad,
//     K = 16) into two TMEM accumulators -- 256 weight columns per tile, so every x block
//     fetched from L2 feeds two MMAs.
//   * Schedule: data-parallel full tiles plus a split-k remainder (Sched below); a tile
//     split along k writes fp32 partials to the workspace and the last of its contributors
//     (ticket) sums them in contributor order -- deterministic -- and stores fp16.
//
// Warp roles (16 warps): 0 panel bulk copies, 1 MMA issuer, 2 x TMA, 3 TMEM allocator,
// 4-7 epilogue (TMEM lanes 32*(w%4) ..), 8-15 dequant (lanes 32*(w%4) .., A half (w-8)/4).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <stdlib.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kBN = kGemmTileN;        // 256 weight columns per tile (two 128-row A operands)
constexpr int kBK = kGemmTileK;        // 64 k per stage (one 128-byte swizzle row of x)
#ifndef FLEXQ_GEMM_DQW
#define FLEXQ_GEMM_DQW 16
#endif
constexpr int kDequantWarps = FLEXQ_GEMM_DQW;   // 8: each warp converts all 64 k of its column;
                                                // 16: two warps per column, one per 32-k half
constexpr int kThreads = (8 + kDequantWarps) * 32;
#ifndef FLEXQ_GEMM_PANEL_STAGES
#define FLEXQ_GEMM_PANEL_STAGES 8
#endif
#ifndef FLEXQ_GEMM_PROBE
#define FLEXQ_GEMM_PROBE 0   // tuning only: 1 skip the A stores to TMEM, 2 skip the dequant arithmetic
#endif
#ifndef FLEXQ_GEMM_TRACE
#define FLEXQ_GEMM_TRACE 0      // tuning only: clock64 stamps of CTA 0's pipeline into the workspace
#endif
#define TRACE(slot, j) \
    do { if (FLEXQ_GEMM_TRACE && blockIdx.x == 0 && (j) < 256) { \
        long long t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)); \
        reinterpret_cast<long long*>(p.partials)[(slot) * 256 + (j)] = t_; } } while (0)
constexpr int kPanelStages = FLEXQ_GEMM_PANEL_STAGES;
constexpr int kPanelCodes = kBN * kBK / 2;      // 8 KB: [k half (2)][column (256)][16 B = 32 codes]
constexpr int kPanelData = kPanelCodes + 1024;  // + 1 KB: [group (4)][k pair (32)][{scale pair, min pair}]
constexpr int kPanelBytes = kGemmPanelBytes;    // per panel in the buffer and per smem stage: data + 16 B flag
constexpr int kPanelFlag = kPanelData;          // smem stage offset of the flag; in global memory the flags
                                                // follow all panels (panel data stays 1 KB-aligned)
constexpr int kMaxAStages = 6;                 // A operand stages in TMEM (64 columns each)
constexpr int kBStages = 6;                    // x stages in smem
constexpr int kDoneSlots = 6;                  // ring of commit barriers, one per group of stages
constexpr int kEpiWarps = 4;
constexpr uint32_t kTmemCols = 512;
// TMEM columns: accumulator h at h * acc_stride (acc_stride = Mpad rounded up to 32), then
// n_a A stages of 64 columns (half h of stage s at a_col + 64 s + 32 h).
constexpr int kSmemLimit = 232448;              // 227 KB opt-in
constexpr uint32_t kEpiScratch = kEpiWarps * 16 * 32 * 2;   // per warp: 16 rows (m) x 32 columns (n) fp16
static_assert(2 * ((kGemmMaxRows + 31) / 32 * 32) + 3 * 64 <= int(kTmemCols), "2 accumulators + 3 A stages");

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory"); }

// UMMA shared-memory descriptor, 128-byte swizzle (layout type 2), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// Polling wait with a sleep between polls, for roles that wait long (the epilogue waits a whole
// tile): spinning try_wait loops compete with the MMA issuer's own barrier and UTCHMMA issue.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t ns) {
    uint32_t ok = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(ns);
    }
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Issued by a whole, converged warp: elect.sync picks the one lane that issues.  (Issuing from
// a lone lane makes ptxas wrap every tcgen05 op in an ELECT/BRA.U.ANY loop: ~45 cycles per
// MMA against ~16 this way -- the issuing warp's latency chain bounds the MMA rate at small N.)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            addr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(su32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts16(uint32_t a, __half v) {
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(__half_as_ushort(v)) : "memory");
}

// ------------------------------------------------------------------ dequant
// A panel code word holds 8 codes of one column for k0 .. k0+7 with nibble positions
// (0, 4) = (k0, k0+1), (1, 5) = (k0+2, k0+3), (2, 6) = (k0+4, k0+5), (3, 7) = (k0+6, k0+7):
// one shift and one LOP3 put a k pair into the mantissas of fp16 1024 + c (exact), HADD2
// removes the 1024 (exact), HFMA2 applies the pair's (scale, min) with one rounding, and
// HMNMX2 clamps at 65504 (reading R; c * scale + min >= min >= -65504 needs no lower clamp).
// The result is the tcgen05 A column word for that k pair (low half = even k).
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
template <bool CLAMP>
__device__ __forceinline__ uint32_t deq_pair(uint32_t t, uint32_t sp, uint32_t mp) {
    uint32_t m;
    asm("lop3.b32 %0, %1, 0x000F000F, 0x64006400, 0xEA;" : "=r"(m) : "r"(t));   // (t & mask) | magic
    const __half2 c = __hsub2(u2h(m), u2h(0x64006400u));                      // c (exact)
    const __half2 v = __hfma2(c, u2h(sp), u2h(mp));
    if constexpr (CLAMP) return h2u(__hmin2(v, u2h(0x7BFF7BFFu)));           // <= 65504
    else return h2u(v);   // the panel's flag says no code can exceed 65504 (flexq_pack_weight)
}
template <bool CLAMP>
__device__ __forceinline__ void deq_word(uint32_t w, uint4 meta_lo, uint4 meta_hi, uint32_t* o) {
    // meta_lo = {s01, m01, s23, m23}, meta_hi = {s45, m45, s67, m67}
    o[0] = deq_pair<CLAMP>(w, meta_lo.x, meta_lo.y);
    o[1] = deq_pair<CLAMP>(w >> 4, meta_lo.z, meta_lo.w);
    o[2] = deq_pair<CLAMP>(w >> 8, meta_hi.x, meta_hi.y);
    o[3] = deq_pair<CLAMP>(w >> 12, meta_hi.z, meta_hi.w);
}

// Store 16 rows (m0 .. m0+15) x 32 columns (n0 .. n0+31) of y from one warp: lane j holds
// column n0 + j's 16 values; a per-warp smem transpose turns them into 16-byte row pieces.
__device__ __forceinline__ void store_rows16(const float (&v)[16], uint32_t scratch, int lane, __half* y, int64_t ldy,
                                             int m0, int M, int n0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) sts16(scratch + uint32_t(i * 64 + lane * 2), __float2half_rn(v[i]));
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int j = lane + 32 * r, row = j >> 2, piece = j & 3;
        const uint4 d = lds128(scratch + uint32_t(row * 64 + piece * 16));
        if (m0 + row < M) *reinterpret_cast<uint4*>(y + int64_t(m0 + row) * ldy + n0 + piece * 8) = d;
    }
    __syncwarp();
}

// ------------------------------------------------------------------ CTA-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of `p`'s counterpart in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
// wait with cluster-scope acquire (the phase was completed by arrivals from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WC_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void umma_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}" ::"r"(
            su32(bar)),
        "h"((unsigned short)3)
        : "memory");
}

template <bool B>
struct BoolTag {
    static constexpr bool value = B;
};

// Ring position without divisions (the issuing thread's instruction count is on the critical path).
struct Ring {
    int slot = 0, n;
    uint32_t phase = 0;
    __device__ explicit Ring(int n_) : n(n_) {}
    __device__ __forceinline__ void next() {
        if (++slot == n) { slot = 0; phase ^= 1u; }
    }
};
// Tracks which commit barrier covers a stage: stage groups of G consecutive stages, one
// done[] slot per group, 6 slots.
struct GroupRing {
    int pos = 0, G;
    Ring q{kDoneSlots};
    __device__ explicit GroupRing(int g) : G(g) {}
    __device__ __forceinline__ bool last_in_group() const { return pos == G - 1; }
    __device__ __forceinline__ void next() {
        if (++pos == G) { pos = 0; q.next(); }
    }
};

// ------------------------------------------------------------------ work schedule
// Data-parallel waves plus a split-k remainder.  CTA c owns the full tiles c, c + G, ...
// (dp_waves of them).  The T mod G remainder tiles are cut along k into S parts of L
// k-blocks; CTA c < R*S takes part c / R of remainder tile c % R -- FIRST, so that the
// fixup by the last of the S contributors overlaps that CTA's data-parallel tiles.
struct Sched {
    int KB;          // k-blocks per tile
    int G;           // CTAs
    int dp_waves;    // full tiles per CTA
    int R, S, L;     // remainder tiles, parts per remainder tile, k-blocks per part
    __device__ __forceinline__ bool has_rem(int c) const { return c < R * S; }
    __device__ __forceinline__ int units(int c) const { return dp_waves + (has_rem(c) ? 1 : 0); }
    // unit u of CTA c -> tile, first k-block, k-block count, remainder part (-1: full tile)
    __device__ __forceinline__ void unit(int c, int u, int& tile, int& kb0, int& nk, int& part) const {
        if (has_rem(c) && u == 0) {
            part = c / R;
            tile = dp_waves * G + c % R;
            kb0 = part * L;
            nk = KB - kb0 < L ? KB - kb0 : L;
        } else {
            part = -1;
            tile = (u - (has_rem(c) ? 1 : 0)) * G + c;
            kb0 = 0;
            nk = KB;
        }
    }
};

struct GemmParams {
    const uint8_t* panels;   // [tiles][KB][9216 B] panel data, then [tiles][KB][16 B] flags
    int64_t n_panels;
    __half* y;               // [M][N]
    float* partials;         // [grid][256 (n)][mpad (m)]
    uint32_t* tickets;       // [remainder tiles]
    int M, N, mpad;
    // Pipeline shape (host-chosen from Mpad): n_a A stages in TMEM, one tcgen05.commit per group
    // of `group` stages (a commit costs the issuing thread ~250 cycles of tensor-pipe time, so
    // small batches, whose accumulators leave room for 6 A stages, commit every 3 stages).
    int n_a, group;
    uint32_t acc_stride, a_col;
    Sched sc;
};

struct Smem {
    uint32_t panel, b, epi, bars, b_stages, total;
};
__host__ __device__ inline Smem smem_plan(int mpad, bool pair) {
    Smem s;
    const uint32_t bstage = uint32_t(pair ? mpad / 2 : mpad) * 128u;   // x rows held by this CTA
    s.panel = 0;
    s.b = (s.panel + kPanelStages * kPanelBytes + 1023u) / 1024u * 1024u;   // x stages: 1024-aligned (SW128)
    const uint32_t bs = kBStages;   // fixed-size plan: 8 * 9 KB + 6 * Mpad * 128 B + 4 KB + bars <= 227 KB
    s.b_stages = bs;
    s.epi = s.b + bs * bstage;
    s.bars = s.epi + kEpiScratch;
    s.total = s.bars + 1024u + 1024u;
    return s;
}

// PAIR: a cluster of two CTAs on one TPC runs cta_group::2 MMAs with M = 256 (each CTA holds the A
// operand of its own 256 weight columns in its TMEM, and half of the x rows in its shared memory);
// the leader (rank 0) issues for both.  Per CTA that halves the MMA instructions, the commits and
// the tensor core's shared-memory reads of x, which together bounded the single-CTA version.
template <bool PAIR>
__global__ void __launch_bounds__(kThreads, 1)
dequant_gemm_kernel(const __grid_constant__ CUtensorMap map_x, const GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
    const Smem L = smem_plan(p.mpad, PAIR);
    const uint32_t s_panel = su32(smem + L.panel);
    const uint32_t s_b = su32(smem + L.b);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* panel_full = bars;
    uint64_t* panel_empty = panel_full + kPanelStages;
    uint64_t* a_full = panel_empty + kPanelStages;
    uint64_t* b_full = a_full + kMaxAStages;
    // done[q % 6] completes when the MMAs of stage group q (stages q*G .. q*G+G-1) have finished
    // reading A (TMEM) and B (smem): one commit frees both rings for the whole group.
    uint64_t* done = b_full + kBStages;
    uint64_t* tmem_full = done + kDoneSlots;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bstage = uint32_t(PAIR ? p.mpad / 2 : p.mpad) * 128u;   // this CTA's x rows per stage
    const int NA = p.n_a, GR = p.group;
    const uint32_t rank = PAIR ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    (void)leader;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kPanelStages; ++i) {
            mbar_init(panel_full + i, 1);
            mbar_init(panel_empty + i, kDequantWarps);
        }
        // in a pair, the peer's dequant warps arrive on the leader's a_full as well (relaxed cluster-scope
        // arrives after tcgen05.wait::st: a release.cluster arrive per warp costs ~1000 cycles)
        for (int i = 0; i < kMaxAStages; ++i)
            mbar_init(a_full + i, PAIR && leader ? 2 * kDequantWarps : kDequantWarps);
        for (int i = 0; i < kBStages; ++i) mbar_init(b_full + i, 1);
        for (int i = 0; i < kDoneSlots; ++i) mbar_init(done + i, 1);
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, (PAIR ? 2 : 1) * kEpiWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 3) {
        if constexpr (PAIR) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                         "n"(kTmemCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                         "n"(kTmemCols)
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
    }
    if (warp == 2 && lane == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();      // the peer's barriers exist before anyone arrives remotely
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // barriers the leader waits on, as seen from this CTA (local in the leader, remote in the peer)
    const uint32_t a_full_l = PAIR ? peer_addr(a_full, 0) : su32(a_full);
    const uint32_t b_full_l = PAIR ? peer_addr(b_full, 0) : su32(b_full);
    const uint32_t tmem_empty_l = PAIR ? peer_addr(tmem_empty, 0) : su32(tmem_empty);

    const Sched& S = p.sc;
    const int c = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);   // schedule index: the pair, or the CTA
    const int nunits = S.units(c);
    const int KB = S.KB;

    if (warp == 0) {
        // ---------------- weight panels: one contiguous 9 KB bulk copy per (tile, k-block), evict-first
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            for (int u = 0; u < nunits; ++u) {
                int tile, kb0, nk, part;
                S.unit(c, u, tile, kb0, nk, part);
                const int t256 = PAIR ? 2 * tile + int(rank) : tile;   // this CTA's 256-column tile
                const int64_t pi0 = int64_t(t256) * KB + kb0;
                const uint8_t* src = p.panels + pi0 * kPanelData;
                const uint8_t* fsrc = p.panels + p.n_panels * kPanelData + pi0 * 16;
                for (int j = 0; j < nk; ++j, src += kPanelData, fsrc += 16) {
                    mbar_wait(panel_empty + s, ph ^ 1);
                    mbar_expect_tx(panel_full + s, kPanelBytes);
                    bulk_g2s(s_panel + uint32_t(s * kPanelBytes), src, kPanelData, panel_full + s, pol);
                    bulk_g2s(s_panel + uint32_t(s * kPanelBytes + kPanelFlag), fsrc, 16, panel_full + s, pol);
                    if (++s == kPanelStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 2) {
        // ---------------- x producer (L2-resident, evict-last)
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            int g = 0;     // global stage index
            Ring rb(kBStages);
            GroupRing prev(GR);   // commit group of stage g - 6
            for (int u = 0; u < nunits; ++u) {
                int tile, kb0, nk, part;
                S.unit(c, u, tile, kb0, nk, part);
                for (int kb = kb0; kb < kb0 + nk; ++kb, ++g) {
                    const int s = rb.slot;
                    if (g >= kBStages) {      // the slot's previous stage (g - 6) has been consumed
                        mbar_wait(done + prev.q.slot, prev.q.phase);
                        prev.next();
                    }
                    rb.next();
                    if constexpr (PAIR) {
                        // both halves complete on the leader's barrier; the leader expects both
                        if (leader) mbar_expect_tx(b_full + s, 2u * bstage);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
                            ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(s_b + uint32_t(s) * bstage),
                            "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(kb * kBK), "r"(int(rank) * p.mpad / 2),
                            "r"(b_full_l + uint32_t(s) * 8u), "l"(pol)
                            : "memory");
                    } else {
                        mbar_expect_tx(b_full + s, bstage);
                        asm volatile(
                            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                            " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(s_b + uint32_t(s) * bstage),
                            "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(kb * kBK), "r"(0), "r"(su32(b_full + s)),
                            "l"(pol)
                            : "memory");
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (the whole warp runs the loop; elect.sync issues); in a pair,
        // only the leader's warp issues, for both CTAs
        if (!PAIR || leader) {
            const uint32_t idesc = (1u << 4)                        // D fp32; A, B fp16, both K-major
                                   | (uint32_t(p.mpad >> 3) << 17)  // N
                                   | (uint32_t((PAIR ? 256 : 128) >> 4) << 24);    // M
            // Lean issue loop (the single issuing thread's own instruction count bounds the MMA
            // rate at small N): descriptors are a precomputed base plus an add on the start-address
            // field (addr >> 4 < 2^14, so the add never carries into the next field).
            const uint64_t bdesc0 = smem_desc(s_b, 16, 1024);
            const uint32_t bstage16 = bstage >> 4;
            auto mma_ = [](uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
                if constexpr (PAIR) umma_ts_pair(d, a, b, id, acc); else umma_ts(d, a, b, id, acc);
            };
            auto wait_a_ = [](uint64_t* bar, uint32_t par) {
                if constexpr (PAIR) mbar_wait_cluster(bar, par); else mbar_wait(bar, par);
            };
            auto commit_ = [](uint64_t* bar) {
                if constexpr (PAIR) umma_commit_pair(bar); else umma_commit_warp(bar);
            };
            Ring ra(NA), rb(kBStages);
            GroupRing grp(GR);
            int gt = 0;   // stage counter (trace only)
            for (int seg = 0; seg < nunits; ++seg) {
                int tile, kb0, nk, part;
                S.unit(c, seg, tile, kb0, nk, part);
                wait_a_(tmem_empty, (uint32_t(seg) & 1u) ^ 1u);
                wait_a_(a_full + ra.slot, ra.phase);
                mbar_wait(b_full + rb.slot, rb.phase);
                tc_fence_after();
                for (int j = 0; j < nk; ++j) {
                    if (lane == 0) TRACE(0, gt);
                    const uint64_t bd0 = bdesc0 + uint64_t(uint32_t(rb.slot) * bstage16);
                    const uint32_t a0 = tmem_base + p.a_col + uint32_t(ra.slot) * 64u;
                    ra.next();
                    rb.next();
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t bd = bd0 + uint64_t(kk * 2);
                        const uint32_t accf = (j > 0 || kk > 0) ? 1u : 0u;
                        mma_(tmem_base, a0 + kk * 8, bd, idesc, accf);
                        mma_(tmem_base + p.acc_stride, a0 + 32 + kk * 8, bd, idesc, accf);
                        if (kk == 0) {
                            if (j + 1 < nk) {
                                // stage g + 1's barriers, waited while stage g's MMAs are still queued
                                if (lane == 0) TRACE(1, gt);
                                wait_a_(a_full + ra.slot, ra.phase);
                                mbar_wait(b_full + rb.slot, rb.phase);
                                tc_fence_after();
                                if (lane == 0) TRACE(2, gt);
                            }
                        }
                    }
                    if (grp.last_in_group()) commit_(done + grp.q.slot);
                    if (lane == 0) TRACE(3, gt);
                    ++gt;
                    grp.next();
                }
                commit_(tmem_full);
            }
            if (grp.pos != 0) commit_(done + grp.q.slot);   // a final partial group
        }
    } else if (warp >= 8) {
        // ---------------- dequant warps: panel (smem) -> fp16 A operand (TMEM lane = weight column)
        const int d = warp - 8;
        const int q = warp & 3, h = (d >> 2) & 1;
        constexpr int kHalves = kDequantWarps == 16 ? 1 : 2;   // 32-k halves converted by this warp
        const int hk0 = kDequantWarps == 16 ? (d >> 3) : 0;
        const int nl = h * 128 + q * 32 + lane;             // column within the 256-column tile
        const uint32_t codes_off = uint32_t(nl) * 16u;
        const uint32_t meta_off = uint32_t(kPanelCodes) + uint32_t(nl >> 6) * 256u;
        const uint32_t a_lane = tmem_base + (uint32_t(q * 32) << 16) + p.a_col + uint32_t(h) * 32u;
        int total = 0;
        for (int u = 0; u < nunits; ++u) {
            int tile, kb0, nk, part;
            S.unit(c, u, tile, kb0, nk, part);
            total += nk;
        }
        int ps = 0;
        uint32_t pph = 0;
        Ring ra(NA);
        GroupRing prev(GR);   // commit group of stage it - NA
        for (int it = 0; it < total; ++it) {
            const int as = ra.slot;
            ra.next();
            if (warp == 8 && lane == 0) TRACE(4, it);
            mbar_wait(panel_full + ps, pph);
            if (warp == 8 && lane == 0) TRACE(5, it);
            if (it >= NA) {     // the A slot's previous stage (it - NA) is done
                mbar_wait(done + prev.q.slot, prev.q.phase);
                prev.next();
            }
            const uint32_t pb = s_panel + uint32_t(ps * kPanelBytes);
            const uint32_t clampf = lds32(pb + uint32_t(kPanelFlag));   // warp-uniform
            uint4 cw[kHalves];
#pragma unroll
            for (int i = 0; i < kHalves; ++i) cw[i] = lds128(pb + uint32_t(hk0 + i) * 4096u + codes_off);
            if (warp == 8 && lane == 0) TRACE(6, it);
            tc_fence_after();
            // the panel's clamp flag selects one of two fully unrolled copies of the conversion
            auto convert = [&](auto clamp_tag) {
                constexpr bool kClamp = decltype(clamp_tag)::value;
#pragma unroll
                for (int i = 0; i < kHalves; ++i) {
                    const int hk = hk0 + i;
                    const uint32_t words[4] = {cw[i].x, cw[i].y, cw[i].z, cw[i].w};
                    uint32_t o[16];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t mo = pb + meta_off + uint32_t((16 * hk + 4 * j) * 8);
#if FLEXQ_GEMM_PROBE == 2     // tuning only (wrong results): no dequant arithmetic, no meta loads
                        o[4 * j] = words[j]; o[4 * j + 1] = words[j] >> 8; o[4 * j + 2] = words[j] >> 16;
                        o[4 * j + 3] = mo;
#else
                        deq_word<kClamp>(words[j], lds128(mo), lds128(mo + 16), o + 4 * j);
#endif
                    }
#if FLEXQ_GEMM_PROBE == 1     // tuning only (wrong results): no TMEM writes
                    if (o[0] == 0x12345678u && o[15] == 0x9abcdef0u)
#endif
                    tmem_st16(a_lane + uint32_t(as) * 64u + uint32_t(hk) * 16u, o);
                }
            };
            if (clampf) convert(BoolTag<true>{});
            else convert(BoolTag<false>{});
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(panel_empty + ps);
                if constexpr (PAIR) mbar_arrive_cluster_relaxed(a_full_l + uint32_t(as) * 8u);   // leader's
                else mbar_arrive(a_full + as);
            }
            if (warp == 8 && lane == 0) TRACE(7, it);
            if (++ps == kPanelStages) { ps = 0; pph ^= 1; }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: TMEM -> fp16 y (or fp32 partials + split-k fixup)
        const int q = warp & 3;                 // TMEM lanes 32q .. 32q+31
        const int nl = q * 32 + lane;           // column within a 128-column half
        const uint32_t scratch = su32(smem + L.epi) + uint32_t(q * 1024);
        const int mp = p.mpad;
        for (int seg = 0; seg < nunits; ++seg) {
            int tile, kb0, nk, part;
            S.unit(c, seg, tile, kb0, nk, part);
            const bool full = part < 0;
            mbar_wait_sleep(tmem_full, uint32_t(seg) & 1u, 2000);
            tc_fence_after();
            const int t256 = PAIR ? 2 * tile + int(rank) : tile;     // this CTA's 256-column tile
            float* slot = p.partials + int64_t(blockIdx.x) * mp * kBN;    // [256 n][mpad m]
            for (int h = 0; h < 2; ++h) {
                const int n0 = t256 * kBN + h * 128 + q * 32;
                for (int m0 = 0; m0 < mp; m0 += 16) {
                    float v[16];
                    tmem_ld16(tmem_base + (uint32_t(q * 32) << 16) + uint32_t(h) * p.acc_stride + uint32_t(m0), v);
                    if (full) {
                        store_rows16(v, scratch, lane, p.y, p.N, m0, p.M, n0);
                    } else {
                        float4* dst = reinterpret_cast<float4*>(slot + int64_t(h * 128 + nl) * mp + m0);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            __stcg(dst + i, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR) mbar_arrive_cluster(tmem_empty_l);   // the leader's MMA waits on both CTAs
                else mbar_arrive(tmem_empty);
            }
            if (!full) {
                // Split-k fixup, spread over the tile's S contributors (CTAs r + R p, all resident:
                // the grid is at most one CTA per SM): each announces its partial on the tile's
                // arrival ticket, waits for all S, then sums a 1/S slice of the rows over the S
                // partials in p order (deterministic) and stores fp16; the last to finish its
                // slice resets both tickets.  (A single last contributor summing every row was
                // latency-bound: ~30 us of the 12288 x 12288 launch.)
                const int r = c % S.R;                                  // remainder tile (pair tile)
                const int tk = PAIR ? 2 * r + int(rank) : r;             // ticket of this CTA's half
                const int ntk = p.N / kBN;                              // done tickets follow
                const int my_part = c / S.R;
                __threadfence();
                epi_bar();
                if (q == 0 && lane == 0) {
                    atomicAdd(p.tickets + tk, 1u);
                    uint32_t seen = 0;
                    while (true) {
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(p.tickets + tk) : "memory");
                        if (seen >= uint32_t(S.S)) break;
                        __nanosleep(256);
                    }
                }
                epi_bar();
                __threadfence();
                const int nmb = mp / 16;
                const int mb0 = my_part * nmb / S.S, mb1 = (my_part + 1) * nmb / S.S;
                for (int h = 0; h < 2; ++h) {
                    const int n0 = t256 * kBN + h * 128 + q * 32;
                    const int64_t col = int64_t(h * 128 + nl) * mp;
                    for (int mb = mb0; mb < mb1; ++mb) {
                        const int m0 = mb * 16;
                        float v[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[i] = 0.f;
                        for (int pp = 0; pp < S.S; pp += 2) {
                            // two contributors per round: 8 independent 16-byte loads in flight
                            float4 a[8];
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const int kp = r + S.R * (pp + u < S.S ? pp + u : pp);   // contributor
                                const int k = PAIR ? 2 * kp + int(rank) : kp;            // its slot
                                const float4* src =
                                    reinterpret_cast<const float4*>(p.partials + int64_t(k) * mp * kBN + col + m0);
#pragma unroll
                                for (int i = 0; i < 4; ++i) a[4 * u + i] = __ldcg(src + i);
                            }
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                if (pp + u >= S.S) break;
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    v[4 * i] += a[4 * u + i].x;
                                    v[4 * i + 1] += a[4 * u + i].y;
                                    v[4 * i + 2] += a[4 * u + i].z;
                                    v[4 * i + 3] += a[4 * u + i].w;
                                }
                            }
                        }
                        store_rows16(v, scratch, lane, p.y, p.N, m0, p.M, n0);
                    }
                }
                epi_bar();
                if (q == 0 && lane == 0) {
                    __threadfence();
                    if (atomicAdd(p.tickets + ntk + tk, 1u) == uint32_t(S.S - 1)) {
                        p.tickets[tk] = 0u;
                        p.tickets[ntk + tk] = 0u;
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) cluster_sync();      // neither CTA frees TMEM the pair's MMAs may still use
    tc_fence_after();
    if (warp == 3) {
        if constexpr (PAIR)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                         : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(kTmemCols)
                         : "memory");
    }
}

// ------------------------------------------------------------------ weight panels
// Pure re-layout of flexq_quantize's output (no arithmetic): panel (t, kb) holds columns
// [256 t, 256 t + 256) and k [64 kb, 64 kb + 64):
//   codes [hk (2)][column (256)][4 words]; word j of (hk, column) holds the codes of
//     k = 32 hk + 8 j + {0..7} at nibble positions {0, 4, 1, 5, 2, 6, 3, 7}
//   meta  [group (4)][k pair (32)][scale pair (half2), min pair (half2)].
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, uint8_t* __restrict__ panels, int64_t K,
                                  int64_t N) {
    const int64_t KB = K / kBK;
    const int64_t total = (N / kBN) * KB * 2 * kBN;      // one thread per (panel, hk, column)
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int col = int(i % kBN);
        const int hk = int((i / kBN) % 2);
        const int64_t panel = i / (2 * kBN);
        const int64_t tile = panel / KB, kb = panel % KB;
        const int64_t n = tile * kBN + col;
        uint32_t w[4] = {0, 0, 0, 0};
        for (int kl = 0; kl < 32; ++kl) {
            const int64_t k = kb * kBK + hk * 32 + kl;
            const uint32_t byte = codes[k * (N / 2) + n / 2];
            const uint32_t c = (n & 1) ? (byte >> 4) : (byte & 15u);
            const int j = kl >> 3, e = kl & 7;
            const int pos = (e & 1) ? 4 + (e >> 1) : (e >> 1);
            w[j] |= c << (4 * pos);
        }
        uint4* dst = reinterpret_cast<uint4*>(panels + panel * kPanelData + hk * 4096 + col * 16);
        *dst = make_uint4(w[0], w[1], w[2], w[3]);
        if (hk == 0 && col == 0)   // the panel's flag; pack_meta_kernel (next in the stream) ORs into it
            *reinterpret_cast<uint4*>(panels + (N / kBN) * KB * kPanelData + panel * 16) = make_uint4(0, 0, 0, 0);
    }
}

__global__ void pack_meta_kernel(const __half2* __restrict__ meta, uint8_t* __restrict__ panels, int64_t K,
                                 int64_t N) {
    const int64_t KB = K / kBK;
    const int64_t G = N / kGroup;
    const int64_t total = (N / kBN) * KB * 4 * 32;       // one thread per (panel, group, k pair)
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
        const int kp = int(i % 32);
        const int g = int((i / 32) % 4);
        const int64_t panel = i / 128;
        const int64_t tile = panel / KB, kb = panel % KB;
        const int64_t gg = tile * 4 + g;
        const int64_t k = kb * kBK + 2 * kp;
        const __half2 a = meta[k * G + gg], b = meta[(k + 1) * G + gg];
        const __half2 sp = __halves2half2(__low2half(a), __low2half(b));    // scales of k, k+1
        const __half2 mp = __halves2half2(__high2half(a), __high2half(b));  // mins of k, k+1
        uint2* dst = reinterpret_cast<uint2*>(panels + panel * kPanelData + kPanelCodes + (g * 32 + kp) * 8);
        *dst = make_uint2(h2u(sp), h2u(mp));
        // clamp flag: some code of this panel may reconstruct above 65504 (c = 15 is the largest
        // value, 15 * scale + min, exact in double), so its fp16 FMA needs the clamp of reading R
        const double top0 = 15.0 * double(__low2float(a)) + double(__high2float(a));
        const double top1 = 15.0 * double(__low2float(b)) + double(__high2float(b));
        if (top0 > 65504.0 || top1 > 65504.0)
            atomicOr(reinterpret_cast<unsigned int*>(panels + (N / kBN) * KB * kPanelData + panel * 16), 1u);
    }
}

// ------------------------------------------------------------------ host side
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiled>(f);
    });
    return fn;
}

}  // namespace

bool make_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
              uint64_t stride1_bytes, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw,
              CUtensorMapL2promotion promo) {
    EncodeTiled enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[2] = {d0, d1};
    const cuuint64_t strides[1] = {stride1_bytes};
    const cuuint32_t box[2] = {b0, b1};
    const cuuint32_t estr[2] = {1, 1};
    return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
               promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

int sm_count() { return device_sm_count(); }

inline int mpad_of(int64_t m) {
    const int64_t r = m < kGemmMaxRows ? m : kGemmMaxRows;
    return int((r + 15) / 16 * 16);
}

}  // namespace

size_t gemm_panel_bytes(int64_t k, int64_t n) { return size_t(n / kBN) * size_t(k / kBK) * kPanelBytes; }

cudaError_t launch_pack_weight(const void* codes, const void* meta, int64_t K, int64_t N, void* panels,
                               cudaStream_t stream) {
    const int blocks = sm_count() * 8;
    pack_codes_kernel<<<blocks, 256, 0, stream>>>(static_cast<const uint8_t*>(codes), static_cast<uint8_t*>(panels),
                                                  K, N);
    pack_meta_kernel<<<blocks, 256, 0, stream>>>(static_cast<const __half2*>(meta), static_cast<uint8_t*>(panels), K,
                                                 N);
    return cudaGetLastError();
}

// Host-only arithmetic (no CUDA call): one partial slot per CTA for at most kGemmMaxGrid CTAs.
size_t dequant_gemm_workspace_bytes(int64_t m, int64_t k, int64_t n) {
    (void)k;
    const int64_t tiles = n / kBN;
    const size_t tickets = size_t((tiles * 8 + 255) / 256 * 256);   // arrival + done ticket per tile
    const size_t tc = tickets + size_t(kGemmMaxGrid) * size_t(mpad_of(m)) * kBN * sizeof(float);
    const size_t gv = m <= kGemvMaxRows ? dequant_gemv_workspace_bytes(n) : 0;
    return tc > gv ? tc : gv;
}

namespace {
// Small-batch path switch (tuning / A-B only): FLEXQ_GEMM_SMALLM=0 sends every batch to the tcgen05 kernel.
bool small_m_path() {
    static const bool on = [] {
        const char* e = getenv("FLEXQ_GEMM_SMALLM");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

cudaError_t launch_dequant_gemm(const void* x, const void* panels, int64_t M, int64_t K, int64_t N, void* y,
                                void* workspace, cudaStream_t stream) {
    if (M <= kGemvMaxRows && small_m_path()) return launch_dequant_gemv(x, panels, M, K, N, y, workspace, stream);
    const int kb = int(K / kBK);
    const int G = sm_count() < kGemmMaxGrid ? sm_count() : kGemmMaxGrid;
    // CTA pairs (cta_group::2, 512-column pair tiles) are opt-in (FLEXQ_GEMM_PAIR=1): measured within 3 %
    // of the single-CTA kernel (165 vs 170 us at 144 x 12288 x 49152), whose bound is the dequant
    // warps' ALU work and the per-stage issue chain rather than the MMA count.
    static const bool pair_ok = [] {
        const char* e = getenv("FLEXQ_GEMM_PAIR");
        return e && e[0] == '1';
    }();
    const bool pair = pair_ok && N % (2 * kBN) == 0 && G >= 2;
    const int64_t tiles = N / (pair ? 2 * kBN : kBN);   // schedule units: pair tiles or CTA tiles
    const int Gs = pair ? G / 2 : G;
    Sched sc;
    sc.KB = kb;
    sc.dp_waves = int(tiles / Gs);
    sc.R = int(tiles % Gs);
    sc.S = 1;
    sc.L = kb;
    if (sc.R > 0) {
        int parts = Gs / sc.R;
        if (parts > kb) parts = kb;
        if (parts < 1) parts = 1;
        sc.L = (kb + parts - 1) / parts;
        sc.S = (kb + sc.L - 1) / sc.L;
    }
    sc.G = Gs;
    const int units = sc.dp_waves > 0 ? Gs : sc.R * sc.S;
    const int grid = pair ? 2 * units : units;
    const size_t tick_bytes = size_t((N / kBN * 8 + 255) / 256 * 256);
    uint32_t* tickets = static_cast<uint32_t*>(workspace);
    float* partials = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + tick_bytes);
    {   // the shared-memory attribute, once per device (under a lock)
        static cudaError_t attr_err[kMaxDevices];
        static std::once_flag attr_once[kMaxDevices];
        const int dev = current_device();
        std::call_once(attr_once[dev], [dev] {
            cudaError_t e = cudaFuncSetAttribute(dequant_gemm_kernel<false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(dequant_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemLimit);
            attr_err[dev] = e;
        });
        if (attr_err[dev] != cudaSuccess) return attr_err[dev];
    }
    for (int64_t m0 = 0; m0 < M; m0 += kGemmMaxRows) {
        const int mrows = int(M - m0 < kGemmMaxRows ? M - m0 : kGemmMaxRows);
        const int mpad = (mrows + 15) / 16 * 16;
        CUtensorMap mx;
        if (!make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, static_cast<const __half*>(x) + m0 * K, uint64_t(K),
                      uint64_t(mrows), uint64_t(K * 2), kBK, uint32_t(pair ? mpad / 2 : mpad),
                      CU_TENSOR_MAP_SWIZZLE_128B))
            return cudaErrorInvalidValue;
        GemmParams p;
        p.panels = static_cast<const uint8_t*>(panels);
        p.n_panels = int64_t(N / kBN) * kb;
        p.y = static_cast<__half*>(y) + m0 * N;
        p.partials = partials;
        p.tickets = tickets;
        p.M = mrows;
        p.N = int(N);
        p.mpad = mpad;
        p.acc_stride = uint32_t((mpad + 31) / 32 * 32);
        p.a_col = 2u * p.acc_stride;
        const int fit = int((kTmemCols - p.a_col) / 64u);
        p.n_a = fit >= 6 ? 6 : (fit >= 4 ? 4 : 3);
        p.group = p.n_a == 6 ? 3 : (p.n_a == 4 ? 2 : 1);
        p.sc = sc;
        const Smem L = smem_plan(mpad, pair);
        cudaError_t e;
        if (pair) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(unsigned(grid));
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = L.total;
            cfg.stream = stream;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            e = cudaLaunchKernelEx(&cfg, dequant_gemm_kernel<true>, mx, p);
        } else {
            dequant_gemm_kernel<false><<<grid, kThreads, L.total, stream>>>(mx, p);
            e = cudaGetLastError();
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace flexq

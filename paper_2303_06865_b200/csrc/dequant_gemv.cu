// dequant_gemv.cu -- the decode linear layer at small batch (M <= 16 rows), SURVEY NEXT-2.
//
//   y[m][n] = sum_k x[m][k] * w^[k][n],   w^[k][n] = min(RN16(c * scale + min), 65504)
// (readings J, G1, G2 in DESIGN.md) over the same 9 KB weight panels
// as dequant_gemm.cu (flexq_pack_weight's output), with the same fp16 dequantized values.
//
// Why a second kernel: at M <= 16 the product is a GEMV -- 2 M flops per 0.56 weight bytes --
// so the bound is the HBM stream of the compressed weight, not the tensor pipe.  The tcgen05
// kernel runs one 9 KB panel per ~850-cycle pipeline step (MMA issue + commit + three rings),
// ~114 us at M = 1 for 340 MB.  Here a panel is one stage of a deep per-SM ring and its math is a
// handful of legacy mma.sync per warp:
//   * Persistent CTAs, one per SM; CTA c streams the contiguous panel range
//     [c T / G, (c + 1) T / G) of the T = tiles x KB panels in (tile, k-block) order
//     (stream-K), so every SM moves the same number of bytes.
//   * Four producer warps take every fourth stage of a 16-stage ring; per stage one lane issues
//     two copies: the 9216-byte panel and the M x 64 tile of x (2-D TMA).  (One producer lane
//     issuing per-row copies of x was the bound of the first version: ~90 cycles per copy, 141 us
//     at M = 1 and 313 us at M = 16.)  The panels' clamp flags (flexq_pack_weight) are OR-ed over
//     the CTA's range once, at the start: the CTA runs the clamp-free conversion unless one of its
//     panels can reconstruct above 65504 (a per-stage flag test stalled on its shared load).
//   * Eight consumer warps each own 32 weight columns of the 256-column tile (two MMA row
//     blocks of 16).  Per stage a lane loads two code words per column (k 8t..8t+7 and
//     32+8t..32+8t+7), dequantizes them into fp16 pairs (LOP3 + HADD2 + HFMA2 [+ HMNMX2] per pair,
//     exactly dequant_gemm.cu's deq_pair), and runs 4 mma.sync.m16n8k16 (f16 x f16 -> f32) per
//     row block and 8 rows of x: A = 16 columns x 16 k, B = x.  The k order inside an MMA is a
//     permutation applied to x identically (below).  The bound of this loop is the shared-memory
//     pipe, not the ALUs: every warp re-reads its group's (scale, min) pairs and the x tile, and a
//     128-bit load costs 4 wavefronts however many lanes share an address -- 16 warps of 16
//     columns needed 576 wavefronts per panel (ncu), 8 warps of 32 columns and x loads only for
//     the rows that exist (M = 1: one of eight) need ~200.
//   * A tile split between CTAs writes fp32 partials; the last of its contributors (ticket)
//     sums them in CTA order -- deterministic -- and stores fp16.
#include <cuda_fp16.h>
#include <stdint.h>

#include <mutex>

#include "flexq_internal.h"

namespace flexq {
namespace {

#ifndef FLEXQ_GEMV_PROBE
#define FLEXQ_GEMV_PROBE 0   // tuning only (wrong results): 1 no x copy, 3 no math, 4 = 1 + 3
#endif
constexpr int kConsumers = 8;                         // consumer warps (32 columns each)
#ifndef FLEXQ_GEMV_CTAS
#define FLEXQ_GEMV_CTAS 2    // CTAs per SM, each with half the ring and two producers: 16 consumer
                             // warps per SM (M <= 8: 70.8 us vs 74.6 us with one CTA of 8)
#endif
constexpr int kCtasV = FLEXQ_GEMV_CTAS;
constexpr int kProducers = kCtasV == 1 ? 4 : 2;       // producer warps (every kProducers-th stage each)
constexpr int kThreadsV = (kConsumers + kProducers) * 32;
constexpr int kStagesV = 16 / kCtasV;                 // a power of two: ring slot / phase by masks
constexpr int kPanelData = kGemmTileN * kGemmTileK / 2 + 1024;   // 9216: codes + meta
constexpr int kXOff = kPanelData;                     // the x tile [M][64] fp16 (128-B aligned for the 2-D TMA)
constexpr int kStageBytes = kXOff + kGemvMaxRows * 128;           // 11264
static_assert(kXOff % 128 == 0 && kStageBytes % 128 == 0, "tensor-copy destination alignment");
constexpr int kSmemV = kStagesV * kStageBytes + 2 * kStagesV * 8 + 16;

struct GemvParams {
    const uint8_t* panels;   // [tiles][KB][9216 B], then [tiles][KB][16 B] flags
    __half* y;               // [M][N]
    float* partials;         // [grid][2][256 n][16 m]
    uint32_t* tickets;       // [tiles]
    int M, N, KB;
    int64_t total;           // panels
    int G;                   // CTAs
};

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
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
// Blocking wait.  The producer lanes wait on "empty" most of the time (the consumers bound the
// loop); a plain try_wait loop returned almost at once and re-polled, ~1/3 of all issued
// instructions of the SM (ncu: 637 spin instructions per 9 KB panel).
// try_wait with an explicit suspend-time hint: the thread is suspended until the phase completes
// (or ~1 ms passes) instead of polling -- test_wait + nanosleep still polled every ~6 ns.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WS_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WS_%=;\n}" ::"r"(su32(b)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            dst),
        "l"(src), "r"(bytes), "r"(su32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_fractional(bool last) {
    uint64_t p;
    if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// dequant_gemm.cu's conversion, operation for operation (reading G2): nibbles 0 and 4 of t ->
// fp16 1024 + c (exact), - 1024 (exact), one fp16 FMA with the pair's (scale, min), clamp.
template <bool CLAMP>
__device__ __forceinline__ uint32_t deq_pair(uint32_t t, uint32_t sp, uint32_t mp, uint32_t magic) {
    uint32_t m;
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0xEA;" : "=r"(m) : "r"(t), "r"(magic));   // (t & mask) | magic
    const __half2 c = __hsub2(u2h(m), u2h(0x64006400u));
    const __half2 v = __hfma2(c, u2h(sp), u2h(mp));
    if constexpr (CLAMP) return h2u(__hmin2(v, u2h(0x7BFF7BFFu)));
    else return h2u(v);
}
// The same value from nibbles 1 and 5 of t without shifting t first: (t & 0x00F000F0) | magic is
// the fp16 pair 1024 + 16 c (exact), and (1024 + 16 c) / 16 - 64 = c exactly (one HFMA2, the
// product is exact and so is the sum), then the same HFMA2 with (scale, min).
template <bool CLAMP>
__device__ __forceinline__ uint32_t deq_pair_hi(uint32_t t, uint32_t sp, uint32_t mp, uint32_t magic) {
    uint32_t m;
    asm("lop3.b32 %0, %1, 0x00F000F0, %2, 0xEA;" : "=r"(m) : "r"(t), "r"(magic));
    const __half2 c = __hfma2(u2h(m), u2h(0x2C002C00u), u2h(0xD400D400u));           // x / 16 - 64
    const __half2 v = __hfma2(c, u2h(sp), u2h(mp));
    if constexpr (CLAMP) return h2u(__hmin2(v, u2h(0x7BFF7BFFu)));
    else return h2u(v);
}
template <bool V>
struct BoolTag {
    static constexpr bool value = V;
};
__device__ __forceinline__ uint32_t magic_h2() {   // 0x64006400 in a register (LOP3 takes one immediate)
    uint32_t m;
    asm volatile("mov.b32 %0, 0x64006400;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void mma_f16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ int64_t range_start(int64_t total, int c, int G) { return int64_t(c) * total / G; }
__device__ __forceinline__ int owner(int64_t total, int G, int64_t i) {   // CTA whose range holds panel i
    return int(((i + 1) * G - 1) / total);
}

// One stage of a consumer warp: 16 columns x 64 k against MB blocks of 8 rows; step s of the
// four accumulates into acc[s].
// Per-lane shared-memory offsets inside a stage (computed once).
struct LaneOff {
    uint32_t cw;     // code word: column n0 + g, hk0 word t
    uint32_t me;     // meta of k pairs 4t .. 4t + 3 of the warp's group
    uint32_t xr;     // x: row g, k 8t
    uint32_t xrows;  // bit mb: x row 8 mb + g exists (< M); other rows only feed discarded outputs
};
template <int MB, bool CLAMP>
__device__ __forceinline__ void stage_math(const uint8_t* st, const LaneOff& lo, uint32_t magic,
                                           float (&acc)[2][2][MB][4]) {
    // meta {scale pair, min pair} of k pairs 4t + s (hk0 word t) and 16 + 4t + s (hk1 word t)
    const uint8_t* me = st + lo.me;
    const uint4 ma0 = *reinterpret_cast<const uint4*>(me);            // pairs 4t, 4t + 1
    const uint4 ma1 = *reinterpret_cast<const uint4*>(me + 16);       // 4t + 2, 4t + 3
    const uint4 mb0 = *reinterpret_cast<const uint4*>(me + 128);      // 16 + 4t, ..
    const uint4 mb1 = *reinterpret_cast<const uint4*>(me + 144);
    const uint32_t slo[4] = {ma0.x, ma0.z, ma1.x, ma1.z}, mlo[4] = {ma0.y, ma0.w, ma1.y, ma1.w};
    const uint32_t shi[4] = {mb0.x, mb0.z, mb1.x, mb1.z}, mhi[4] = {mb0.y, mb0.w, mb1.y, mb1.w};
    // k order of the 4 MMA steps: step s takes code word hk = s / 2 of each column (hk0 word t:
    // k 8t .. 8t+7; hk1 word t: 32 + 8t ..) and its sub-pairs 2 (s % 2) (MMA k pair t) and
    // 2 (s % 2) + 1 (k pair t + 4), i.e. k = 32 hk + 8t + 4 (s % 2) + {0, 1} and {2, 3}: the B
    // fragment (b0, b1) of step s is then one 8-byte run of the x row, adjacent registers of one
    // LDS.128 (x row 8 mb + g: k 8t .. 8t+7 -> steps 0, 1; 32 + 8t .. -> steps 2, 3)
    uint4 xa[MB], xb[MB];
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
        xa[mb] = xb[mb] = make_uint4(0u, 0u, 0u, 0u);
        if (lo.xrows & (1u << mb)) {
            const uint8_t* xr = st + lo.xr + mb * 8 * 128;
            xa[mb] = *reinterpret_cast<const uint4*>(xr);
            xb[mb] = *reinterpret_cast<const uint4*>(xr + 64);
        }
    }
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
    // code words: column n0 + 16 nb + g (A rows 0..7) and + 8 (rows 8..15); hk0 word t, hk1 word t
    const uint8_t* cw = st + lo.cw + nb * 16 * 16;
    const uint32_t w00 = *reinterpret_cast<const uint32_t*>(cw);
    const uint32_t w01 = *reinterpret_cast<const uint32_t*>(cw + 4096);
    const uint32_t w10 = *reinterpret_cast<const uint32_t*>(cw + 8 * 16);
    const uint32_t w11 = *reinterpret_cast<const uint32_t*>(cw + 8 * 16 + 4096);
    // sub-pair q of a word: nibbles q, 4 + q; q = 0, 1 straight from the word, q = 2, 3 from w >> 8
    const uint32_t v00 = w00 >> 8, v01 = w01 >> 8, v10 = w10 >> 8, v11 = w11 >> 8;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int hk = s >> 1, q0 = 2 * (s & 1);         // word, first sub-pair
        const uint32_t r0 = hk ? w01 : w00, r8 = hk ? w11 : w10;             // rows g, g + 8
        const uint32_t u0 = hk ? v01 : v00, u8 = hk ? v11 : v10;
        const uint32_t* sc = hk ? shi : slo;
        const uint32_t* mn = hk ? mhi : mlo;
        const uint32_t x0 = q0 ? u0 : r0, x8 = q0 ? u8 : r8;               // sub-pairs q0 (even), q0 + 1 (odd)
        const uint32_t a0 = deq_pair<CLAMP>(x0, sc[q0], mn[q0], magic);
        const uint32_t a1 = deq_pair<CLAMP>(x8, sc[q0], mn[q0], magic);
        const uint32_t a2 = deq_pair_hi<CLAMP>(x0, sc[q0 + 1], mn[q0 + 1], magic);
        const uint32_t a3 = deq_pair_hi<CLAMP>(x8, sc[q0 + 1], mn[q0 + 1], magic);
#pragma unroll
        for (int mb = 0; mb < MB; ++mb) {
            const uint4& xv = hk ? xb[mb] : xa[mb];
            const uint32_t b0 = (s & 1) ? xv.z : xv.x;
            const uint32_t b1 = (s & 1) ? xv.w : xv.y;
            mma_f16(acc[nb][s & 1][mb], a0, a1, a2, a3, b0, b1);
        }
    }
    }
}

// y (fp16) of the lane's fragment values: v[mb] = (column col0 + n0 + g, rows 8 mb + 2t, +1) and
// (column + 8, same rows)
template <int MB>
__device__ __forceinline__ void store_y(const GemvParams& p, int col0, int n0, int lane, const float (&vv)[2][MB][4]) {
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int mb = 0; mb < MB; ++mb) {
        const int col = col0 + n0 + 16 * nb + g;
        const float (&v)[MB][4] = vv[nb];
        const int m = 8 * mb + 2 * t;
        if (m < p.M) {
            p.y[int64_t(m) * p.N + col] = __float2half_rn(v[mb][0]);
            p.y[int64_t(m) * p.N + col + 8] = __float2half_rn(v[mb][2]);
        }
        if (m + 1 < p.M) {
            p.y[int64_t(m + 1) * p.N + col] = __float2half_rn(v[mb][1]);
            p.y[int64_t(m + 1) * p.N + col + 8] = __float2half_rn(v[mb][3]);
        }
    }
}

template <int MB>
__global__ void __launch_bounds__(kThreadsV, kCtasV)
dequant_gemv_kernel(const __grid_constant__ CUtensorMap map_x, const GemvParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesV * kStageBytes);
    uint64_t* empty = full + kStagesV;
    uint32_t* flag = reinterpret_cast<uint32_t*>(empty + kStagesV);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = blockIdx.x;
    const int64_t i0 = range_start(p.total, c, p.G), i1 = range_start(p.total, c + 1, p.G);
    const int n = int(i1 - i0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesV; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumers);
        }
        flag[1] = 0u;   // the CTA's clamp flag (consumers OR the panels' flags into it)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= kConsumers) {
        // ---------------- producers: warp kConsumers + r issues stages j = r, r + 4, ... (lane 0)
        if (lane == 0) {
            const int r = warp - kConsumers;
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
            const uint64_t pol_w = policy_fractional(false), pol_x = policy_fractional(true);
            constexpr bool kNoX = FLEXQ_GEMV_PROBE == 1 || FLEXQ_GEMV_PROBE == 4;
            const uint32_t bytes = uint32_t(kPanelData + (kNoX ? 0 : p.M * 128));
            int64_t i = i0 + r;
            int kb = int(i % p.KB);
            for (int j = r; j < n; j += kProducers, i += kProducers) {
                const int s = j & (kStagesV - 1);
                mbar_wait_sleep(empty + s, ((j / kStagesV) & 1) ^ 1);
                const uint32_t dst = su32(smem + s * kStageBytes);
                mbar_expect_tx(full + s, bytes);
                bulk_g2s(dst, p.panels + i * kPanelData, kPanelData, full + s, pol_w);
                if (!kNoX) asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
                    " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst + kXOff),
                    "l"(reinterpret_cast<uint64_t>(&map_x)), "r"(kb * kGemmTileK), "r"(0), "r"(su32(full + s)),
                    "l"(pol_x)
                    : "memory");
                kb += kProducers;
                while (kb >= p.KB) kb -= p.KB;
            }
        }
        return;
    }

    // ---------------- consumers: warp owns columns n0 .. n0 + 31 of the tile (two row blocks)
    const int n0 = warp * 32;
    const int t = lane & 3, g = lane >> 2;
    const LaneOff lo{uint32_t((n0 + g) * 16 + 4 * t),
                     uint32_t(kGemmTileN * kGemmTileK / 2 + (n0 >> 6) * 256 + 32 * t),
                     uint32_t(kXOff + g * 128 + 16 * t),
                     (g < p.M ? 1u : 0u) | (8 + g < p.M ? 2u : 0u)};
    {   // the CTA's clamp flag: OR of its panels' flags (first word of each 16-byte flag)
        const uint32_t* flags = reinterpret_cast<const uint32_t*>(p.panels + p.total * kPanelData);
        uint32_t f = 0;
        for (int k = int(threadIdx.x); k < n; k += kConsumers * 32) f |= __ldg(flags + (i0 + k) * 4);
        if (__any_sync(0xffffffffu, f != 0) && lane == 0) atomicOr(flag + 1, 1u);
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
    }
    const bool clamp_cta = flag[1] != 0u;
    const uint32_t magic = magic_h2();
    float acc[2][2][MB][4];    // [row block][step parity][8-row block of x][fragment]
    int s = 0;                 // ring slot and its phase
    uint32_t ph = 0;
    int64_t i = i0;
    const int64_t first_tile = i0 / p.KB;
    while (i < i1) {
        const int64_t tile = i / p.KB;
        const int64_t seg_end = min(i1, (tile + 1) * p.KB);
        const bool whole = (i == tile * p.KB) && (seg_end == (tile + 1) * p.KB);
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int mb = 0; mb < MB; ++mb)
                    acc[nb][q][mb][0] = acc[nb][q][mb][1] = acc[nb][q][mb][2] = acc[nb][q][mb][3] = 0.0f;
        auto run = [&](auto clamp_tag) {
            constexpr bool kClamp = decltype(clamp_tag)::value;
            int left = int(seg_end - i);
#if FLEXQ_GEMV_PROBE < 3
            // two stages per iteration: their loads and conversions interleave; both are
            // released together
#pragma unroll 1
            for (; left >= 2; left -= 2) {
                const int s1 = s + 1 == kStagesV ? 0 : s + 1;
                const uint32_t ph1 = s1 == 0 ? ph ^ 1u : ph;
                mbar_wait_sleep(full + s, ph);
                mbar_wait_sleep(full + s1, ph1);
                stage_math<MB, kClamp>(smem + s * kStageBytes, lo, magic, acc);
                stage_math<MB, kClamp>(smem + s1 * kStageBytes, lo, magic, acc);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(empty + s);
                    mbar_arrive(empty + s1);
                }
                s = s1 + 1 == kStagesV ? 0 : s1 + 1;
                ph = s == 0 ? ph1 ^ 1u : ph1;
            }
#endif
#pragma unroll 1
            for (; left > 0; --left) {
                mbar_wait_sleep(full + s, ph);
                const uint8_t* st = smem + s * kStageBytes;
#if FLEXQ_GEMV_PROBE >= 3
                if (lane == 0 && *reinterpret_cast<const uint32_t*>(st) == 0x12345678u) acc[0][0][0][0] += 1.0f;
#else
                stage_math<MB, kClamp>(st, lo, magic, acc);
#endif
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
                if (++s == kStagesV) {
                    s = 0;
                    ph ^= 1u;
                }
            }
        };
        if (clamp_cta) run(BoolTag<true>{});
        else run(BoolTag<false>{});
        i = seg_end;
        float v[2][MB][4];   // the two step-parity accumulators, summed in a fixed order
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int mb = 0; mb < MB; ++mb)
#pragma unroll
                for (int r = 0; r < 4; ++r) v[nb][mb][r] = acc[nb][0][mb][r] + acc[nb][1][mb][r];
        const int col0 = int(tile) * kGemmTileN;
        if (whole) {
            store_y<MB>(p, col0, n0, lane, v);
            continue;
        }
        // a split tile: partial [256 n][16 m] in this CTA's slot (0: its first tile, 1: its last)
        const int slot = tile == first_tile ? 0 : 1;
        float* part = p.partials + (int64_t(c) * 2 + slot) * kGemmTileN * 16;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
            const int cl0 = n0 + 16 * nb + g;
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
                const int m = 8 * mb + 2 * t;
                __stcg(reinterpret_cast<float2*>(part + cl0 * 16 + m), make_float2(v[nb][mb][0], v[nb][mb][1]));
                __stcg(reinterpret_cast<float2*>(part + (cl0 + 8) * 16 + m), make_float2(v[nb][mb][2], v[nb][mb][3]));
            }
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        const int cf = owner(p.total, p.G, tile * p.KB), cl = owner(p.total, p.G, (tile + 1) * p.KB - 1);
        if (threadIdx.x == 0) {
            const uint32_t old = atomicAdd(p.tickets + tile, 1u);
            const bool last = old == uint32_t(cl - cf);
            if (last) p.tickets[tile] = 0u;
            *flag = last ? 1u : 0u;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
        if (*flag) {
            __threadfence();
            float y[2][MB][4];
#pragma unroll
            for (int nb = 0; nb < 2; ++nb)
#pragma unroll
                for (int mb = 0; mb < MB; ++mb) y[nb][mb][0] = y[nb][mb][1] = y[nb][mb][2] = y[nb][mb][3] = 0.0f;
            for (int cc = cf; cc <= cl; ++cc) {   // contributors in CTA order: deterministic
                const int sl = (tile == range_start(p.total, cc, p.G) / p.KB) ? 0 : 1;
                const float* pp = p.partials + (int64_t(cc) * 2 + sl) * kGemmTileN * 16;
#pragma unroll
                for (int nb = 0; nb < 2; ++nb) {
                    const int cl0 = n0 + 16 * nb + g;
#pragma unroll
                    for (int mb = 0; mb < MB; ++mb) {
                        const int m = 8 * mb + 2 * t;
                        const float2 a2 = __ldcg(reinterpret_cast<const float2*>(pp + cl0 * 16 + m));
                        const float2 b2 = __ldcg(reinterpret_cast<const float2*>(pp + (cl0 + 8) * 16 + m));
                        y[nb][mb][0] += a2.x;
                        y[nb][mb][1] += a2.y;
                        y[nb][mb][2] += b2.x;
                        y[nb][mb][3] += b2.y;
                    }
                }
            }
            store_y<MB>(p, col0, n0, lane, y);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");   // *flag reuse
    }
}

}  // namespace

size_t dequant_gemv_workspace_bytes(int64_t n) {
    const size_t tickets = size_t((n / kGemmTileN * 4 + 255) / 256 * 256);
    return tickets + size_t(kCtasV) * kGemmMaxGrid * 2 * kGemmTileN * 16 * sizeof(float);
}

cudaError_t launch_dequant_gemv(const void* x, const void* panels, int64_t M, int64_t K, int64_t N, void* y,
                                void* workspace, cudaStream_t stream) {
    const int KB = int(K / kGemmTileK);
    const int64_t total = (N / kGemmTileN) * KB;
    const int sms = device_sm_count();
    const int cap = kCtasV * (sms < kGemmMaxGrid ? sms : kGemmMaxGrid);
    const int G = int(total < cap ? total : cap);
    {   // the shared-memory attribute, once per device (under a lock)
        static cudaError_t attr_err[kMaxDevices];
        static std::once_flag attr_once[kMaxDevices];
        const int dev = current_device();
        std::call_once(attr_once[dev], [dev] {
            cudaError_t e = cudaFuncSetAttribute(dequant_gemv_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 kSmemV);
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(dequant_gemv_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemV);
            attr_err[dev] = e;
        });
        if (attr_err[dev] != cudaSuccess) return attr_err[dev];
    }
    GemvParams p;
    p.panels = static_cast<const uint8_t*>(panels);
    p.y = static_cast<__half*>(y);
    p.tickets = static_cast<uint32_t*>(workspace);
    p.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) +
                                          (N / kGemmTileN * 4 + 255) / 256 * 256);
    p.M = int(M);
    p.N = int(N);
    p.KB = KB;
    p.total = total;
    p.G = G;
    CUtensorMap mx;   // x [M][K] fp16, box 64 k x M rows, rows 128 B apart in the stage
    if (!make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, x, uint64_t(K), uint64_t(M), uint64_t(K * 2),
                  uint32_t(kGemmTileK), uint32_t(M), CU_TENSOR_MAP_SWIZZLE_NONE))
        return cudaErrorInvalidValue;
    if (M <= 8) dequant_gemv_kernel<1><<<G, kThreadsV, kSmemV, stream>>>(mx, p);
    else dequant_gemv_kernel<2><<<G, kThreadsV, kSmemV, stream>>>(mx, p);
    return cudaGetLastError();
}

}  // namespace flexq

// decode_attention_variants.cu -- decode attention over the b in {2, 3, 4, 8} x g in {32, 64, 128}
// KV caches (SURVEY 8(f) NEXT-3 variants; the b = 4, g = 64 cache in its default (dense) layout has
// its own tensor-core kernel, decode_attention.cu; in the token-major layout it runs here).
//
// The method is the same (P:271-274 with the cache dequantized as in P:845, reading M):
//   out = softmax(q . K^[0:cur_len]^T / sqrt(D)) . V^[0:cur_len],  K^, V^ = fmaf(c, scale, min)
// Cache layout (include/flexq.h): 32-token chunks [codes 32 x CB][meta 32 x MB] per (b, h), CB =
// D b / 8 (each token's row a little-endian bit stream, K and V alike), MB = 4 D / g.
//
// Mapping: one 128-thread CTA per (head, split); a split is a run of 128-token tiles (4 chunks).
// Per tile:
//   K pass  -- thread i owns token t0 + i: its code row comes straight from global memory (a warp
//              reads 32 consecutive rows, so the lines are fully used through L1; b = 8 stages the
//              rows in shared memory first, see KSM), its meta from global memory, and
//              score = sum_g (scale_g sum_{d in g} q_d c_d + min_g sum_{d in g} q_d) in fp32, q from
//              shared memory (broadcast reads); the per-group factoring is the exact identity of
//              sum_d q_d (c_d s_g + m_g) (reordered fp32 rounding, within reading Q).  b in
//              {2, 4, 8} forms sum q_d c_d with IDP.4A on a 22-bit fixed-point q (see IDP).
//   softmax -- block max, p = 2^(score - max) (log2 domain), running (max, sum) per CTA.
//   V pass  -- the V tile (4 chunks, contiguous) was staged into shared memory with cp.async while
//              the K pass ran; warp w takes chunk w's 32 tokens, lane group h (LPT lanes) the tokens
//              h, h + 32 / LPT, ..., lane l of it the D / LPT dims at bit l (D / LPT) b of the row
//              (whole words, or one funnel shift out of two words), and accumulates
//              acc_d += (p s_g) c_d and acc_m += p m_g (the same identity).
// Splits > 1 write (max, sum, acc[D]) partials to the workspace and a combine kernel merges them.
// CUDA cores only: one generic kernel per (b, g, D) instead of the b = 4, g = 64 kernel's
// tensor-core passes; it is instruction-issue-bound at about two instructions per code.
#include <cuda_fp16.h>
#include <stdint.h>

#include <mutex>

#include "flexq_internal.h"

namespace flexq {
namespace {

constexpr int kVThreads = 128;

struct VarParams {
    const __half* q;
    const uint8_t* kc;
    const uint8_t* vc;
    __half* out;
    float* part;          // [bh][splits][D + 2] (splits > 1)
    int64_t chunks;       // chunks per (b, h)
    int cur_len, tiles_per_split, splits;
    float scale_log2;     // log2(e) / sqrt(D)
};

// Codes become floats without a conversion instruction: (word & (mask << sh)) | 0x4B000000 is the
// float 2^23 + c 2^sh (one LOP3, exact while sh + b <= 23), and one packed FADD2 of -2^23 per pair
// leaves c 2^sh exactly.  The 2^sh factors are folded into q (K pass: qsc_d = q_d 2^-sh_d, exact)
// or removed from the accumulators at the end (V pass), so every product is the exact q_d c_d /
// p s c_d of the plain formula.
//
// Where element d of a token's bit stream is read from (K pass): bit P = d b of word i = P / 32 at
// s = P % 32; s + b > 32 (b = 3 only) -> funnel shift of words i, i + 1 (shift 0); s + b <= 23 ->
// word i at shift s; else the word's upper half w >> 16 at shift s - 16 (<= 16 - b).
template <int B>
struct ElemSrc {
    int word, kind, sh;   // kind 0: word, 1: word >> 16, 2: funnel(word, word + 1)
};
template <int B>
__host__ __device__ constexpr ElemSrc<B> elem_src(int d) {
    const int P = d * B, i = P >> 5, s = P & 31;
    return (s + B > 32) ? ElemSrc<B>{i, 2, 0} : (s + B <= 23) ? ElemSrc<B>{i, 0, s} : ElemSrc<B>{i, 1, s - 16};
}
constexpr uint32_t kMagic = 0x4B000000u;
// w | 2^23's bit pattern, opaque to the compiler: (w | M) & (K | M) == (w & K) | M is then ONE
// LOP3 with an immediate per element (given as (w & K) | M, ptxas emits two).
__device__ __forceinline__ uint32_t or_magic(uint32_t w) {
    uint32_t r;
    asm("or.b32 %0, %1, 0x4B000000;" : "=r"(r) : "r"(w));
    return r;
}
// (w >> 16) | M in one PRMT: bytes (w.2, w.3, 0, 0x4B)
__device__ __forceinline__ uint32_t hi_magic(uint32_t w) { return __byte_perm(w, kMagic, 0x7432); }

// sum_i a.u8[i] * b.s8[i] + c (exact int32)
__device__ __forceinline__ int dp4a_us(uint32_t a, uint32_t b, int c) {
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int B, int G, int D>
__global__ void __launch_bounds__(kVThreads)
attention_variant_kernel(VarParams p) {
    constexpr int CB = D * B / 8, MB = 4 * D / G, NG = D / G, CHB = kChunk * (CB + MB);
    constexpr int NWR = CB / 4;                   // code words per token row
    constexpr uint32_t kMask = (1u << B) - 1u;
    // V pass: LPT lanes per token, DPL dims per lane.  b = 8, D = 128: 8 lanes (16 dims, 4 whole
    // words; 396 -> 359 us at g = 64); else 16 lanes (one funnel-shifted word, or two words at
    // b = 8, D = 64) -- 8 lanes measured slower at b = 2 and 4 (251 -> 270 us at b = 2, g = 32)
    constexpr int LPT = (B == 8 && D == 128) ? 8 : 16;
    constexpr int TPS = 32 / LPT;                 // tokens per warp step
    constexpr int DPL = D / LPT;
    constexpr int NWIN = (DPL * B + 31) / 32;     // words of a lane's V codes
    static_assert((DPL * B) % 32 == 0 || NWIN == 1, "a lane's V codes: whole words or one funnel-shifted word");

    __shared__ __align__(16) float q_s[D];     // q_d 2^-sh_d (K pass source shift)
    __shared__ float qg_s[NG];
    __shared__ float2 psm_s[kVarTile * NG];      // V side per (token, group): (p scale, p min)
    __shared__ float red_s[kVThreads / 32];
    __shared__ __align__(16) uint8_t vbuf[4 * CHB];
    // b = 8: K codes of the tile staged in shared memory, one row per token, padded so that
    // lane-per-row LDS.128 reads of 8 consecutive rows hit 8 distinct 16-B bank groups.  With
    // 128-B rows read straight from global memory, a warp's LDG.128 touches 32 lines and the
    // small L1 left beside the shared memory re-fetches them from L2 (ncu: 1.8x the DRAM bytes
    // through L2; 433-576 -> 398-433 us).  b <= 4 reads its rows from global memory (the extra
    // copy and barrier cost more than they save there: 295 -> 307 us at b = 2).
    constexpr bool KSM = B == 8;
    constexpr int KRS = CB + (((CB / 16) % 2 == 0) ? 16 : 32);
    __shared__ __align__(16) uint8_t kbuf[KSM ? kVarTile * KRS : 16];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t bh = blockIdx.x;
    const int split = blockIdx.y;
    const int n_tiles = (p.cur_len + kVarTile - 1) / kVarTile;
    const int tile_a = split * p.tiles_per_split;
    const int tile_b = min(tile_a + p.tiles_per_split, n_tiles);

    if (tid < NG) {
        float s = 0.0f;
        for (int d = 0; d < G; ++d) s += __half2float(p.q[bh * D + tid * G + d]);
        qg_s[tid] = s;
    }
    for (int d = tid; d < D; d += kVThreads)
        q_s[d] = ldexpf(__half2float(p.q[bh * D + d]), -elem_src<B>(d).sh);
    // b in {2, 4, 8}: K pass on IDP.4A.  q in 22-bit fixed point relative to the head's max |q|,
    // Q_d = RN(q_d 2^(21 - e)) (|q| < 2^e, error <= 2^-22 of max |q|), as three signed 8-bit digits
    // Q = d0 + 2^8 d1 + 2^16 d2 (|d2| <= 32).  The codes of one 32-bit word become byte vectors with
    // one mask: (w >> b k) & (2^b - 1) * 0x01010101 holds elements 8 i / b + k (i = 0..3) of the
    // word, so digit words are stored in that order.  dp4a(u8 codes, s8 digits) sums are exact.
    constexpr bool IDP = B != 3;
    constexpr int EPW = 32 / B, KPW = 8 / B;            // elements per word, byte vectors per word
    __shared__ __align__(16) uint32_t qd_s[IDP ? 3 * (D / 4) : 4];
    float qfix = 0.0f;                                  // 2^(e - 21)
    if constexpr (IDP) {
        float a = 0.0f;
        for (int d = tid; d < D; d += kVThreads) a = fmaxf(a, fabsf(__half2float(p.q[bh * D + d])));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
        if (lane == 0) red_s[warp] = a;
        __syncthreads();
        a = fmaxf(fmaxf(red_s[0], red_s[1]), fmaxf(red_s[2], red_s[3]));
        int e = 0;
        if (a > 0.0f) frexpf(a, &e);                    // a = f 2^e, f in [0.5, 1)
        qfix = ldexpf(1.0f, e - 21);
        int8_t* qb = reinterpret_cast<int8_t*>(qd_s);
        for (int d = tid; d < D; d += kVThreads) {
            const int Q = __float2int_rn(ldexpf(__half2float(p.q[bh * D + d]), 21 - e));
            const int d0 = (Q << 24) >> 24, r1 = (Q - d0) >> 8, d1 = (r1 << 24) >> 24, d2 = (r1 - d1) >> 8;
            const int W = d / EPW, ew = d % EPW, k = ew % KPW, i = ew / KPW;
            const int byte = (W * KPW + k) * 4 + i;
            qb[byte] = int8_t(d0);
            qb[D + byte] = int8_t(d1);
            qb[2 * D + byte] = int8_t(d2);
        }
    }
    __syncthreads();

    const uint8_t* kbase = p.kc + bh * p.chunks * CHB;
    const uint8_t* vbase = p.vc + bh * p.chunks * CHB;
    const int tsub = lane / LPT, lsub = lane % LPT;
    const int vbit = lsub * DPL * B, vwi = vbit >> 5, vsh = vbit & 31, vgi = lsub * DPL / G;

    float m_run = -INFINITY, l_part = 0.0f, acc[DPL], acc_m = 0.0f;
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[e] = 0.0f;

    for (int tile = tile_a; tile < tile_b; ++tile) {
        const int t0 = tile * kVarTile;
        const int tcount = min(kVarTile, p.cur_len - t0);
        // stage the tile: K codes (padded rows) as one cp.async group, then the V chunks as a second
        // group that lands while the K pass runs
        {
            const int nch = (tcount + kChunk - 1) / kChunk;
            if constexpr (KSM) {
                const uint8_t* ksrc = kbase + int64_t(t0 / kChunk) * CHB;
                for (int i = tid; i < nch * kChunk * (CB / 16); i += kVThreads) {
                    const int r = i / (CB / 16), c = i % (CB / 16);
                    cp_async16(kbuf + r * KRS + 16 * c, ksrc + (r / kChunk) * CHB + (r % kChunk) * CB + 16 * c);
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
            const uint8_t* src = vbase + int64_t(t0 / kChunk) * CHB;
            for (int i = tid; i < nch * CHB / 16; i += kVThreads) cp_async16(vbuf + 16 * i, src + 16 * i);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if constexpr (KSM) {
            asm volatile("cp.async.wait_group 1;" ::: "memory");   // the K group
            __syncthreads();
        }
        // K pass: thread tid owns token t0 + tid
        float score = -INFINITY;
        if (tid < tcount) {
            const int t = t0 + tid;
            const uint8_t* chunk = kbase + int64_t(t / kChunk) * CHB;
            const int slot = t & (kChunk - 1);
            uint32_t w[NWR + 1];
            const uint8_t* row = KSM ? kbuf + tid * KRS : chunk + slot * CB;
            if constexpr (CB % 16 == 0) {
#pragma unroll
                for (int i = 0; i < CB / 16; ++i) {
                    const uint4 v = *reinterpret_cast<const uint4*>(row + 16 * i);
                    w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < CB / 8; ++i) {
                    const uint2 v = *reinterpret_cast<const uint2*>(row + 8 * i);
                    w[2 * i] = v.x; w[2 * i + 1] = v.y;
                }
            }
            w[NWR] = 0;
            const __half2* meta = reinterpret_cast<const __half2*>(chunk + kChunk * CB + slot * MB);
            float s = 0.0f;
            if constexpr (IDP) {
                constexpr uint32_t kByteMask = kMask * 0x01010101u;
                int acc[3][NG];
#pragma unroll
                for (int gi = 0; gi < NG; ++gi) acc[0][gi] = acc[1][gi] = acc[2][gi] = 0;
#pragma unroll
                for (int W = 0; W < NWR; ++W) {
                    const int gi = W * EPW / G;
#pragma unroll
                    for (int k = 0; k < KPW; ++k) {
                        const uint32_t v = B == 8 ? w[W] : (w[W] >> (B * k)) & kByteMask;
                        const int idx = W * KPW + k;
#pragma unroll
                        for (int j = 0; j < 3; ++j) acc[j][gi] = dp4a_us(v, qd_s[j * (D / 4) + idx], acc[j][gi]);
                    }
                }
#pragma unroll
                for (int gi = 0; gi < NG; ++gi) {
                    const float dot = fmaf(65536.0f, float(acc[2][gi]), fmaf(256.0f, float(acc[1][gi]), float(acc[0][gi])));
                    const float2 sm = __half22float2(meta[gi]);
                    s = fmaf(sm.x * qfix, dot, fmaf(sm.y, qg_s[gi], s));
                }
            } else {
            uint32_t wm[NWR], hm[NWR];
#pragma unroll
            for (int i = 0; i < NWR; ++i) {
                wm[i] = or_magic(w[i]);
                hm[i] = hi_magic(w[i]);
            }
            const float2 nbias = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                float2 dot[2] = {make_float2(0.0f, 0.0f), make_float2(0.0f, 0.0f)};
#pragma unroll
                for (int dd = 0; dd < G; dd += 4) {
                    const float4 qq = *reinterpret_cast<const float4*>(&q_s[gi * G + dd]);
                    float f[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const ElemSrc<B> es = elem_src<B>(gi * G + dd + e);
                        const uint32_t src =
                            es.kind == 0   ? wm[es.word]
                            : es.kind == 1 ? hm[es.word]
                                           : or_magic(__funnelshift_r(w[es.word], w[es.word + 1], (gi * G + dd + e) * B & 31));
                        f[e] = __uint_as_float(src & ((kMask << es.sh) | kMagic));
                    }
                    const float2 c01 = __fadd2_rn(make_float2(f[0], f[1]), nbias);
                    const float2 c23 = __fadd2_rn(make_float2(f[2], f[3]), nbias);
                    dot[0] = __ffma2_rn(make_float2(qq.x, qq.y), c01, dot[0]);
                    dot[1] = __ffma2_rn(make_float2(qq.z, qq.w), c23, dot[1]);
                }
                const float2 sm = __half22float2(meta[gi]);
                s = fmaf(sm.x, (dot[0].x + dot[0].y) + (dot[1].x + dot[1].y), fmaf(sm.y, qg_s[gi], s));
            }
            }
            score = s * p.scale_log2;
        }
        // block max -> running max, probabilities
        float mx = score;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) red_s[warp] = mx;
        __syncthreads();
        mx = fmaxf(fmaxf(red_s[0], red_s[1]), fmaxf(red_s[2], red_s[3]));
        const float m_new = fmaxf(m_run, mx);
        const float alpha = exp2f(m_run - m_new);
        const float pt = (tid < tcount) ? exp2f(score - m_new) : 0.0f;
        l_part = fmaf(l_part, alpha, pt);
        m_run = m_new;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] *= alpha;
        acc_m *= alpha;
        cp_async_wait_all();
        __syncthreads();
        // the V meta of token tid, times its probability, once per (token, group)
        if (tid < tcount) {
            const __half2* vm = reinterpret_cast<const __half2*>(vbuf + (tid >> 5) * CHB + kChunk * CB +
                                                                 (tid & (kChunk - 1)) * MB);
#pragma unroll
            for (int gi = 0; gi < NG; ++gi) {
                const float2 sm = __half22float2(vm[gi]);
                psm_s[tid * NG + gi] = make_float2(pt * sm.x, pt * sm.y);
            }
        }
        __syncthreads();
        // V pass: warp w takes chunk w of the tile
        const int nj = min(kChunk, tcount - warp * kChunk);
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(vbuf + warp * CHB);
        const float2* pw = psm_s + warp * kChunk * NG + vgi;
#pragma unroll 2
        for (int j = tsub; j < nj; j += TPS) {   // lane group h takes tokens h, h + TPS, ...
            uint32_t x[NWIN];
            if constexpr ((DPL * B) % 32 != 0) {
                x[0] = __funnelshift_r(cw[j * NWR + vwi], cw[j * NWR + vwi + 1], vsh);
            } else {
#pragma unroll
                for (int i = 0; i < NWIN; ++i) x[i] = cw[j * NWR + vwi + i];
            }
            uint32_t xm[NWIN], xh[NWIN];
#pragma unroll
            for (int i = 0; i < NWIN; ++i) {
                xm[i] = or_magic(x[i]);
                xh[i] = hi_magic(x[i]);
            }
            const float2 pp = pw[j * NG];
            const float ps = pp.x;
            acc_m += pp.y;
            float f[DPL];
#pragma unroll
            for (int e = 0; e < DPL; ++e) {   // element e at bit e b of the window: 2^23 + c 2^sh_e
                const int wi = e * B / 32, sh = e * B % 32;
                f[e] = __uint_as_float(sh + B <= 23 ? (xm[wi] & ((kMask << sh) | kMagic))
                                                    : (xh[wi] & ((kMask << (sh - 16)) | kMagic)));
            }
#pragma unroll
            for (int e = 0; e < DPL; e += 2) {
                const float2 c = __fadd2_rn(make_float2(f[e], f[e + 1]), make_float2(-8388608.0f, -8388608.0f));
                const float2 r = __ffma2_rn(make_float2(ps, ps), c, make_float2(acc[e], acc[e + 1]));
                acc[e] = r.x;
                acc[e + 1] = r.y;
            }
        }
        __syncthreads();   // vbuf / psm_s are rewritten by the next tile
    }

    // combine: the warp's lane groups by shuffles, then the 4 warps (all share m_run)
#pragma unroll
    for (int o = LPT; o < 32; o <<= 1) {
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
        acc_m += __shfl_xor_sync(0xffffffffu, acc_m, o);
    }
    float* comb = reinterpret_cast<float*>(vbuf);   // [4][D]: fits every variant's 4 staged chunks
    static_assert(4 * D * 4 <= 4 * CHB, "combine buffer");
    if (tsub == 0) {
#pragma unroll
        for (int e = 0; e < DPL; ++e) {   // remove the 2^sh factor of element e (exact)
            const int s0 = e * B % 32, sh = s0 + B <= 23 ? s0 : s0 - 16;
            comb[warp * D + lsub * DPL + e] = ldexpf(acc[e], -sh) + acc_m;
        }
    }
    float l = l_part;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) red_s[warp] = l;
    __syncthreads();
    l = (red_s[0] + red_s[1]) + (red_s[2] + red_s[3]);
    for (int d = tid; d < D; d += kVThreads) {
        const float o = (comb[d] + comb[D + d]) + (comb[2 * D + d] + comb[3 * D + d]);
        if (p.splits == 1) {
            p.out[bh * D + d] = __float2half_rn(o / l);
        } else {
            float* part = p.part + (bh * p.splits + split) * (D + 2);
            if (d == 0) {
                part[0] = m_run;
                part[1] = l;
            }
            part[2 + d] = o;
        }
    }
}

// out = sum_i 2^(m_i - m) acc_i / sum_i 2^(m_i - m) l_i over the splits of one head
template <int D>
__global__ void __launch_bounds__(D)
attention_variant_combine(const float* __restrict__ part, __half* __restrict__ out, int splits) {
    const int64_t bh = blockIdx.x;
    const int d = threadIdx.x;
    const float* pp = part + bh * splits * (D + 2);
    float m = -INFINITY;
    for (int i = 0; i < splits; ++i) m = fmaxf(m, pp[i * (D + 2)]);
    float num = 0.0f, den = 0.0f;
    for (int i = 0; i < splits; ++i) {
        const float w = exp2f(pp[i * (D + 2)] - m);
        den = fmaf(w, pp[i * (D + 2) + 1], den);
        num = fmaf(w, pp[i * (D + 2) + 2 + d], num);
    }
    out[bh * D + d] = __float2half_rn(num / den);
}

int sm_count() { return device_sm_count(); }

template <int B, int G, int D>
cudaError_t launch_var(const AttnArgs& a, cudaStream_t stream) {
    const int64_t bhs = int64_t(a.batch) * a.heads;
    const int n_tiles = (a.cur_len + kVarTile - 1) / kVarTile;
    const int64_t target = int64_t(sm_count()) * 8;                   // CTAs to fill the GPU
    int want = int((target + bhs - 1) / bhs);
    if (want > n_tiles) want = n_tiles;
    if (want < 1) want = 1;
    const int tps = (n_tiles + want - 1) / want;
    const int splits = (n_tiles + tps - 1) / tps;
    VarParams p;
    p.q = static_cast<const __half*>(a.q);
    p.kc = static_cast<const uint8_t*>(a.k_cache);
    p.vc = static_cast<const uint8_t*>(a.v_cache);
    p.out = static_cast<__half*>(a.out);
    p.part = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + 256);
    p.chunks = a.chunks;
    p.cur_len = a.cur_len;
    p.tiles_per_split = tps;
    p.splits = splits;
    p.scale_log2 = 1.4426950408889634f / sqrtf(float(D));
    attention_variant_kernel<B, G, D><<<dim3(unsigned(bhs), unsigned(splits)), kVThreads, 0, stream>>>(p);
    if (splits > 1) attention_variant_combine<D><<<unsigned(bhs), D, 0, stream>>>(p.part, p.out, splits);
    return cudaGetLastError();
}

template <int B, int G>
cudaError_t launch_var_d(const AttnArgs& a, cudaStream_t stream) {
    if (a.head_dim == 128) return launch_var<B, G, 128>(a, stream);
    if constexpr (G <= 64) return launch_var<B, G, 64>(a, stream);
    return cudaErrorInvalidValue;
}

}  // namespace

size_t attention_variant_workspace_bytes(int batch, int heads, int head_dim, int t_cap) {
    const size_t tiles = size_t((t_cap + kVarTile - 1) / kVarTile);
    return 256 + (size_t(batch) * heads * tiles * size_t(head_dim + 2) * 4 + 15) / 16 * 16;
}

cudaError_t launch_decode_attention_variant(const AttnArgs& a, int bits, int group, cudaStream_t stream) {
    switch (bits * 1000 + group) {
        case 2032: return launch_var_d<2, 32>(a, stream);
        case 2064: return launch_var_d<2, 64>(a, stream);
        case 2128: return launch_var_d<2, 128>(a, stream);
        case 3032: return launch_var_d<3, 32>(a, stream);
        case 3064: return launch_var_d<3, 64>(a, stream);
        case 3128: return launch_var_d<3, 128>(a, stream);
        case 4032: return launch_var_d<4, 32>(a, stream);
        case 4064: return launch_var_d<4, 64>(a, stream);   // the (4, 64) cache in the token-major layout
        case 4128: return launch_var_d<4, 128>(a, stream);
        case 8032: return launch_var_d<8, 32>(a, stream);
        case 8064: return launch_var_d<8, 64>(a, stream);
        case 8128: return launch_var_d<8, 128>(a, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace flexq

/*
 * flexq_oracle.c -- plain, slow, obviously-correct CPU oracle for the FlexGen
 * compressed-KV decode-attention hot path (arXiv 2303.06865).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2303_06865_b200/, libflexq.so) never links, imports
 * or calls anything in oracle/, and this file shares no code, header, table
 * or constant generator with paper_2303_06865_b200/csrc/.
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math -shared -fPIC
 *        (no FMA contraction: every float operation below rounds once, in the
 *         order written; fmaf() is called explicitly where a fused op is meant.)
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * SURVEY 8(c) rows O1..O8 / readings A..S are restated in DESIGN.md.
 *
 *   O1  fp16 codec (own bit-level implementation; pinned vs numpy in tests)
 *   O2  grouping: g contiguous elements along the last axis
 *   O3  group min / max
 *   O4  x_quant = round((x - min)/(max - min) * (2^b - 1))
 *         fp32, literal operand order, IEEE division, round-half-even  (readings A, B)
 *         degenerate max == min -> codes 0                          (reading C)
 *   O5  metadata (scale, min) as fp16, scale = (max-min)/(2^b-1)   (reading E)
 *   O6  pack two 4-bit codes per byte, even element in low nibble  (reading H);
 *         any b: a little-endian bit stream per row (NEXT-3 variants)
 *   O7  dequantize: f16(clamp(fmaf(code, scale, min), +-65504))    (readings R)
 *   O8  decode attention softmax(q K^T / sqrt(D)) V over the dequantized cache
 *         (P:271-274), K^ and V^ = fmaf(code, scale, min) in fp32   (reading M)
 *   A4  KV update x_K <- Concat(x_K, t w_K): append quantized rows
 *   G1  decode linear layer y = t . w^ over a 4-bit weight grouped along the
 *         output channel, w^ = O7 fp16 (NEXT-2)
 *
 * Parity pins: see tests/test_oracle_*.py (each function is pinned there to
 * something other than itself: exact rational arithmetic, brute-force search,
 * closed forms, invariants, numpy's fp16 codec).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OK 0
#define ERR_ARG 2
#define ERR_UNSUPPORTED 4

/* ------------------------------------------------------------------ O1 */
/* f16 -> f32, exact.  IEEE binary16: 1 sign, 5 exponent (bias 15), 10 fraction. */
float oracle_f16_to_f32(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    float v;
    if (e == 0) {
        v = ldexpf((float)m, -24);              /* subnormal: m * 2^-24 */
    } else if (e == 31) {
        v = (m == 0) ? INFINITY : NAN;
    } else {
        v = ldexpf((float)(1024 + m), e - 25);  /* (1 + m/1024) * 2^(e-15) */
    }
    return sign ? -v : v;
}

/* Round a non-negative float that is < 2^23 to the nearest integer, ties to
 * even.  t - floor(t) is exact in this range. */
static float round_half_even(float t)
{
    float f = floorf(t);
    float d = t - f;
    if (d > 0.5f) return f + 1.0f;
    if (d < 0.5f) return f;
    return (fmodf(f, 2.0f) == 0.0f) ? f : f + 1.0f;
}

/* f32 -> f16, round to nearest even; overflow -> inf; subnormals kept. */
uint16_t oracle_f32_to_f16(float f)
{
    if (isnan(f)) return 0x7e00;
    uint16_t sign = signbit(f) ? 0x8000 : 0;
    float a = fabsf(f);
    if (a >= 65520.0f) return sign | 0x7c00;    /* midpoint of 65504 and 2^16 rounds to even = inf */
    if (a < ldexpf(1.0f, -14)) {
        /* subnormal range: units of 2^-24; m == 1024 is the smallest normal 0x0400 */
        float m = round_half_even(ldexpf(a, 24));
        return sign | (uint16_t)m;
    }
    int e;
    frexpf(a, &e);                              /* a = fr * 2^e, fr in [0.5, 1) */
    e -= 1;                                     /* a in [2^e, 2^(e+1)) */
    float sig = round_half_even(ldexpf(a, 10 - e));   /* in [1024, 2048] */
    if (sig == 2048.0f) { sig = 1024.0f; e += 1; }
    if (e > 15) return sign | 0x7c00;
    return sign | (uint16_t)(((e + 15) << 10) | ((int)sig - 1024));
}

/* ------------------------------------------------------------------ O3-O5 */
/* Quantize one group of g fp16 values.  codes: one code per byte. */
static void quantize_group(const uint16_t *x, int g, int bits,
                           uint8_t *codes, uint16_t *scale16, uint16_t *min16)
{
    const float levels = (float)((1 << bits) - 1);       /* 2^b - 1 */
    float mn = oracle_f16_to_f32(x[0]);
    float mx = mn;
    for (int j = 1; j < g; ++j) {                         /* O3: exact extrema */
        float v = oracle_f16_to_f32(x[j]);
        if (v < mn) mn = v;
        if (v > mx) mx = v;
    }
    if (mn == 0.0f) mn = 0.0f;                            /* reading P: -0 -> +0 */
    float r = mx - mn;                                    /* RN32(max - min) */
    *min16 = oracle_f32_to_f16(mn);                       /* exact: mn is an fp16 value */
    if (r == 0.0f) {                                      /* reading C: degenerate group */
        for (int j = 0; j < g; ++j) codes[j] = 0;
        *scale16 = 0;
        return;
    }
    *scale16 = oracle_f32_to_f16(r / levels);             /* O5: f16(RN32(r / (2^b-1))) */
    for (int j = 0; j < g; ++j) {                         /* O4, literal order of P:843 */
        float xv = oracle_f16_to_f32(x[j]);
        float a = xv - mn;                                /* RN32(x - min)            */
        float u = a / r;                                  /* RN32(a / (max - min))    */
        float t = u * levels;                             /* RN32(u * (2^b - 1))      */
        t = fminf(fmaxf(t, 0.0f), levels);                /* reading D: no-op clamp   */
        codes[j] = (uint8_t)round_half_even(t);           /* reading A: half to even  */
    }
}

/* Quantize x[rows][cols] (fp16 bits) in groups of `group` along cols.
 * codes: rows*cols bytes, one code per element (unpacked).
 * meta:  rows*(cols/group)*2 uint16: {scale16, min16} per group (reading E). */
int oracle_quantize(const uint16_t *x, int64_t rows, int64_t cols, int bits, int group,
                    uint8_t *codes, uint16_t *meta)
{
    if (rows < 0 || cols < 0 || bits < 1 || bits > 8 || group < 1) return ERR_ARG;
    if (cols % group != 0) return ERR_UNSUPPORTED;        /* reading I: no partial groups */
    int64_t ng = cols / group;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t k = 0; k < ng; ++k) {
            int64_t off = r * cols + k * group;
            int64_t mo = (r * ng + k) * 2;
            quantize_group(x + off, group, bits, codes + off, &meta[mo], &meta[mo + 1]);
        }
    return OK;
}

/* ------------------------------------------------------------------ O6 */
/* Byte k = code[2k] | code[2k+1] << 4  (reading H).  n must be even. */
int oracle_pack4(const uint8_t *codes, int64_t n, uint8_t *packed)
{
    if (n < 0 || (n & 1)) return ERR_ARG;
    for (int64_t k = 0; k < n / 2; ++k)
        packed[k] = (uint8_t)((codes[2 * k] & 0xf) | ((codes[2 * k + 1] & 0xf) << 4));
    return OK;
}

int oracle_unpack4(const uint8_t *packed, int64_t n, uint8_t *codes)
{
    if (n < 0 || (n & 1)) return ERR_ARG;
    for (int64_t k = 0; k < n / 2; ++k) {
        codes[2 * k] = packed[k] & 0xf;
        codes[2 * k + 1] = packed[k] >> 4;
    }
    return OK;
}

/* O6 for any bit width b in [1, 8] (NEXT-3 variants): the codes of n elements form a
 * little-endian bit stream, "codes packed little-endian bit-order within bytes":
 * bit i of code j is stream bit j*b + i, stream bit s is bit s % 8 of byte s / 8.
 * For b = 4 this is oracle_pack4's byte k = code[2k] | code[2k+1] << 4.
 * n * b must be a multiple of 8 (whole bytes). */
int oracle_pack_bits(const uint8_t *codes, int64_t n, int bits, uint8_t *packed)
{
    if (n < 0 || bits < 1 || bits > 8 || (n * bits) % 8 != 0) return ERR_ARG;
    for (int64_t k = 0; k < n * bits / 8; ++k) packed[k] = 0;
    for (int64_t j = 0; j < n; ++j)
        for (int i = 0; i < bits; ++i) {
            int64_t sbit = j * bits + i;
            if ((codes[j] >> i) & 1) packed[sbit / 8] |= (uint8_t)(1u << (sbit % 8));
        }
    return OK;
}

int oracle_unpack_bits(const uint8_t *packed, int64_t n, int bits, uint8_t *codes)
{
    if (n < 0 || bits < 1 || bits > 8 || (n * bits) % 8 != 0) return ERR_ARG;
    for (int64_t j = 0; j < n; ++j) {
        unsigned c = 0;
        for (int i = 0; i < bits; ++i) {
            int64_t sbit = j * bits + i;
            c |= (unsigned)((packed[sbit / 8] >> (sbit % 8)) & 1) << i;
        }
        codes[j] = (uint8_t)c;
    }
    return OK;
}

/* ------------------------------------------------------------------ O7 */
/* Dequantized value in fp32, before any fp16 rounding (reading M). */
static float dequant_f32(uint8_t code, uint16_t scale16, uint16_t min16)
{
    return fmaf((float)code, oracle_f16_to_f32(scale16), oracle_f16_to_f32(min16));
}

/* out[rows][cols] fp16 = f16(clamp(fmaf(code, scale, min), -65504, 65504))  (reading R) */
int oracle_dequantize(const uint8_t *codes, const uint16_t *meta, int64_t rows, int64_t cols,
                      int bits, int group, uint16_t *out)
{
    if (rows < 0 || cols < 0 || bits < 1 || bits > 8 || group < 1) return ERR_ARG;
    if (cols % group != 0) return ERR_UNSUPPORTED;
    int64_t ng = cols / group;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < cols; ++c) {
            int64_t mo = (r * ng + c / group) * 2;
            float v = dequant_f32(codes[r * cols + c], meta[mo], meta[mo + 1]);
            v = fminf(fmaxf(v, -65504.0f), 65504.0f);
            out[r * cols + c] = oracle_f32_to_f16(v);
        }
    return OK;
}

/* ------------------------------------------------------------------ A4 */
/* KV update: quantize the n_new new tokens of every (b, h) in
 * groups along the head dimension and write them at cache positions
 * [pos, pos + n_new).  k_new, v_new: fp16 [B][H][n_new][D].
 * caches: codes [B][H][T_cap][D] (unpacked), meta [B][H][T_cap][D/group][2]. */
int oracle_append_kv(const uint16_t *k_new, const uint16_t *v_new,
                     int B, int H, int D, int T_cap, int pos, int n_new, int bits, int group,
                     uint8_t *k_codes, uint16_t *k_meta, uint8_t *v_codes, uint16_t *v_meta)
{
    if (B < 1 || H < 1 || D < 1 || T_cap < 1 || bits < 1 || bits > 8 || group < 1) return ERR_ARG;
    if (pos < 0 || n_new < 1 || pos + n_new > T_cap) return ERR_ARG;
    if (D % group != 0) return ERR_UNSUPPORTED;
    int ng = D / group;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
            for (int t = 0; t < n_new; ++t) {
                int64_t src = (((int64_t)b * H + h) * n_new + t) * D;
                int64_t row = ((int64_t)b * H + h) * T_cap + pos + t;
                for (int k = 0; k < ng; ++k) {
                    int64_t mo = (row * ng + k) * 2;
                    quantize_group(k_new + src + k * group, group, bits,
                                   k_codes + row * D + k * group, &k_meta[mo], &k_meta[mo + 1]);
                    quantize_group(v_new + src + k * group, group, bits,
                                   v_codes + row * D + k * group, &v_meta[mo], &v_meta[mo + 1]);
                }
            }
    return OK;
}

/* ------------------------------------------------------------------ O8 */
/* Dequantized cache element of head (b,h), token t, column j, as fp32 (reading M:
 * fmaf(code, scale, min), never rounded to fp16). */
static float cache_elem(const uint8_t *codes, const uint16_t *meta, int64_t row, int D, int group, int j)
{
    int64_t mo = (row * (D / group) + j / group) * 2;
    return dequant_f32(codes[row * D + j], meta[mo], meta[mo + 1]);
}

/* Textbook decode attention in double (reading K: sqrt(head_dim)):
 *   s_t = (sum_j q_j K^_tj) / sqrt(D),  p_t = exp(s_t - max s) / sum exp(.),
 *   o_j = sum_t p_t V^_tj,   t in [0, cur_len).
 * q: fp16 [B][H][D]; caches as in oracle_append_kv; out: double [B][H][D].
 * probs (optional, may be NULL): double [B][H][cur_len] softmax weights. */
int oracle_attention_f64(const uint16_t *q, const uint8_t *k_codes, const uint16_t *k_meta,
                         const uint8_t *v_codes, const uint16_t *v_meta,
                         int B, int H, int D, int T_cap, int cur_len, int group,
                         double *out, double *probs)
{
    if (B < 1 || H < 1 || D < 1 || T_cap < 1 || group < 1) return ERR_ARG;
    if (cur_len < 1 || cur_len > T_cap) return ERR_ARG;
    if (D % group != 0) return ERR_UNSUPPORTED;
    double *s = (double *)malloc(sizeof(double) * (size_t)cur_len);
    if (!s) return ERR_ARG;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h) {
            int64_t bh = (int64_t)b * H + h;
            const uint16_t *qh = q + bh * D;
            double mx = -INFINITY;
            for (int t = 0; t < cur_len; ++t) {
                int64_t row = bh * T_cap + t;
                double acc = 0.0;
                for (int j = 0; j < D; ++j)
                    acc += (double)oracle_f16_to_f32(qh[j]) *
                           (double)cache_elem(k_codes, k_meta, row, D, group, j);
                s[t] = acc / sqrt((double)D);
                if (s[t] > mx) mx = s[t];
            }
            double z = 0.0;
            for (int t = 0; t < cur_len; ++t) { s[t] = exp(s[t] - mx); z += s[t]; }
            for (int t = 0; t < cur_len; ++t) {
                s[t] /= z;
                if (probs) probs[bh * cur_len + t] = s[t];
            }
            for (int j = 0; j < D; ++j) {
                double o = 0.0;
                for (int t = 0; t < cur_len; ++t)
                    o += s[t] * (double)cache_elem(v_codes, v_meta, bh * T_cap + t, D, group, j);
                out[bh * D + j] = o;
            }
        }
    free(s);
    return OK;
}

/* The same definition evaluated in fp32: sigma = 1/sqrtf(D),
 * s_t = sigma * sum_{j asc} q_j K^_tj, e_t = expf(s_t - M), o_j = (sum_t e_t V^_tj) / Z. */
int oracle_attention_f32(const uint16_t *q, const uint8_t *k_codes, const uint16_t *k_meta,
                         const uint8_t *v_codes, const uint16_t *v_meta,
                         int B, int H, int D, int T_cap, int cur_len, int group,
                         float *out)
{
    if (B < 1 || H < 1 || D < 1 || T_cap < 1 || group < 1) return ERR_ARG;
    if (cur_len < 1 || cur_len > T_cap) return ERR_ARG;
    if (D % group != 0) return ERR_UNSUPPORTED;
    float *e = (float *)malloc(sizeof(float) * (size_t)cur_len);
    if (!e) return ERR_ARG;
    const float sigma = 1.0f / sqrtf((float)D);
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h) {
            int64_t bh = (int64_t)b * H + h;
            const uint16_t *qh = q + bh * D;
            float mx = -INFINITY;
            for (int t = 0; t < cur_len; ++t) {
                int64_t row = bh * T_cap + t;
                float acc = 0.0f;
                for (int j = 0; j < D; ++j)
                    acc += oracle_f16_to_f32(qh[j]) * cache_elem(k_codes, k_meta, row, D, group, j);
                e[t] = sigma * acc;
                if (e[t] > mx) mx = e[t];
            }
            float z = 0.0f;
            for (int t = 0; t < cur_len; ++t) { e[t] = expf(e[t] - mx); z += e[t]; }
            for (int j = 0; j < D; ++j) {
                float o = 0.0f;
                for (int t = 0; t < cur_len; ++t)
                    o += e[t] * cache_elem(v_codes, v_meta, bh * T_cap + t, D, group, j);
                out[bh * D + j] = o / z;
            }
        }
    free(e);
    return OK;
}

/* ------------------------------------------------------------------ NEXT-1 */
/* Top-K sparse attention ("for each query, we calculate the indices
 * of its Top-K tokens from the K cache ... drop the other tokens and only load
 * a subset of the V cache"): scores s_t as in oracle_attention_f64;
 * keep the `keep` highest scores (equal scores: lower token index first);
 * softmax renormalised over the kept set; o = sum_kept p_t V^_t.
 * sel_in (optional): 0/1 mask [B][H][cur_len] of a kept set to evaluate
 * instead of selecting (lets a test score a set chosen elsewhere).
 * sel_out (optional): the kept mask; scores_out (optional): s_t (double).
 * Selection is the definition written out: token t is kept iff
 * #{u : s_u > s_t or (s_u == s_t and u < t)} < keep  (O(n^2)). */
int oracle_attention_topk_f64(const uint16_t *q, const uint8_t *k_codes, const uint16_t *k_meta,
                              const uint8_t *v_codes, const uint16_t *v_meta,
                              int B, int H, int D, int T_cap, int cur_len, int group, int keep,
                              const uint8_t *sel_in, uint8_t *sel_out, double *scores_out, double *out)
{
    if (B < 1 || H < 1 || D < 1 || T_cap < 1 || group < 1) return ERR_ARG;
    if (cur_len < 1 || cur_len > T_cap || keep < 1 || keep > cur_len) return ERR_ARG;
    if (D % group != 0) return ERR_UNSUPPORTED;
    double *s = (double *)malloc(sizeof(double) * (size_t)cur_len);
    uint8_t *kept = (uint8_t *)malloc((size_t)cur_len);
    if (!s || !kept) { free(s); free(kept); return ERR_ARG; }
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h) {
            int64_t bh = (int64_t)b * H + h;
            const uint16_t *qh = q + bh * D;
            for (int t = 0; t < cur_len; ++t) {
                int64_t row = bh * T_cap + t;
                double acc = 0.0;
                for (int j = 0; j < D; ++j)
                    acc += (double)oracle_f16_to_f32(qh[j]) *
                           (double)cache_elem(k_codes, k_meta, row, D, group, j);
                s[t] = acc / sqrt((double)D);
                if (scores_out) scores_out[bh * cur_len + t] = s[t];
            }
            for (int t = 0; t < cur_len; ++t) {
                if (sel_in) {
                    kept[t] = sel_in[bh * cur_len + t] ? 1 : 0;
                } else {
                    int rank = 0;
                    for (int u = 0; u < cur_len; ++u)
                        if (s[u] > s[t] || (s[u] == s[t] && u < t)) ++rank;
                    kept[t] = rank < keep;
                }
                if (sel_out) sel_out[bh * cur_len + t] = kept[t];
            }
            double mx = -INFINITY;
            for (int t = 0; t < cur_len; ++t)
                if (kept[t] && s[t] > mx) mx = s[t];
            double z = 0.0;
            for (int t = 0; t < cur_len; ++t)
                if (kept[t]) z += exp(s[t] - mx);
            for (int j = 0; j < D; ++j) {
                double o = 0.0;
                for (int t = 0; t < cur_len; ++t)
                    if (kept[t])
                        o += exp(s[t] - mx) / z *
                             (double)cache_elem(v_codes, v_meta, bh * T_cap + t, D, group, j);
                out[bh * D + j] = o;
            }
        }
    free(s);
    free(kept);
    return OK;
}

/* ------------------------------------------------------------------ G1 */
/* Decode-step linear layer over a group-wise 4-bit weight:
 * y = t . w with w in R^{h1 x h2}, stored quantized
 * ("compress both [weights and KV cache] to 4 bits with a group
 * size of 64"), grouped "along the output channel dimension" (reading
 * J: contiguous groups along the last axis of the [in][out] matrix), and
 * "converted back to FP16 before computation": the operand is
 * O7's fp16 value, exactly what oracle_dequantize returns.
 *
 *   x     fp16 [M][K]            (M = batch b, K = in features)
 *   codes u8   [K][N] unpacked   (N = out features)
 *   meta  u16  [K][N/group][2]   ({scale, min} fp16 bit patterns)
 *   out   f64  [M][N] = sum_k x[m][k] * w^[k][n], summed in double, k ascending.
 * The plain definition of a matrix product (no blocking, no reordering). */
int oracle_dequant_gemm_f64(const uint16_t *x, const uint8_t *codes, const uint16_t *meta,
                            int64_t M, int64_t K, int64_t N, int bits, int group, double *out)
{
    if (M < 0 || K < 0 || N < 0 || bits < 1 || bits > 8 || group < 1) return ERR_ARG;
    if (N % group != 0) return ERR_UNSUPPORTED;
    int64_t ng = N / group;
    /* O7 per weight element, then the product. */
    double *w = (double *)malloc(sizeof(double) * (size_t)(K * N > 0 ? K * N : 1));
    if (!w) return ERR_ARG;
    for (int64_t k = 0; k < K; ++k)
        for (int64_t n = 0; n < N; ++n) {
            int64_t mo = (k * ng + n / group) * 2;
            float v = dequant_f32(codes[k * N + n], meta[mo], meta[mo + 1]);
            v = fminf(fmaxf(v, -65504.0f), 65504.0f);
            w[k * N + n] = (double)oracle_f16_to_f32(oracle_f32_to_f16(v));
        }
    for (int64_t m = 0; m < M; ++m)
        for (int64_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += (double)oracle_f16_to_f32(x[m * K + k]) * w[k * N + n];
            out[m * N + n] = acc;
        }
    free(w);
    return OK;
}

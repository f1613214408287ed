/*
 * flexq.h -- C ABI of the B200 (sm_100a) compressed-KV decode-attention library.
 *
 * The library implements the data-parallel hot path of FlexGen's approximate
 * method (Sheng et al., arXiv 2303.06865, Sec. 4 "Approximate Methods"):
 * group-wise asymmetric b-bit quantization of the KV cache, grouped along the
 * hidden dimension, and decode-step attention over that
 * compressed cache, with dequantization fused into the attention
 * kernel.  Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n; the
 * readings of ambiguous passages (A..S) are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a CUDA device pointer on the current device and
 *    must be 16-byte aligned (else FLEXQ_ERR_ALIGN).  The caller owns all
 *    buffers; the library never allocates, frees or synchronizes.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    stream-ordered and asynchronous, and are safe to capture in CUDA graphs.
 *  - Argument validation runs first, on the host, before any CUDA call; a
 *    rejected call returns its status and writes nothing.  FLEXQ_ERR_CUDA is
 *    returned when the launch itself fails; faults inside a kernel surface at
 *    the caller's next synchronization.
 *  - Inputs must be finite; NaN / Inf inputs give unspecified codes.
 *  - fp16 = IEEE binary16 (`half`); half2 meta = {.x = scale, .y = min}.
 *  - The library keeps no mutable global state beyond per-device launch facts (SM count,
 *    kernel occupancy, the shared-memory attribute), computed once per device under a lock:
 *    calls are reentrant and may target several devices.
 */
#ifndef FLEXQ_H
#define FLEXQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLEXQ_ABI_VERSION 2   /* 2: the kv_layout argument of the KV-cache calls */

typedef enum {
    FLEXQ_OK = 0,
    FLEXQ_ERR_NULL = 1,        /* a required pointer is NULL                                  */
    FLEXQ_ERR_ARG = 2,         /* size / index out of range: a dimension < 1, bits not in
                                  [1, 8], group_size < 1, pos < 0,
                                  pos + n_new > prompt_len + gen_len, cur_len not in
                                  [1, prompt_len + gen_len]                                  */
    FLEXQ_ERR_ALIGN = 3,       /* a tensor pointer is not 16-byte aligned                     */
    FLEXQ_ERR_UNSUPPORTED = 4, /* legal per the paper but not built: (bits, group_size) other
                                  than (4, 64) -- except flexq_quantize /
                                  flexq_dequantize, which also build bits in {2, 3, 8} and
                                  group_size in {32, 128}; head_dim not in {64, 128},
                                  cols % group_size != 0 (reading I)                          */
    FLEXQ_ERR_WORKSPACE = 5,   /* workspace NULL or smaller than the size query              */
    FLEXQ_ERR_CUDA = 6         /* a CUDA launch / attribute call failed                       */
} flexq_status;

/* = FLEXQ_ABI_VERSION. */
int flexq_abi_version(void);

/* KV cache layouts: the `kv_layout` argument of every call that reads or writes a KV cache
 * (layouts below, at "KV cache layout").  Any other value -> FLEXQ_ERR_ARG.
 *   FLEXQ_KV_DENSE        the default.  (4, 64): K token-major, V quad-interleaved and swizzled
 *                         (the operand order of the tensor-core decode kernel); the variants:
 *                         K and V token-major.
 *   FLEXQ_KV_TOKEN_MAJOR  K and V token-major for every built (bits, group_size).  At (4, 64) it is
 *                         the layout of Top-K sparse attention (one kept token = one contiguous
 *                         V row); dense decode attention over it runs the CUDA-core kernel
 *                         of the variants.  For the variants it equals FLEXQ_KV_DENSE. */
typedef enum { FLEXQ_KV_DENSE = 0, FLEXQ_KV_TOKEN_MAJOR = 1 } flexq_kv_layout;

/* Static, never-NULL description of a status code (unknown codes included). */
const char *flexq_status_string(int status);

/* Group-wise quantize (reading B): x fp16 [rows][cols] row-major;
 * groups are runs of group_size contiguous elements along cols (for weights,
 * the output-channel axis of the paper's x.w orientation).
 * Per group: min, max; code = RNE(RN32(RN32(RN32(x-min) / RN32(max-min)) * (2^bits - 1)));
 * max == min -> codes 0, scale 0 (reading C).
 *   codes_u8 [rows][cols*bits/8]: each row's codes as a little-endian bit stream, "codes
 *            packed little-endian bit-order within bytes": bit i of element j is
 *            stream bit j*bits + i = bit (j*bits + i) % 8 of byte (j*bits + i) / 8.  For
 *            bits = 4: element 2k in the low nibble of byte k.
 *   meta_h2  [rows][cols/group_size] half2 {scale = f16((max-min)/(2^bits - 1)), min}.
 * Built: bits in {2, 3, 4, 8} x group_size in {32, 64, 128} (P:846's b = 4, g = 64 plus the
 * NEXT-3 variants; other legal values -> FLEXQ_ERR_UNSUPPORTED); rows * cols / group_size
 * < 2^31 (else FLEXQ_ERR_ARG).  rows == 0 or cols == 0 is a no-op. */
flexq_status flexq_quantize(const void *x_f16, int64_t rows, int64_t cols, int bits, int group_size,
                            void *codes_u8, void *meta_h2, void *stream);

/* Inverse of flexq_quantize: out fp16 [rows][cols] =
 * f16_RNE(clamp(fmaf(code, scale, min), -65504, 65504)) (reading R).  Same layouts and
 * built (bits, group_size) set as flexq_quantize. */
flexq_status flexq_dequantize(const void *codes_u8, const void *meta_h2, int64_t rows, int64_t cols,
                              int bits, int group_size, void *out_f16, void *stream);

/* KV cache layout for one layer: a K cache buffer and a V cache buffer of
 * identical size.  Capacity T_cap = prompt_len + gen_len tokens,
 * stored in chunks of 32 tokens per (batch, head); T_stride = T_cap rounded
 * up to a multiple of 32.  With D = head_dim, CB = D/2 code bytes and
 * MB = D/16 metadata bytes per token, one chunk is 18*D bytes:
 *     [codes 32 x CB][meta 32 x MB]
 * and each buffer is u8 [batch][heads][T_stride/32][18*D].  Token t of head
 * (b, h) lives in chunk (b*heads + h)*T_stride/32 + t/32, slot s = t%32.
 * Meta (both caches): 32*CB + s*MB, D/64 half2 {scale, min} (groups of 64
 * along D).  Codes: two codes per byte, column 2i in the low nibble
 * (S:520), and
 *   K: token-major -- byte i of the token's row at s*CB + i;
 *   V: quad-interleaved and swizzled -- byte k of the 32-bit word at
 *      ((s/4)*CB + (i ^ (((s/4) & 3) << 3)))*4 is token 4*(s/4) + k's byte i
 *      (one word holds 4 tokens of a column pair, the shape the P.V integer
 *      matrix product consumes; the XOR spreads the four quads a tensor-core
 *      fragment reads at once over distinct shared-memory banks).
 * The chunks of one head are contiguous, so the attention kernel streams any
 * run of them with one 1-D TMA bulk copy.  Tokens [T_cap, T_stride) are
 * padding the library never writes.
 *
 * Variants: bits in {2, 3, 4, 8} x group_size in {32, 64, 128} other than
 * (4, 64), with head_dim % group_size == 0.  Same 32-token chunks with CB = D*bits/8 code bytes
 * and MB = 4*D/group_size meta bytes per token, chunk = 32*(CB + MB) bytes:
 *     [codes 32 x CB][meta 32 x MB]
 * K and V alike token-major: token s's codes at s*CB as a little-endian bit stream (bit i of
 * column j is stream bit j*bits + i), its D/group_size half2 {scale, min} at 32*CB + s*MB.
 * FLEXQ_KV_TOKEN_MAJOR at (4, 64) is this layout too (V laid out exactly like K); the buffer
 * sizes do not depend on the layout.
 *
 * *cache_bytes (may be NULL) receives the size of ONE buffer (K or V),
 * *token_stride (may be NULL) T_stride.  Supported: head_dim in {64, 128}; (bits, group_size)
 * = (4, 64) or a variant above (other legal values -> FLEXQ_ERR_UNSUPPORTED). */
flexq_status flexq_kv_cache_bytes(int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                  int bits, int group_size, size_t *cache_bytes, int *token_stride);

/* KV update x_K <- Concat(x_K, t.w_K), same for V: quantizes
 * k_new, v_new fp16 [batch][heads][n_new][head_dim] group-wise along head_dim
 * and writes cache tokens [pos, pos + n_new) of every (batch, head)
 * into k_cache / v_cache (layout above).  Prompt fill is pos = 0,
 * n_new = prompt_len; a decode step is n_new = 1.  Touches no other cache
 * position. */
flexq_status flexq_append_kv(const void *k_new_f16, const void *v_new_f16,
                             int batch, int heads, int head_dim, int prompt_len, int gen_len,
                             int pos, int n_new, int bits, int group_size, int kv_layout,
                             void *k_cache, void *v_cache, void *stream);

/* Conversion between the plain quantized KV layout and the cache layout above.  The paper
 * keeps the KV cache "in the quantized format" without fixing a layout; the plain one
 * is flexq_quantize's output for the token rows of each head, four arrays per layer:
 *     k_codes_u8, v_codes_u8  u8    [batch][heads][plain_tokens][head_dim*bits/8]
 *                             (each token row a little-endian bit stream; bits = 4:
 *                              column 2i in the low nibble of byte i)
 *     k_meta_h2, v_meta_h2    half2 [batch][heads][plain_tokens][head_dim/group_size]
 *                             {scale, min} (groups along head_dim)
 * flexq_kv_import copies tokens [t0, t0 + n_tok) of the plain arrays into the same positions
 * of k_cache / v_cache and touches no other cache byte; flexq_kv_export copies those tokens of
 * the caches into the plain arrays and touches nothing else there.  Bytes are moved, never
 * recomputed: import of flexq_quantize's rows gives exactly flexq_append_kv's cache bytes.
 * Requires 0 <= t0, t0 + n_tok <= min(plain_tokens, prompt_len + gen_len) (else
 * FLEXQ_ERR_ARG); n_tok == 0 is a no-op.  Same (bits, group_size, head_dim) support as the
 * cache; every pointer 16-byte aligned. */
flexq_status flexq_kv_import(const void *k_codes_u8, const void *k_meta_h2, const void *v_codes_u8,
                             const void *v_meta_h2, int batch, int heads, int head_dim, int prompt_len,
                             int gen_len, int plain_tokens, int t0, int n_tok, int bits, int group_size,
                             int kv_layout, void *k_cache, void *v_cache, void *stream);
flexq_status flexq_kv_export(const void *k_cache, const void *v_cache, int batch, int heads, int head_dim,
                             int prompt_len, int gen_len, int plain_tokens, int t0, int n_tok, int bits,
                             int group_size, int kv_layout, void *k_codes_u8, void *k_meta_h2, void *v_codes_u8,
                             void *v_meta_h2, void *stream);

/* Workspace bytes flexq_decode_attention needs for these dimensions (0 on bad
 * arguments).  Layout (b = 4, g = 64): 2 KB of scheduler counters (item tickets), 4 B per
 * (batch, head) of merge tickets, then per (batch, head) 32 slots of split-K partials (D
 * floats each) and 32 (m, l) float pairs; variants: 256 B (unused), then (D + 2) floats per
 * (batch, head, 128-token tile) of split-K partials.  The workspace must be zero-filled
 * ONCE after allocation; every call restores the counters and tickets to
 * zero before it completes (the partials are scratch), so one buffer serves
 * any number of stream-ordered calls (not concurrent ones). */
size_t flexq_decode_attention_workspace_size(int batch, int heads, int head_dim, int prompt_len,
                                             int gen_len, int bits, int group_size, int kv_layout);

/* Decode-step attention over the compressed cache (reading K):
 *   out fp16 [batch][heads][head_dim] =
 *     softmax(q . K^[0:cur_len]^T / sqrt(head_dim)) . V^[0:cur_len]
 * with K^, V^ = fmaf(code, scale, min) in fp32, never rounded to fp16 (reading
 * M); q fp16 [batch][heads][head_dim].  Cache layout as above; tokens at
 * positions >= cur_len do not influence the result (the kernel may stream the
 * rest of the last 32-token chunk into shared memory and discard it).  Accuracy: |out - exact| <=
 * max(2e-3, 1e-2 |exact|) per element (reading Q).  (4, 64) runs the tensor-core kernel
 * (cur_len <= 17408, else FLEXQ_ERR_UNSUPPORTED); the variants a CUDA-core split-K kernel
 * (+ a combine launch when a head is split). */
flexq_status flexq_decode_attention(const void *q_f16, const void *k_cache, const void *v_cache,
                                    int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                    int cur_len, int bits, int group_size, int kv_layout, void *out_f16,
                                    void *workspace, size_t workspace_bytes, void *stream);

/* One decode step of one layer in a single launch:
 * exactly flexq_append_kv(k_new, v_new, pos = cur_len - 1, n_new = 1)
 * followed by flexq_decode_attention(q, ..., cur_len) -- the new token is
 * quantized first and attends to itself (reading L).
 * k_new_f16, v_new_f16: fp16 [batch][heads][head_dim] (the token's K and V).
 * The cache bytes written for position cur_len - 1 are identical to those of
 * flexq_append_kv; nothing else in the cache is touched; the output
 * satisfies flexq_decode_attention's accuracy bound.  Arguments, workspace
 * and errors as for flexq_decode_attention (+ FLEXQ_ERR_NULL / _ALIGN for
 * k_new / v_new).  Variants: the append kernel, then the attention kernel (two launches). */
flexq_status flexq_append_decode_attention(const void *q_f16, const void *k_new_f16, const void *v_new_f16,
                                           void *k_cache, void *v_cache, int batch, int heads,
                                           int head_dim, int prompt_len, int gen_len, int cur_len, int bits,
                                           int group_size, int kv_layout, void *out_f16, void *workspace,
                                           size_t workspace_bytes, void *stream);

/* Workspace bytes flexq_decode_attention_topk needs (0 on bad arguments or a configuration
 * Top-K does not build): 2 KB of scheduler counters, then the kept lists -- an int32 token
 * index and an fp32 weight per (batch, head, kept token), sized for keep <= prompt_len +
 * gen_len (8 B per cached token position: 60 MB at OPT-175B's 144 x 96 heads x 544 tokens).
 * Zero-filled once after allocation; every call leaves the counters zero again. */
size_t flexq_decode_attention_topk_workspace_size(int batch, int heads, int head_dim, int prompt_len,
                                                  int gen_len, int bits, int group_size, int kv_layout);

/* Top-K sparse decode attention, FlexGen's "4-bit-S":
 * scores s_t = q . K^_t / sqrt(head_dim) for t in [0, cur_len); the `keep`
 * highest scores are kept (equal scores: lower token index first); out fp16
 * [batch][heads][head_dim] = sum over kept t of p_t V^_t, softmax
 * renormalised over the kept set.  Only the kept V rows are read
 * (P:856).  The paper keeps the top 10%: keep = ceil(0.1 * cur_len).
 * sel_i32 (optional, may be NULL): int32 [batch][heads][keep] receives the
 * kept token indices in ascending order.  Workspace: >=
 * flexq_decode_attention_topk_workspace_size(...) bytes.  Two launches (select, then gather
 * of the kept V rows).  Both layouts are read; FLEXQ_KV_TOKEN_MAJOR makes a kept token one
 * contiguous V row (the dense layout spreads it over its 4-token quad row).  Supported:
 * bits = 4, group_size = 64, cur_len <= 1152 (else FLEXQ_ERR_UNSUPPORTED);
 * 1 <= keep <= cur_len (else FLEXQ_ERR_ARG). */
flexq_status flexq_decode_attention_topk(const void *q_f16, const void *k_cache, const void *v_cache,
                                         int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                         int cur_len, int keep, int bits, int group_size, int kv_layout,
                                         void *out_f16, void *sel_i32, void *workspace, size_t workspace_bytes,
                                         void *stream);

/* Decode-step linear layer over a group-wise 4-bit weight:
 *   y[m][n] = sum_k x[m][k] * w^[k][n],   y = t . w,
 * w in R^{h1 x h2} row-major [k][n], quantized by flexq_quantize with groups of group_size
 * contiguous elements along the output channel n (reading J), and "converted back to
 * FP16 before computation" inside the kernel: w^ = min(RN16(c*scale + min),
 * 65504), one fp16 FMA -- equal to flexq_dequantize's output except where RN32 of the exact
 * value lands on an fp16 tie (reading G2; at most 1 fp16 ulp).  Products are
 * exact and accumulate in fp32 on the tensor cores; y is rounded once to fp16.
 *
 * Built: bits = 4, group_size = 64, n % 256 == 0, k % 64 == 0 (else FLEXQ_ERR_UNSUPPORTED).
 *
 * flexq_pack_weight: one-time re-layout (no arithmetic) of flexq_quantize's output for a
 * [k][n] weight -- codes_u8 u8 [k][n/2], meta_h2 half2 [k][n/group_size] -- into
 * flexq_gemm_panel_bytes(k, n) bytes of "panels" (one 9216-byte panel per 256 columns x 64 k:
 * codes column-major along k, then that block's (scale, min) pairs; after all panels, one
 * 16-byte flag per panel whose first word is 1 when some code of the panel can reconstruct above
 * 65504 -- the kernel then applies reading R's clamp), the operand format of
 * flexq_dequant_gemm: the bytes of codes + meta plus 16 per panel.  Writes only `panels`.
 *
 * flexq_dequant_gemm:
 *   x_f16   fp16 [m][k] row-major (m = decode batch b, k = in features); any m >= 1
 *           (rows are processed 160 at a time)
 *   panels  flexq_pack_weight's output for the [k][n] weight
 *   y_f16   fp16 [m][n] row-major; every element is written.
 *   m == 0 or n == 0: FLEXQ_OK, nothing written; k == 0: FLEXQ_ERR_UNSUPPORTED.
 *   workspace: >= flexq_dequant_gemm_workspace_size(...) bytes, 16-byte aligned, ZEROED by
 *   the caller before its first use.  It holds per-tile tickets (first n/256 * 4 bytes,
 *   rounded up to 256) and split-k fp32 partial sums (scratch); every call leaves the
 *   tickets zero again, so the workspace may be reused across calls on one stream but not
 *   shared by calls that can run concurrently. */
size_t flexq_gemm_panel_bytes(int64_t k, int64_t n, int bits, int group_size);
flexq_status flexq_pack_weight(const void *codes_u8, const void *meta_h2, int64_t k, int64_t n, int bits,
                               int group_size, void *panels, void *stream);
size_t flexq_dequant_gemm_workspace_size(int64_t m, int64_t k, int64_t n, int bits, int group_size);
flexq_status flexq_dequant_gemm(const void *x_f16, const void *panels, int64_t m, int64_t k, int64_t n, int bits,
                                int group_size, void *y_f16, void *workspace, size_t workspace_bytes,
                                void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FLEXQ_H */

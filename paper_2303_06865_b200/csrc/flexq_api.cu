// flexq_api.cu -- the C ABI declared in include/flexq.h: host-side argument
// validation (no CUDA call before it passes), then the kernel launchers.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flexq.h"
#include "flexq_internal.h"

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Shared checks for the quantizer configuration (b = 4, g = 64).
flexq_status check_bits_group(int bits, int group_size) {
    if (bits < 1 || bits > 8 || group_size < 1) return FLEXQ_ERR_ARG;
    if (bits != flexq::kBits || group_size != flexq::kGroup) return FLEXQ_ERR_UNSUPPORTED;
    return FLEXQ_OK;
}

flexq_status check_kv_dims(int batch, int heads, int head_dim, int prompt_len, int gen_len, int bits,
                           int group_size) {
    if (batch < 1 || heads < 1 || head_dim < 1 || prompt_len < 0 || gen_len < 0 ||
        int64_t(prompt_len) + gen_len < 1 || int64_t(prompt_len) + gen_len > INT32_MAX - flexq::kChunk)
        return FLEXQ_ERR_ARG;
    if (bits < 1 || bits > 8 || group_size < 1) return FLEXQ_ERR_ARG;
    if (!flexq::quant_variant_built(bits, group_size)) return FLEXQ_ERR_UNSUPPORTED;
    if (head_dim != 64 && head_dim != 128) return FLEXQ_ERR_UNSUPPORTED;
    if (head_dim % group_size != 0) return FLEXQ_ERR_UNSUPPORTED;
    return FLEXQ_OK;
}

// b = 4, g = 64 in the dense layout runs the tensor-core kernels; the other built (b, g),
// and (4, 64) in the token-major layout, the CUDA-core variant kernels over token-major rows
bool is_variant(int bits, int group_size) { return bits != flexq::kBits || group_size != flexq::kGroup; }
bool token_major(int bits, int group_size, int kv_layout) {
    return is_variant(bits, group_size) || kv_layout == FLEXQ_KV_TOKEN_MAJOR;
}
bool layout_ok(int kv_layout) { return kv_layout == FLEXQ_KV_DENSE || kv_layout == FLEXQ_KV_TOKEN_MAJOR; }

size_t attn_ws_bytes(int batch, int heads, int head_dim, int t_cap, int bits, int group_size, int kv_layout) {
    const size_t var = flexq::attention_variant_workspace_bytes(batch, heads, head_dim, t_cap);
    const size_t dense = flexq::attention_workspace_bytes(batch, heads, head_dim, t_cap);
    if (is_variant(bits, group_size)) return var;
    // (4, 64) token-major: the variant attention kernel, or Top-K (the dense kernel's workspace)
    return kv_layout == FLEXQ_KV_TOKEN_MAJOR ? (var > dense ? var : dense) : dense;
}

flexq_status from_cuda(cudaError_t e) { return e == cudaSuccess ? FLEXQ_OK : FLEXQ_ERR_CUDA; }

}  // namespace

extern "C" {

int flexq_abi_version(void) { return FLEXQ_ABI_VERSION; }

const char* flexq_status_string(int s) {
    switch (s) {
        case FLEXQ_OK: return "ok";
        case FLEXQ_ERR_NULL: return "null pointer";
        case FLEXQ_ERR_ARG: return "argument out of range";
        case FLEXQ_ERR_ALIGN: return "pointer not 16-byte aligned";
        case FLEXQ_ERR_UNSUPPORTED: return "unsupported configuration (bits/group/head_dim/cols)";
        case FLEXQ_ERR_WORKSPACE: return "workspace missing or too small";
        case FLEXQ_ERR_CUDA: return "CUDA launch failed";
        default: return "unknown status";
    }
}

// Quantize / dequantize also build the NEXT-3 variants: b in {2, 3, 8}, g in {32, 128}.
static flexq_status check_quant_variant(int bits, int group_size) {
    if (bits < 1 || bits > 8 || group_size < 1) return FLEXQ_ERR_ARG;
    if (!flexq::quant_variant_built(bits, group_size)) return FLEXQ_ERR_UNSUPPORTED;
    return FLEXQ_OK;
}

flexq_status flexq_quantize(const void* x_f16, int64_t rows, int64_t cols, int bits, int group_size,
                            void* codes_u8, void* meta_h2, void* stream) {
    if (rows < 0 || cols < 0) return FLEXQ_ERR_ARG;
    flexq_status s = check_quant_variant(bits, group_size);
    if (s != FLEXQ_OK) return s;
    if (cols % group_size != 0) return FLEXQ_ERR_UNSUPPORTED;
    if (rows == 0 || cols == 0) return FLEXQ_OK;
    if (rows > (int64_t(1) << 31) / (cols / group_size)) return FLEXQ_ERR_ARG;   // < 2^31 groups
    if (!x_f16 || !codes_u8 || !meta_h2) return FLEXQ_ERR_NULL;
    if (!aligned16(x_f16) || !aligned16(codes_u8) || !aligned16(meta_h2)) return FLEXQ_ERR_ALIGN;
    return from_cuda(flexq::launch_quantize(x_f16, rows, cols, bits, group_size, codes_u8, meta_h2,
                                            static_cast<cudaStream_t>(stream)));
}

flexq_status flexq_dequantize(const void* codes_u8, const void* meta_h2, int64_t rows, int64_t cols,
                              int bits, int group_size, void* out_f16, void* stream) {
    if (rows < 0 || cols < 0) return FLEXQ_ERR_ARG;
    flexq_status s = check_quant_variant(bits, group_size);
    if (s != FLEXQ_OK) return s;
    if (cols % group_size != 0) return FLEXQ_ERR_UNSUPPORTED;
    if (rows == 0 || cols == 0) return FLEXQ_OK;
    if (rows > (int64_t(1) << 31) / (cols / group_size)) return FLEXQ_ERR_ARG;
    if (!codes_u8 || !meta_h2 || !out_f16) return FLEXQ_ERR_NULL;
    if (!aligned16(codes_u8) || !aligned16(meta_h2) || !aligned16(out_f16)) return FLEXQ_ERR_ALIGN;
    return from_cuda(flexq::launch_dequantize(codes_u8, meta_h2, rows, cols, bits, group_size, out_f16,
                                              static_cast<cudaStream_t>(stream)));
}

flexq_status flexq_kv_cache_bytes(int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                  int bits, int group_size, size_t* cache_bytes, int* token_stride) {
    // bytes of ONE cache buffer (K or V)
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s != FLEXQ_OK) return s;
    const int64_t stride = flexq::kv_token_stride(int64_t(prompt_len) + gen_len);
    if (cache_bytes)
        *cache_bytes = size_t(batch) * heads * size_t(stride / flexq::kChunk) * size_t(flexq::kv_chunk_bytes(head_dim, bits, group_size));
    if (token_stride) *token_stride = int(stride);
    return FLEXQ_OK;
}

flexq_status flexq_append_kv(const void* k_new_f16, const void* v_new_f16, int batch, int heads,
                             int head_dim, int prompt_len, int gen_len, int pos, int n_new, int bits,
                             int group_size, int kv_layout, void* k_cache, void* v_cache, void* stream) {
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s == FLEXQ_ERR_ARG || !layout_ok(kv_layout)) return FLEXQ_ERR_ARG;
    const int64_t t_cap = int64_t(prompt_len) + gen_len;
    if (pos < 0 || n_new < 1 || int64_t(pos) + n_new > t_cap) return FLEXQ_ERR_ARG;
    if (s != FLEXQ_OK) return s;
    if (!k_new_f16 || !v_new_f16 || !k_cache || !v_cache) return FLEXQ_ERR_NULL;
    if (!aligned16(k_new_f16) || !aligned16(v_new_f16) || !aligned16(k_cache) || !aligned16(v_cache))
        return FLEXQ_ERR_ALIGN;
    const int64_t rows = int64_t(batch) * heads * n_new;
    if (rows * (head_dim / group_size) >= (int64_t(1) << 31)) return FLEXQ_ERR_ARG;   // < 2^31 groups
    const flexq::KvDst d{n_new, pos, flexq::kv_token_stride(t_cap) / flexq::kChunk};
    return from_cuda(flexq::launch_append_kv(k_new_f16, v_new_f16, rows, head_dim, bits, group_size, k_cache, v_cache, d,
                                             static_cast<cudaStream_t>(stream),
                                             kv_layout == FLEXQ_KV_TOKEN_MAJOR));
}

size_t flexq_decode_attention_workspace_size(int batch, int heads, int head_dim, int prompt_len,
                                             int gen_len, int bits, int group_size, int kv_layout) {
    if (check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size) != FLEXQ_OK) return 0;
    if (!layout_ok(kv_layout)) return 0;
    return attn_ws_bytes(batch, heads, head_dim, prompt_len + gen_len, bits, group_size, kv_layout);
}

flexq_status flexq_decode_attention(const void* q_f16, const void* k_cache, const void* v_cache, int batch,
                                    int heads,
                                    int head_dim, int prompt_len, int gen_len, int cur_len, int bits,
                                    int group_size, int kv_layout, void* out_f16, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s == FLEXQ_ERR_ARG || !layout_ok(kv_layout)) return FLEXQ_ERR_ARG;
    const int t_cap = prompt_len + gen_len;
    if (cur_len < 1 || cur_len > t_cap) return FLEXQ_ERR_ARG;
    if (s != FLEXQ_OK) return s;
    if (!q_f16 || !k_cache || !v_cache || !out_f16) return FLEXQ_ERR_NULL;
    if (!aligned16(q_f16) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out_f16))
        return FLEXQ_ERR_ALIGN;
    if (!workspace || workspace_bytes < attn_ws_bytes(batch, heads, head_dim, t_cap, bits, group_size, kv_layout))
        return FLEXQ_ERR_WORKSPACE;
    if (!aligned16(workspace)) return FLEXQ_ERR_ALIGN;
    flexq::AttnArgs a{q_f16, k_cache, v_cache, out_f16, workspace, batch, heads, head_dim,
                      int(flexq::kv_token_stride(t_cap) / flexq::kChunk), cur_len, t_cap};
    if (token_major(bits, group_size, kv_layout))
        return from_cuda(flexq::launch_decode_attention_variant(a, bits, group_size, static_cast<cudaStream_t>(stream)));
    if (cur_len > flexq::kDenseMaxTokens) return FLEXQ_ERR_UNSUPPORTED;
    return from_cuda(flexq::launch_decode_attention(a, static_cast<cudaStream_t>(stream)));
}

flexq_status flexq_append_decode_attention(const void* q_f16, const void* k_new_f16, const void* v_new_f16,
                                           void* k_cache, void* v_cache, int batch, int heads, int head_dim,
                                           int prompt_len, int gen_len, int cur_len, int bits, int group_size,
                                           int kv_layout, void* out_f16, void* workspace, size_t workspace_bytes,
                                           void* stream) {
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s == FLEXQ_ERR_ARG || !layout_ok(kv_layout)) return FLEXQ_ERR_ARG;
    const int t_cap = prompt_len + gen_len;
    if (cur_len < 1 || cur_len > t_cap) return FLEXQ_ERR_ARG;
    if (s != FLEXQ_OK) return s;
    if (!q_f16 || !k_new_f16 || !v_new_f16 || !k_cache || !v_cache || !out_f16) return FLEXQ_ERR_NULL;
    if (!aligned16(q_f16) || !aligned16(k_new_f16) || !aligned16(v_new_f16) || !aligned16(k_cache) ||
        !aligned16(v_cache) || !aligned16(out_f16))
        return FLEXQ_ERR_ALIGN;
    if (!workspace || workspace_bytes < attn_ws_bytes(batch, heads, head_dim, t_cap, bits, group_size, kv_layout))
        return FLEXQ_ERR_WORKSPACE;
    if (!aligned16(workspace)) return FLEXQ_ERR_ALIGN;
    flexq::AttnArgs a{q_f16, k_cache, v_cache, out_f16, workspace, batch, heads, head_dim,
                      int(flexq::kv_token_stride(t_cap) / flexq::kChunk), cur_len, t_cap, k_new_f16, v_new_f16};
    if (token_major(bits, group_size, kv_layout)) {   // token-major rows: the append kernel, then the attention kernel
        const flexq::KvDst d{1, cur_len - 1, a.chunks};
        cudaError_t e = flexq::launch_append_kv(k_new_f16, v_new_f16, int64_t(batch) * heads, head_dim, bits,
                                                group_size, k_cache, v_cache, d, static_cast<cudaStream_t>(stream),
                                                kv_layout == FLEXQ_KV_TOKEN_MAJOR);
        if (e != cudaSuccess) return FLEXQ_ERR_CUDA;
        a.k_new = a.v_new = nullptr;
        return from_cuda(flexq::launch_decode_attention_variant(a, bits, group_size, static_cast<cudaStream_t>(stream)));
    }
    if (cur_len > flexq::kDenseMaxTokens) return FLEXQ_ERR_UNSUPPORTED;
    return from_cuda(flexq::launch_decode_attention(a, static_cast<cudaStream_t>(stream)));
}

size_t flexq_decode_attention_topk_workspace_size(int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                                  int bits, int group_size, int kv_layout) {
    if (check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size) != FLEXQ_OK) return 0;
    if (!layout_ok(kv_layout) || is_variant(bits, group_size)) return 0;
    return flexq::topk_workspace_bytes(batch, heads, prompt_len + gen_len);
}

flexq_status flexq_decode_attention_topk(const void* q_f16, const void* k_cache, const void* v_cache,
                                         int batch, int heads, int head_dim, int prompt_len, int gen_len,
                                         int cur_len, int keep, int bits, int group_size, int kv_layout,
                                         void* out_f16, void* sel_i32, void* workspace, size_t workspace_bytes,
                                         void* stream) {
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s == FLEXQ_ERR_ARG || !layout_ok(kv_layout)) return FLEXQ_ERR_ARG;
    const int t_cap = prompt_len + gen_len;
    if (cur_len < 1 || cur_len > t_cap || keep < 1 || keep > cur_len) return FLEXQ_ERR_ARG;
    if (s != FLEXQ_OK) return s;
    if (is_variant(bits, group_size)) return FLEXQ_ERR_UNSUPPORTED;   // Top-K: b = 4, g = 64 only
    if (cur_len > flexq::kTopkMaxTokens) return FLEXQ_ERR_UNSUPPORTED;
    if (!q_f16 || !k_cache || !v_cache || !out_f16) return FLEXQ_ERR_NULL;
    if (!aligned16(q_f16) || !aligned16(k_cache) || !aligned16(v_cache) || !aligned16(out_f16) ||
        (sel_i32 && !aligned16(sel_i32)))
        return FLEXQ_ERR_ALIGN;
    if (!workspace || workspace_bytes < flexq::topk_workspace_bytes(batch, heads, t_cap)) return FLEXQ_ERR_WORKSPACE;
    if (!aligned16(workspace)) return FLEXQ_ERR_ALIGN;
    flexq::TopkArgs a{q_f16, k_cache, v_cache, out_f16, sel_i32, workspace, batch, heads, head_dim,
                      int(flexq::kv_token_stride(t_cap) / flexq::kChunk), cur_len, keep,
                      kv_layout == FLEXQ_KV_TOKEN_MAJOR ? 1 : 0};
    return from_cuda(flexq::launch_decode_attention_topk(a, static_cast<cudaStream_t>(stream)));
}

static flexq_status kv_interop(bool import_, void* k_codes, void* k_meta, void* v_codes, void* v_meta, int batch,
                               int heads, int head_dim, int prompt_len, int gen_len, int plain_tokens, int t0,
                               int n_tok, int bits, int group_size, int kv_layout, void* k_cache, void* v_cache,
                               void* stream) {
    flexq_status s = check_kv_dims(batch, heads, head_dim, prompt_len, gen_len, bits, group_size);
    if (s == FLEXQ_ERR_ARG || !layout_ok(kv_layout)) return FLEXQ_ERR_ARG;
    const int64_t t_cap = int64_t(prompt_len) + gen_len;
    if (plain_tokens < 1 || t0 < 0 || n_tok < 0 || int64_t(t0) + n_tok > t_cap || t0 + n_tok > plain_tokens)
        return FLEXQ_ERR_ARG;
    if (s != FLEXQ_OK) return s;
    if (n_tok == 0) return FLEXQ_OK;
    if (!k_codes || !k_meta || !v_codes || !v_meta || !k_cache || !v_cache) return FLEXQ_ERR_NULL;
    if (!aligned16(k_codes) || !aligned16(k_meta) || !aligned16(v_codes) || !aligned16(v_meta) ||
        !aligned16(k_cache) || !aligned16(v_cache))
        return FLEXQ_ERR_ALIGN;
    flexq::KvInterop x{k_codes, k_meta, v_codes, v_meta, k_cache, v_cache, int64_t(batch) * heads,
                       flexq::kv_token_stride(t_cap) / flexq::kChunk, plain_tokens, t0, n_tok, head_dim, bits,
                       group_size, kv_layout == FLEXQ_KV_TOKEN_MAJOR ? 1 : 0};
    return from_cuda(flexq::launch_kv_interop(import_, x, static_cast<cudaStream_t>(stream)));
}

flexq_status flexq_kv_import(const void* k_codes_u8, const void* k_meta_h2, const void* v_codes_u8,
                             const void* v_meta_h2, int batch, int heads, int head_dim, int prompt_len, int gen_len,
                             int plain_tokens, int t0, int n_tok, int bits, int group_size, int kv_layout,
                             void* k_cache, void* v_cache, void* stream) {
    return kv_interop(true, const_cast<void*>(k_codes_u8), const_cast<void*>(k_meta_h2), const_cast<void*>(v_codes_u8),
                      const_cast<void*>(v_meta_h2), batch, heads, head_dim, prompt_len, gen_len, plain_tokens, t0,
                      n_tok, bits, group_size, kv_layout, k_cache, v_cache, stream);
}

flexq_status flexq_kv_export(const void* k_cache, const void* v_cache, int batch, int heads, int head_dim,
                             int prompt_len, int gen_len, int plain_tokens, int t0, int n_tok, int bits,
                             int group_size, int kv_layout, void* k_codes_u8, void* k_meta_h2, void* v_codes_u8,
                             void* v_meta_h2, void* stream) {
    return kv_interop(false, k_codes_u8, k_meta_h2, v_codes_u8, v_meta_h2, batch, heads, head_dim, prompt_len,
                      gen_len, plain_tokens, t0, n_tok, bits, group_size, kv_layout, const_cast<void*>(k_cache),
                      const_cast<void*>(v_cache), stream);
}

// Shared checks for the decode linear layer's weight shape (NEXT-2).
static flexq_status check_gemm_weight(int64_t k, int64_t n, int bits, int group_size) {
    if (k < 0 || n < 0) return FLEXQ_ERR_ARG;
    flexq_status s = check_bits_group(bits, group_size);
    if (s != FLEXQ_OK) return s;
    if (n % group_size != 0) return FLEXQ_ERR_UNSUPPORTED;
    if (k == 0 || n == 0) return FLEXQ_OK;
    if (n % flexq::kGemmTileN != 0 || k % flexq::kGemmTileK != 0) return FLEXQ_ERR_UNSUPPORTED;
    if (k > (int64_t(1) << 30) || n > (int64_t(1) << 30)) return FLEXQ_ERR_ARG;
    return FLEXQ_OK;
}

size_t flexq_gemm_panel_bytes(int64_t k, int64_t n, int bits, int group_size) {
    if (check_gemm_weight(k, n, bits, group_size) != FLEXQ_OK) return 0;
    return flexq::gemm_panel_bytes(k, n);
}

flexq_status flexq_pack_weight(const void* codes_u8, const void* meta_h2, int64_t k, int64_t n, int bits,
                               int group_size, void* panels, void* stream) {
    flexq_status s = check_gemm_weight(k, n, bits, group_size);
    if (s != FLEXQ_OK) return s;
    if (k == 0 || n == 0) return FLEXQ_OK;
    if (!codes_u8 || !meta_h2 || !panels) return FLEXQ_ERR_NULL;
    if (!aligned16(codes_u8) || !aligned16(meta_h2) || !aligned16(panels)) return FLEXQ_ERR_ALIGN;
    return from_cuda(flexq::launch_pack_weight(codes_u8, meta_h2, k, n, panels, static_cast<cudaStream_t>(stream)));
}

size_t flexq_dequant_gemm_workspace_size(int64_t m, int64_t k, int64_t n, int bits, int group_size) {
    if (m < 1 || k < 1 || n < 1 || check_gemm_weight(k, n, bits, group_size) != FLEXQ_OK) return 0;
    return flexq::dequant_gemm_workspace_bytes(m, k, n);
}

flexq_status flexq_dequant_gemm(const void* x_f16, const void* panels, int64_t m, int64_t k, int64_t n, int bits,
                                int group_size, void* y_f16, void* workspace, size_t workspace_bytes, void* stream) {
    if (m < 0) return FLEXQ_ERR_ARG;
    flexq_status s = check_gemm_weight(k, n, bits, group_size);
    if (s != FLEXQ_OK) return s;
    if (m == 0 || n == 0) return FLEXQ_OK;
    if (k == 0) return FLEXQ_ERR_UNSUPPORTED;     // an empty sum would need a zero fill, not built
    if (m * n >= (int64_t(1) << 40)) return FLEXQ_ERR_ARG;
    if (!x_f16 || !panels || !y_f16) return FLEXQ_ERR_NULL;
    if (!aligned16(x_f16) || !aligned16(panels) || !aligned16(y_f16)) return FLEXQ_ERR_ALIGN;
    if (!workspace || workspace_bytes < flexq::dequant_gemm_workspace_bytes(m, k, n)) return FLEXQ_ERR_WORKSPACE;
    if (!aligned16(workspace)) return FLEXQ_ERR_ALIGN;
    return from_cuda(flexq::launch_dequant_gemm(x_f16, panels, m, k, n, y_f16, workspace,
                                                static_cast<cudaStream_t>(stream)));
}

}  // extern "C"

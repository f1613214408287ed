// flexq_internal.h -- launchers shared between the C-ABI layer and the kernels.
// Internal to paper_2303_06865_b200/csrc (the oracle shares nothing with it).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace flexq {

// Fixed by the paper's configuration: 4-bit codes, groups of 64.
constexpr int kBits = 4;
constexpr int kGroup = 64;

// Token stride of the KV cache: capacity rounded up to a multiple of 8 (include/flexq.h).
inline int64_t kv_token_stride(int64_t t_cap) { return (t_cap + 7) / 8 * 8; }

// Row remapping for the quantizer: src row r -> dst row
//   (r / n_new) * t_stride + pos + r % n_new   (KV append)
// or identity when n_new == 0 (plain weight / tensor quantize).
struct RowMap {
    int64_t n_new;   // 0 = identity
    int64_t t_cap;   // token stride of the cache
    int64_t pos;
};

cudaError_t launch_quantize(const void* x, int64_t rows, int64_t cols, void* codes, void* meta,
                            const void* x2, void* codes2, void* meta2, RowMap map,
                            cudaStream_t stream);

cudaError_t launch_dequantize(const void* codes, const void* meta, int64_t rows, int64_t cols,
                              void* out, cudaStream_t stream);

struct AttnArgs {
    const void* q;
    const void* k_codes;
    const void* k_meta;
    const void* v_codes;
    const void* v_meta;
    void* out;
    void* workspace;
    int batch, heads, head_dim, t_stride, cur_len;
};

size_t attention_workspace_bytes(int batch, int heads, int head_dim, int t_cap);
cudaError_t launch_decode_attention(const AttnArgs& a, cudaStream_t stream);

}  // namespace flexq

// flexq_internal.h -- launchers shared between the C-ABI layer and the kernels.
// Internal to paper_2303_06865_b200/csrc (the oracle shares nothing with it).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace flexq {

// Per-device launch facts (device_info.cu), computed once per device under a lock.
constexpr int kMaxDevices = 64;
int current_device();
int device_sm_count();

// Fixed by the paper's configuration: 4-bit codes, groups of 64.
constexpr int kBits = 4;
constexpr int kGroup = 64;

// KV cache layout (include/flexq.h): K and V caches each hold, per (batch,
// head), a run of chunks of kChunk tokens; chunk = [codes kChunk x D/2][meta kChunk x D/16].
constexpr int kChunk = 32;
inline int64_t kv_token_stride(int64_t t_cap) { return (t_cap + kChunk - 1) / kChunk * kChunk; }
inline int64_t kv_chunk_bytes(int64_t d, int bits = kBits, int group = kGroup) {   // 18 d at b = 4, g = 64
    return int64_t(kChunk) * (d * bits / 8 + 4 * d / group);
}

// Destination of a KV append: source rows are (bh, t) with t in [0, n_new),
// written at token pos + t of head bh.
struct KvDst {
    int64_t n_new;
    int64_t pos;
    int64_t chunks;   // chunks per (batch, head) = token stride / kChunk
};

// bits in {2, 3, 4, 8}, group in {32, 64, 128} (b = 4, g = 64 is the tuned kernel; the others
// are NEXT-3 variants).  Codes are a little-endian bit stream per row.
inline bool quant_variant_built(int bits, int group) {
    return (bits == 2 || bits == 3 || bits == 4 || bits == 8) && (group == 32 || group == 64 || group == 128);
}
cudaError_t launch_quantize(const void* x, int64_t rows, int64_t cols, int bits, int group, void* codes, void* meta,
                            cudaStream_t stream);
// v_tm: the (4, 64) cache's V rows token-major (FLEXQ_KV_TOKEN_MAJOR) instead of quad-interleaved
cudaError_t launch_append_kv(const void* k, const void* v, int64_t rows, int head_dim, int bits, int group,
                             void* k_cache, void* v_cache, KvDst dst, cudaStream_t stream, bool v_tm = false);
cudaError_t launch_dequantize(const void* codes, const void* meta, int64_t rows, int64_t cols, int bits, int group,
                              void* out, cudaStream_t stream);

// Plain quantized KV layout <-> chunked cache (kv_interop.cu): byte moves only.
struct KvInterop {
    void* k_codes;        // plain u8 [rows][plain_tokens][D*bits/8]
    void* k_meta;         // plain half2 [rows][plain_tokens][D/group]
    void* v_codes;
    void* v_meta;
    void* k_cache;        // chunked caches (include/flexq.h)
    void* v_cache;
    int64_t rows;         // batch * heads
    int64_t chunks;       // chunks per (b, h)
    int plain_tokens, t0, n, head_dim, bits, group;
    int v_tm = 0;         // 1: the (4, 64) cache's V rows are token-major (FLEXQ_KV_TOKEN_MAJOR)
};
cudaError_t launch_kv_interop(bool import_, const KvInterop& x, cudaStream_t stream);

struct AttnArgs {
    const void* q;
    const void* k_cache;
    const void* v_cache;
    void* out;
    void* workspace;
    int batch, heads, head_dim, chunks, cur_len, t_cap;
    const void* k_new = nullptr;   // fused append of token cur_len - 1 (NEXT-3), or nullptr
    const void* v_new = nullptr;
};

size_t attention_workspace_bytes(int batch, int heads, int head_dim, int t_cap);
// Longest context of the (4, 64) tensor-core kernel: 16 pieces of its 1088-token score buffer.
constexpr int kDenseMaxTokens = 16 * 1088;
cudaError_t launch_decode_attention(const AttnArgs& a, cudaStream_t stream);

// Decode attention over the (b, g) variant caches (NEXT-3; decode_attention_variants.cu):
// token-major bit-stream rows for K and V, CUDA-core arithmetic, split-K over 128-token tiles.
constexpr int kVarTile = 128;
size_t attention_variant_workspace_bytes(int batch, int heads, int head_dim, int t_cap);
cudaError_t launch_decode_attention_variant(const AttnArgs& a, int bits, int group, cudaStream_t stream);

// Top-K sparse attention, two launches: a select kernel (one warp per (b, h), so
// the context is bounded by the per-warp score buffer) writes each head's kept list, a gather
// kernel reads only the kept V rows.
constexpr int kTopkMaxTokens = 1152;
struct TopkArgs {
    const void* q;
    const void* k_cache;
    const void* v_cache;
    void* out;
    void* sel;          // optional int32 [batch*heads][keep]
    void* workspace;    // topk_workspace_bytes: 2 KB of scheduler counters, then the kept lists
    int batch, heads, head_dim, chunks, cur_len, keep;
    int v_tm = 0;       // 1: V rows token-major (FLEXQ_KV_TOKEN_MAJOR): one contiguous row per kept token
};
size_t topk_workspace_bytes(int batch, int heads, int t_cap);
cudaError_t launch_decode_attention_topk(const TopkArgs& a, cudaStream_t stream);

// Decode linear layer over a 4-bit weight (NEXT-2, dequant_gemm.cu): y [M][N] = x [M][K] . w^ [K][N].
// The quantized weight is re-laid out once into panels of 256 columns x 64 k (9 KB each);
// rows are processed in chunks of kGemmMaxRows (the MMA N dimension); N % 256 == 0, K % 64 == 0.
constexpr int kGemmMaxRows = 160;
constexpr int kGemmTileN = 256;
constexpr int kGemmTileK = 64;
constexpr int kGemmPanelBytes = kGemmTileN * kGemmTileK / 2 + 4 * 32 * 8 + 16;   // 9232: codes, meta, flag
constexpr int kGemmMaxGrid = 160;   // persistent CTAs (one per SM, B200: 148)
size_t gemm_panel_bytes(int64_t k, int64_t n);
cudaError_t launch_pack_weight(const void* codes, const void* meta, int64_t k, int64_t n, void* panels,
                               cudaStream_t stream);
size_t dequant_gemm_workspace_bytes(int64_t m, int64_t k, int64_t n);
cudaError_t launch_dequant_gemm(const void* x, const void* panels, int64_t m, int64_t k, int64_t n, void* y,
                                void* workspace, cudaStream_t stream);
// Small batches (m <= kGemvMaxRows) take the HBM-streaming kernel over the same panels
// (dequant_gemv.cu: CUDA-core dequant + mma.sync, stream-K over panels).
constexpr int kGemvMaxRows = 16;
size_t dequant_gemv_workspace_bytes(int64_t n);
// 2-D TMA descriptor (dequant_gemm.cu; the driver entry point is looked up once)
bool make_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t d0, uint64_t d1,
              uint64_t stride1_bytes, uint32_t b0, uint32_t b1, CUtensorMapSwizzle sw,
              CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
cudaError_t launch_dequant_gemv(const void* x, const void* panels, int64_t m, int64_t k, int64_t n, void* y,
                                void* workspace, cudaStream_t stream);

}  // namespace flexq

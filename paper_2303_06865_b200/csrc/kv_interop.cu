// kv_interop.cu -- conversion between the plain quantized KV layout and the chunked cache.
//
// The paper stores the KV cache "in the quantized format" without fixing a
// layout; the plain one -- SURVEY 8(b)'s four arrays, what flexq_quantize produces for the
// token rows of one head -- is
//     codes u8 [B][H][T][CB]     (CB = D*bits/8: the row's codes as a little-endian bit stream,
//                                 S:520; bits = 4: column 2i in the low nibble of byte i)
//     meta  half2 [B][H][T][D/g] ({scale, min} per group of g along D)
// for K and for V.  The cache the attention kernels read (include/flexq.h) regroups the same
// bytes into 32-token chunks [codes 32 x CB][meta 32 x MB], K token-major and -- for
// (bits, group) = (4, 64) -- V quad-interleaved and swizzled.  These kernels move bytes only
// (no arithmetic): import writes cache tokens [t0, t0 + n) from the plain arrays, export
// writes the plain arrays from the cache.  Every byte of the cache belongs to one token, so a
// partial range never rewrites a neighbour (V bytes are stored one by one).
#include <cuda_runtime.h>
#include <stdint.h>

#include "flexq_internal.h"

namespace flexq {
namespace {

struct InteropArgs {
    int64_t rows;        // B * H
    int64_t chunks;      // chunks per (b, h) in the cache
    int plain_t;         // token extent of the plain arrays
    int t0, n;           // token range
    int cb, mb;          // code / meta bytes per token
    bool swz;            // V quad-interleaved + swizzled (bits = 4, group = 64)
};

// byte offset, inside its chunk, of token slot s's code byte i in the swizzled V layout
__device__ __forceinline__ int v_swz_off(int s, int i, int cb) {
    const int quad = s >> 2;
    return (quad * cb + (i ^ ((quad & 3) << 3))) * 4 + (s & 3);
}

// One warp per (b*h, token): lanes stride over the code bytes (16 B pieces where rows are
// contiguous), lanes stride over the meta words.
template <bool IMPORT>
__global__ void __launch_bounds__(256) kv_interop_kernel(const InteropArgs a, uint8_t* k_plain_c, uint8_t* k_plain_m,
                                                         uint8_t* v_plain_c, uint8_t* v_plain_m, uint8_t* k_cache,
                                                         uint8_t* v_cache) {
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= a.rows * a.n) return;
    const int64_t bh = warp / a.n;
    const int t = a.t0 + int(warp - bh * a.n);
    const int s = t & (kChunk - 1);
    const int64_t chunk_off = (bh * a.chunks + (t >> 5)) * int64_t(kChunk) * (a.cb + a.mb);
    const int64_t prow = bh * a.plain_t + t;
    uint8_t* kc = k_cache + chunk_off;
    uint8_t* vc = v_cache + chunk_off;
    uint8_t* kpc = k_plain_c + prow * a.cb;
    uint8_t* vpc = v_plain_c + prow * a.cb;
    uint8_t* kpm = k_plain_m + prow * a.mb;
    uint8_t* vpm = v_plain_m + prow * a.mb;
    // K codes: the row is contiguous in both layouts (cb is a multiple of 4 for every built (bits, D))
    for (int i = lane * 4; i < a.cb; i += 128) {
        uint32_t* c = reinterpret_cast<uint32_t*>(kc + s * a.cb + i);
        uint32_t* p = reinterpret_cast<uint32_t*>(kpc + i);
        if (IMPORT) *c = *p; else *p = *c;
    }
    // V codes
    if (a.swz) {
        for (int i = lane; i < a.cb; i += 32) {
            uint8_t* c = vc + v_swz_off(s, i, a.cb);
            if (IMPORT) *c = vpc[i]; else vpc[i] = *c;
        }
    } else {
        for (int i = lane * 4; i < a.cb; i += 128) {
            uint32_t* c = reinterpret_cast<uint32_t*>(vc + s * a.cb + i);
            uint32_t* p = reinterpret_cast<uint32_t*>(vpc + i);
            if (IMPORT) *c = *p; else *p = *c;
        }
    }
    // meta: token-major after the chunk's codes, in both caches
    for (int i = lane * 4; i < a.mb; i += 128) {
        uint32_t* ck = reinterpret_cast<uint32_t*>(kc + kChunk * a.cb + s * a.mb + i);
        uint32_t* cv = reinterpret_cast<uint32_t*>(vc + kChunk * a.cb + s * a.mb + i);
        uint32_t* pk = reinterpret_cast<uint32_t*>(kpm + i);
        uint32_t* pv = reinterpret_cast<uint32_t*>(vpm + i);
        if (IMPORT) { *ck = *pk; *cv = *pv; } else { *pk = *ck; *pv = *cv; }
    }
}

}  // namespace

cudaError_t launch_kv_interop(bool import_, const KvInterop& x, cudaStream_t stream) {
    InteropArgs a;
    a.rows = x.rows;
    a.chunks = x.chunks;
    a.plain_t = x.plain_tokens;
    a.t0 = x.t0;
    a.n = x.n;
    a.cb = x.head_dim * x.bits / 8;
    a.mb = 4 * x.head_dim / x.group;
    a.swz = x.bits == kBits && x.group == kGroup && !x.v_tm;   // only the dense (4, 64) V is quad-swizzled
    const int64_t warps = a.rows * a.n;
    const int64_t blocks = (warps * 32 + 255) / 256;
    if (blocks > INT32_MAX) return cudaErrorInvalidValue;
    auto k = import_ ? kv_interop_kernel<true> : kv_interop_kernel<false>;
    k<<<unsigned(blocks), 256, 0, stream>>>(a, static_cast<uint8_t*>(x.k_codes), static_cast<uint8_t*>(x.k_meta),
                                            static_cast<uint8_t*>(x.v_codes), static_cast<uint8_t*>(x.v_meta),
                                            static_cast<uint8_t*>(x.k_cache), static_cast<uint8_t*>(x.v_cache));
    return cudaGetLastError();
}

}  // namespace flexq

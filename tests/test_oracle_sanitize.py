"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer ("host oracle under
-fsanitize=address,undefined"): a standalone C driver includes flexq_oracle.c, runs every entry
point on small random inputs (all bit widths, degenerate and extreme groups, exact-size buffers
so any overrun is caught) and must exit cleanly.  CPU only."""
import os
import shutil
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE = os.path.join(os.path.dirname(HERE), "oracle", "flexq_oracle.c")

DRIVER = r"""
#include "FLEXQ_ORACLE"
#include <stdio.h>

static uint64_t st = 0x9E3779B97F4A7C15ull;
static uint32_t rnd(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (uint32_t)st; }
static uint16_t rhalf(int kind) {
    uint32_t u = rnd();
    switch (kind) {
        case 0: return oracle_f32_to_f16(((float)(u % 2001) - 1000.0f) / 256.0f);
        case 1: return (uint16_t)(u & 0x83FF);                       /* subnormal / zero */
        case 2: return (u & 1) ? 0x7BFF : 0xFBFF;                    /* +-65504 */
        default: { uint16_t b = (uint16_t)u; if (((b >> 10) & 0x1F) == 0x1F) b &= 0xFBFF; return b; }
    }
}
#define ALLOC(T, n) ((T *)malloc(sizeof(T) * (size_t)(n)))

int main(void) {
    int fails = 0;
    for (int bits = 1; bits <= 8; ++bits)
        for (int g = 8; g <= 128; g *= 2) {
            const int rows = 3, cols = 2 * g;
            uint16_t *x = ALLOC(uint16_t, rows * cols);
            uint8_t *c = ALLOC(uint8_t, rows * cols), *c2 = ALLOC(uint8_t, rows * cols);
            uint16_t *m = ALLOC(uint16_t, rows * cols / g * 2), *y = ALLOC(uint16_t, rows * cols);
            for (int i = 0; i < rows * cols; ++i) x[i] = rhalf((i / g) % 4);
            for (int i = 0; i < g; ++i) x[i] = x[0];                  /* a constant group */
            fails += oracle_quantize(x, rows, cols, bits, g, c, m) != 0;
            fails += oracle_dequantize(c, m, rows, cols, bits, g, y) != 0;
            uint8_t *p = ALLOC(uint8_t, rows * cols * bits / 8);
            fails += oracle_pack_bits(c, rows * cols, bits, p) != 0;
            fails += oracle_unpack_bits(p, rows * cols, bits, c2) != 0;
            for (int i = 0; i < rows * cols; ++i) fails += c[i] != c2[i];
            free(x); free(c); free(c2); free(m); free(y); free(p);
        }
    /* KV append + attention (dense, f32 twin, Top-K) */
    const int B = 2, H = 3, D = 64, T = 40, cur = 37, grp = 64;
    uint16_t *kn = ALLOC(uint16_t, B * H * T * D), *vn = ALLOC(uint16_t, B * H * T * D), *q = ALLOC(uint16_t, B * H * D);
    for (int i = 0; i < B * H * T * D; ++i) { kn[i] = rhalf(i % 3 == 0 ? 3 : 0); vn[i] = rhalf(0); }
    for (int i = 0; i < B * H * D; ++i) q[i] = rhalf(0);
    uint8_t *kc = ALLOC(uint8_t, B * H * T * D), *vc = ALLOC(uint8_t, B * H * T * D);
    uint16_t *km = ALLOC(uint16_t, B * H * T * (D / grp) * 2), *vm = ALLOC(uint16_t, B * H * T * (D / grp) * 2);
    fails += oracle_append_kv(kn, vn, B, H, D, T, 0, T, 4, grp, kc, km, vc, vm) != 0;
    double *o = ALLOC(double, B * H * D), *pr = ALLOC(double, B * H * cur), *sc = ALLOC(double, B * H * cur);
    float *of = ALLOC(float, B * H * D);
    uint8_t *sel = ALLOC(uint8_t, B * H * cur);
    fails += oracle_attention_f64(q, kc, km, vc, vm, B, H, D, T, cur, grp, o, pr) != 0;
    fails += oracle_attention_f64(q, kc, km, vc, vm, B, H, D, T, cur, grp, o, NULL) != 0;
    fails += oracle_attention_f32(q, kc, km, vc, vm, B, H, D, T, cur, grp, of) != 0;
    fails += oracle_attention_topk_f64(q, kc, km, vc, vm, B, H, D, T, cur, grp, 4, NULL, sel, sc, o) != 0;
    fails += oracle_attention_f64(q, kc, km, vc, vm, B, H, D, T, T + 1, grp, o, NULL) == 0;   /* rejected */
    /* decode linear layer */
    const int M = 3, K = 16, N = 128;
    uint16_t *xw = ALLOC(uint16_t, M * K), *w = ALLOC(uint16_t, K * N), *wm = ALLOC(uint16_t, K * N / 64 * 2);
    uint8_t *wc = ALLOC(uint8_t, K * N);
    double *yo = ALLOC(double, M * N);
    for (int i = 0; i < M * K; ++i) xw[i] = rhalf(0);
    for (int i = 0; i < K * N; ++i) w[i] = rhalf(i % 4);
    fails += oracle_quantize(w, K, N, 4, 64, wc, wm) != 0;
    fails += oracle_dequant_gemm_f64(xw, wc, wm, M, K, N, 4, 64, yo) != 0;
    free(kn); free(vn); free(q); free(kc); free(vc); free(km); free(vm); free(o); free(pr); free(sc); free(of);
    free(sel); free(xw); free(w); free(wm); free(wc); free(yo);
    printf("oracle sanitize fails=%d\n", fails);
    return fails != 0;
}
"""


def test_oracle_under_asan_ubsan():
    cc = shutil.which("gcc")
    if not cc:
        pytest.skip("gcc not available")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "drv.c")
        exe = os.path.join(d, "drv")
        open(src, "w").write(DRIVER.replace("FLEXQ_ORACLE", ORACLE))
        r = subprocess.run([cc, "-std=c11", "-O1", "-g", "-ffp-contract=off", "-fno-fast-math",
                            "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-o", exe, src, "-lm"],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1"))
        assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
        assert "oracle sanitize fails=0" in r.stdout

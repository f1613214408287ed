"""Host check of the division identity the quantize kernel relies on (quant.cu):
for the operands of P:843's (x - min) / (max - min) in fp32 -- a = RN(x - min),
r = RN(max - min) with x, min, max fp16 -- one correctly rounded reciprocal
y = RN(1/r) plus the Markstein correction q0 = RN(a y), e = fma(-q0, r, a),
u = RN(q0 + e y) equals the IEEE quotient RN(a / r) bit for bit (reading B:
the GPU may use this form only if it is bit-identical to IEEE a / r).

Samples: uniformly random finite fp16 triples (every exponent), Irwin-Hall
values at random scales, and constructed exact ties a = (2k+1) m 2^e,
r = 30 m 2^e.  Written in C (gcc -ffp-contract=off); shares no code with
csrc/ or oracle/.
"""
import os

import pytest
import subprocess
import tempfile

SRC = r"""
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
static uint64_t st = 88172645463325252ull;
static uint64_t xr(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return st; }
static float h2f(uint16_t h) { int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  float v = e ? ldexpf(1024 + m, e - 25) : ldexpf(m, -24); return s ? -v : v; }
static uint16_t rh(void) { for (;;) { uint16_t h = (uint16_t)xr(); if (((h >> 10) & 31) != 31) return h; } }
static float f16r(float v) { _Float16 h = (_Float16)v; return (float)h; }
static long bad = 0, tested = 0;
static void check(float a, float r) {
  float u = a / r;
  float y = 1.0f / r, q0 = a * y, e = fmaf(-q0, r, a), q1 = fmaf(e, y, q0);
  tested++;
  if (memcmp(&u, &q1, 4) != 0 && !(u == 0.0f && q1 == 0.0f)) {
    if (bad < 5) printf("MISMATCH a=%a r=%a ieee=%a markstein=%a\n", a, r, u, q1);
    bad++;
  }
}
static void triple(float x, float y, float z) {
  float v[3] = {x, y, z};
  for (int p = 0; p < 3; p++) for (int q = p + 1; q < 3; q++) if (v[q] < v[p]) { float t = v[p]; v[p] = v[q]; v[q] = t; }
  float mn = v[0] == 0.0f ? 0.0f : v[0];
  float r = v[2] - mn;
  if (r == 0.0f || !isfinite(r)) return;
  check(v[1] - mn, r);
}
int main(int argc, char **argv) {
  long n = atol(argv[1]);
  for (long i = 0; i < n; i++) {
    triple(h2f(rh()), h2f(rh()), h2f(rh()));
    int sc = (int)(xr() % 40) - 24;
    float v[3];
    for (int k = 0; k < 3; k++) { double s = 0; for (int j = 0; j < 4; j++) s += (double)(xr() >> 40) / (double)(1ull << 24);
      v[k] = f16r((float)ldexp(s - 2.0, sc)); }
    triple(v[0], v[1], v[2]);
    int k = xr() % 15, m = 1 + xr() % 2047, ex = (int)(xr() % 60) - 40;
    check(ldexpf((float)((2 * k + 1) * m), ex), ldexpf((float)(30 * m), ex));
  }
  printf("tested %ld bad %ld\n", tested, bad);
  return bad != 0;
}
"""


def test_markstein_division_equals_ieee():
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "div.c")
        exe = os.path.join(d, "div")
        open(c, "w").write(SRC)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-o", exe, c, "-lm"])
        out = subprocess.run([exe, "4000000"], capture_output=True, text=True)
        assert out.returncode == 0, out.stdout
        tested = int(out.stdout.split()[-3])
        assert tested > 10_000_000


SRC15 = r"""
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <math.h>
int main(int argc, char **argv) {
  /* every fp32 r in [2^-24, 131008] (a superset of RN(max - min) over fp16 groups) */
  const float L = argc > 1 ? (float)atoi(argv[1]) : 15.0f;   /* 2^b - 1 */
  const float y = 1.0f / L;
  uint32_t lo, hi; float flo = ldexpf(1.0f, -24), fhi = 131008.0f;
  memcpy(&lo, &flo, 4); memcpy(&hi, &fhi, 4);
  long bad = 0, tested = 0;
  for (uint32_t b = lo; b <= hi; b++) {
    float r; memcpy(&r, &b, 4);
    float u = r / L;
    float s0 = r * y, s1 = fmaf(fmaf(-s0, L, r), y, s0);
    tested++;
    if (memcmp(&u, &s1, 4) != 0) { if (bad < 5) printf("MISMATCH r=%a ieee=%a markstein=%a\n", r, u, s1); bad++; }
  }
  printf("y=%a tested %ld bad %ld\n", y, tested, bad);
  return bad != 0;
}
"""


@pytest.mark.parametrize("levels,recip", [(15, "0x1.111112p-4"), (3, "0x1.555556p-2"), (7, "0x1.24924ap-3"),
                                          (255, "0x1.010102p-8")])
def test_scale_division_exhaustive(levels, recip):
    """RN(r / L) (the stored scale, O5, L = 2^b - 1) as s0 = RN(r * RN(1/L)), RN(s0 + fma(-s0, L, r) * RN(1/L)):
    equal to IEEE division for every fp32 r in the operand range (the quantize and fused append kernels'
    form), for b = 4 and the NEXT-3 variants b = 2, 3, 8."""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "div15.c")
        exe = os.path.join(d, "div15")
        open(c, "w").write(SRC15)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-o", exe, c, "-lm"])
        out = subprocess.run([exe, str(levels)], capture_output=True, text=True)
        assert out.returncode == 0, out.stdout
        assert f"y={recip}" in out.stdout                # RN(1/L), the kernels' constant
        assert int(out.stdout.split()[-3]) > 300_000_000

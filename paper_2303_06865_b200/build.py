"""Build libflexq.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

    python -m paper_2303_06865_b200.build         # incremental
    python -m paper_2303_06865_b200.build --force

quant.cu is compiled with -fmad=false (the fp32 quantize formula must not be
contracted, reading B); decode_attention.cu keeps FMA contraction on.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libflexq.so")
BUILD = os.path.join(HERE, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
          "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES = {
    "flexq_api.cu": [],
    "quant.cu": ["-fmad=false", "-prec-div=true", "-ftz=false"],
    "decode_attention.cu": [],
    "decode_attention_topk.cu": [],
    "decode_attention_variants.cu": [],
    "dequant_gemm.cu": [],
    "dequant_gemv.cu": [],
    "kv_interop.cu": [],
    "device_info.cu": [],
}


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), tag: str = "") -> str:
    """Build libflexq.so (or, for A/B tuning, libflexq_<tag>.so with extra -D defines)."""
    build_dir = BUILD + ("_" + tag if tag else "")
    lib = LIB if not tag else LIB.replace("libflexq.so", f"libflexq_{tag}.so")
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, "flexq_internal.h"), os.path.join(CSRC, "attn_common.cuh"),
               os.path.join(INCLUDE, "flexq.h"), __file__]
    objs = []
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [nvcc(), *ARCH, *COMMON, *extra, *[f"-D{d}" for d in defines], "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(o + ".ptxas.txt", "w") as f:
                f.write(r.stderr)
    if force or _stale(lib, objs):
        tmp = lib + ".tmp%d" % os.getpid()
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--deq-ab" in sys.argv:
        print(build(force="--force" in sys.argv, defines=("FLEXQ_DEQ_UNROLL=1", "FLEXQ_DEQ_CS=0"), tag="deq1"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_DEQ_UNROLL=4", "FLEXQ_DEQ_CS=0"), tag="deq4n"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_DEQ_UNROLL=2",), tag="deq2"))
    if "--gemv-ab" in sys.argv:
        for v in (1, 3, 4):
            print(build(force="--force" in sys.argv, defines=(f"FLEXQ_GEMV_PROBE={v}",), tag=f"gemv{v}"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_GEMV_CTAS=1",), tag="gemv1cta"))
    if "--l2pf-ab" in sys.argv:
        for n in (4, 9):
            print(build(force="--force" in sys.argv, defines=(f"FLEXQ_ATTN_L2PF={n}",), tag=f"l2pf{n}"))
    if "--trace" in sys.argv:
        print(build(force="--force" in sys.argv, defines=("FLEXQ_ATTN_TRACE=1",), tag="trace"))
    if "--topk-hint-ab" in sys.argv:
        print(build(force="--force" in sys.argv, defines=("FLEXQ_TOPK_L2HINT=0",), tag="nohint"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_TOPK_GATHER_MINB=4",), tag="gmin4"))
    if "--topk-ab" in sys.argv:
        for w, m in ((2, 8), (4, 4), (2, 6), (3, 5)):
            print(build(force="--force" in sys.argv, defines=(f"FLEXQ_TOPK_WPC={w}", f"FLEXQ_TOPK_MINB={m}"),
                        tag=f"topk_w{w}m{m}"))
    if "--gemm-ab" in sys.argv:
        print(build(force="--force" in sys.argv, defines=("FLEXQ_GEMM_DQW=8",), tag="dqw8"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_GEMM_TRACE=1",), tag="trace"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_GEMM_PROBE=1",), tag="nostt"))
        print(build(force="--force" in sys.argv, defines=("FLEXQ_GEMM_PROBE=2",), tag="nomath"))

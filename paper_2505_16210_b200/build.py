"""Builds the in-tree C-ABI library libnqkv.so for sm_100a with nvcc.

Flags: -O3 -lineinfo, IEEE-exact fp32 (no --use_fast_math, --ftz, or
--prec-div=false: the quantize path relies on correctly rounded division and
reciprocal).
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libnqkv.so")
SOURCES = [os.path.join(CSRC, "nqkv.cu"), os.path.join(CSRC, "levels.cpp")]
DEPS = sorted(glob.glob(os.path.join(CSRC, "*"))) + [os.path.join(ROOT, "include", "nqkv.h"),
                                                    os.path.abspath(__file__)]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def source_id() -> str:
    """sha256 (16 hex digits) of every source the library is built from."""
    import hashlib
    h = hashlib.sha256()
    for d in DEPS:
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def built_id(lib: str = LIB) -> str | None:
    """The build id embedded in a built library, read from the file (loading it
    here would pin the old image in this process: dlopen caches by path)."""
    try:
        with open(lib, "rb") as f:
            data = f.read()
    except OSError:
        return None
    i = data.find(b"NQKV_BUILD_ID=")
    if i < 0:
        return None
    j = data.find(b"\0", i)
    return data[i + 14:j].decode(errors="replace")


def needs_build() -> bool:
    """Rebuild when the library is missing or was built from other sources
    (embedded build id != hash of the current sources)."""
    if not os.path.exists(LIB):
        return True
    return built_id() != source_id()


def build_library(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    tmp = LIB + ".tmp"
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", tmp,
                                   f'-DNQKV_BUILD_ID="{source_id()}"'] + SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stdout + r.stderr)
    os.replace(tmp, LIB)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    return LIB


def build_variant(out: str, defines: dict) -> str:
    """Development: build a tuning variant (e.g. {"NQKV_DECODE_WARPS": 16}) to `out`."""
    cmd = [nvcc()] + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-o", out] + \
        [f"-D{k}={v}" for k, v in defines.items()] + SOURCES
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    return out


if __name__ == "__main__":
    print(build_library(force=True, verbose=True))

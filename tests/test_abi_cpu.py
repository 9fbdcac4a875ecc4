"""C-ABI checks that need no GPU: the library loads, exports every symbol the
header declares, host entry points agree with the oracle, and host-checkable
argument errors return the documented status without launching anything."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__

__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402
from oracle import nqkv_oracle as O  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FAKE = 0x10000   # 16-byte aligned, never dereferenced: validation fails first


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "nqkv.h")).read()
    declared = set(re.findall(r"\b(nqkv_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(N.EXPORTED)
    lib = ctypes.CDLL(N._LIB_PATH)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.nqkv_abi_version() == 4


def test_host_levels_and_thresholds_match_oracle_bits():
    # two independent Phi^-1 implementations (C++ erfc-Halley vs scipy ndtri)
    assert np.array_equal(N.nqkv_levels().view(np.uint32), O.nf_levels_f32().view(np.uint32))
    assert np.array_equal(N.nqkv_thresholds().view(np.uint32), O.thresholds_f32().view(np.uint32))


def test_status_strings():
    for s in range(-7, 1):
        assert N._lib.nqkv_status_string(s)


def _q(**kw):
    a = dict(x=FAKE, sb=64 * 12 * 512, st=64 * 12, sh=64, B=1, H=12, hd=64, n=512, blk=64,
             pos=FAKE, Tc=512, codes=FAKE, scales=FAKE, stream=None)
    a.update(kw)
    return N._lib.nqkv_quantize(a["x"], a["sb"], a["st"], a["sh"], a["B"], a["H"], a["hd"], a["n"],
                                a["blk"], a["pos"], a["Tc"], a["codes"], a["scales"], a["stream"])


def test_quantize_argument_errors():
    assert _q(x=None) == -1 and _q(pos=None) == -1 and _q(codes=None) == -1
    assert _q(hd=96) == -3 and _q(blk=16) == -3 and _q(blk=512) == -3
    # blk > hd: a block spans blk/hd heads; H must hold whole head groups
    assert _q(blk=128, hd=64, n=0) == 0 and _q(blk=256, hd=64, n=0) == 0
    assert _q(blk=256, hd=64, H=6, n=0) == -2 and _q(blk=256, hd=128, H=7, n=0) == -2
    assert _q(Tc=500) == -2 and _q(B=-1) == -2
    assert _q(x=FAKE + 2) == -4 and _q(sh=60) == -4 and _q(codes=FAKE + 8) == -4
    assert _q(B=0) == 0 and _q(n=0) == 0          # nothing to do, nothing launched


def _d(**kw):
    a = dict(q=FAKE, kc=FAKE, ks=FAKE, vc=FAKE, vs=FAKE, lens=FAKE, B=2, H=4, hd=128, blk=64,
             Tc=256, scale=0.088, out=FAKE, ws=FAKE, ws_bytes=None, stream=None)
    a.update(kw)
    if a["ws_bytes"] is None:
        a["ws_bytes"] = N.nqkv_decode_workspace_bytes(a["B"], a["H"], a["hd"], a["Tc"])
    return N._lib.nqkv_decode_attention(a["q"], a["kc"], a["ks"], a["vc"], a["vs"], a["lens"],
                                        a["B"], a["H"], a["hd"], a["blk"], a["Tc"], a["scale"],
                                        a["out"], a["ws"], a["ws_bytes"], a["stream"])


def test_decode_argument_errors():
    assert _d(q=None) == -1 and _d(lens=None) == -1 and _d(ws=None) == -1
    assert _d(hd=256) == -3 and _d(blk=8) == -3
    assert _d(Tc=100) == -2
    assert _d(blk=256, H=3) == -2                     # 1.5 head groups of 2 heads
    assert _d(q=FAKE + 4) == -4 and _d(out=FAKE + 8) == -4 and _d(ks=FAKE + 2) == -4
    assert _d(ws_bytes=16) == -5
    assert _d(B=0) == 0


def test_decode_step_argument_errors():
    f = N._lib.nqkv_decode_step
    ws = N.nqkv_decode_workspace_bytes(2, 4, 128, 256)
    args = [FAKE, FAKE, 4 * 128, 128, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 2, 4, 128, 64, 256,
            0.088, FAKE, FAKE, ws, None]
    a = list(args); a[0] = None
    assert f(*a) == -1
    a = list(args); a[3] = 100                        # stride not a multiple of 8
    assert f(*a) == -4
    a = list(args); a[12] = 96
    assert f(*a) == -3
    a = list(args); a[18] = 8
    assert f(*a) == -5
    a = list(args); a[10] = 5000                      # B > kMaxBatch (1024)
    assert f(*a) == -2


def test_dequant_argument_errors():
    f = N._lib.nqkv_dequantize
    assert f(None, FAKE, 1, 1, 64, 64, 64, 64, 0, FAKE, None) == -1
    assert f(FAKE, FAKE, 1, 1, 64, 64, 64, 65, 0, FAKE, None) == -2       # n_tokens > Tc
    assert f(FAKE, FAKE, 1, 1, 64, 64, 64, 64, 2, FAKE, None) == -3       # bad dtype
    assert f(FAKE, FAKE, 1, 1, 64, 64, 64, 0, 0, FAKE, None) == 0


def test_workspace_size_grows_with_geometry():
    a = N.nqkv_decode_workspace_bytes(8, 32, 64, 2112)
    b = N.nqkv_decode_workspace_bytes(8, 32, 128, 2112)
    c = N.nqkv_decode_workspace_bytes(16, 32, 64, 2112)
    assert 0 < a < b and a < c and a % 256 == 0
    assert N.nqkv_decode_workspace_bytes(8, 32, 96, 2112) == 0        # unsupported hd
    # per-(b, h) int32 counters first, then per-CTA split partials (o[hd], m, l)
    assert N.nqkv_decode_counter_bytes(8, 32) == 8 * 32 * 4
    assert a >= N.nqkv_decode_counter_bytes(8, 32) + 148 * 2 * (64 + 2) * 8     # tagged 64-bit words


def test_missing_library_fails_loudly(tmp_path):
    import subprocess
    import sys
    code = ("import sys, os; sys.path.insert(0, %r); "
            "import paper_2505_16210_b200.nqkv as m" % str(tmp_path))
    pkg = tmp_path / "paper_2505_16210_b200"
    pkg.mkdir()
    (pkg / "__init__.py").write_text("")
    (pkg / "nqkv.py").write_text(open(N.__file__).read())
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert r.returncode != 0 and "not built" in r.stderr


def test_plan_argument_errors():
    f = N._lib.nqkv_decode_plan
    nb = N._lib.nqkv_decode_plan_bytes()
    assert f(None, 4, 8, 64, 256, 0, FAKE, nb, None) == -1
    assert f(FAKE, 4, 8, 96, 256, 0, FAKE, nb, None) == -3        # unsupported head_dim
    assert f(FAKE, 4, 8, 64, 100, 0, FAKE, nb, None) == -2        # Tc not a multiple of 64
    assert f(FAKE, 4, 8, 64, 256, 0, FAKE + 4, nb, None) == -4    # misaligned plan
    assert f(FAKE, 4, 8, 64, 256, 0, FAKE, nb - 16, None) == -5   # plan buffer too small


def test_scale_f16_flag_validation():
    f16 = N.SCALE_F16
    # n = 0: every check runs, nothing is launched
    assert _q(blk=64 | f16, n=0) == 0                              # accepted
    assert _q(blk=64 | 0x200, n=0) == -3                           # unknown flag bit
    assert _q(blk=64 | f16, scales=FAKE + 2, n=0) == 0             # fp16 scales: 2-byte alignment suffices
    assert _q(blk=64, scales=FAKE + 2, n=0) == -4                  # fp32 scales need 4
    assert _q(blk=64 | f16, scales=FAKE + 1, n=0) == -4


def test_decode_gather_argument_errors():
    f = N._lib.nqkv_decode_step_gather
    ws = N.nqkv_decode_workspace_bytes(2, 4, 128, 256)
    base = [FAKE, FAKE, 4 * 128, 128, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 2, 4, 128, 64, 256, 0.088,
            FAKE, FAKE, 2, 0, 8, 1, None, FAKE, ws, FAKE, 0, None]
    a = list(base); a[16] = None                     # peer output array
    assert f(*a) == -1
    a = list(base); a[25] = None                     # plan
    assert f(*a) == -1
    a = list(base); a[19] = 2                        # rank >= G
    assert f(*a) == -2
    a = list(base); a[20] = 12                       # H_total != G * H
    assert f(*a) == -2
    a = list(base); a[21] = 0                        # epoch 0 is reserved (without d_epoch)
    assert f(*a) == -2
    assert N._lib.nqkv_gather_epoch_bump(None, None) == -1
    assert N._lib.nqkv_gather_wait(None, 4, FAKE, None) == -1
    assert N._lib.nqkv_gather_wait(FAKE, -1, FAKE, None) == -2
    assert N._lib.nqkv_gather_wait(FAKE, 0, FAKE, None) == 0
    a = list(base); a[12] = 96
    assert f(*a) == -3


def test_build_id_matches_sources():
    """The library embeds the hash of the sources it was built from; build()
    rebuilds on a mismatch, so a stale library is never reused."""
    from paper_2505_16210_b200 import build as bld
    from paper_2505_16210_b200 import nqkv as N
    assert bld.built_id() == bld.source_id()
    assert N._lib.nqkv_build_id().decode() == bld.source_id()
    assert not bld.needs_build()


def _dkv(lay, **kw):
    a = dict(q=FAKE, B=2, H=8, hd=128, blk=64, Tc=512, ws=FAKE, wsb=1 << 30)
    a.update(kw)
    return N._lib.nqkv_decode_attention_kv(a["q"], FAKE, FAKE, FAKE, FAKE, FAKE, a["B"], a["H"], a["hd"],
                                           a["blk"], a["Tc"], None if lay is None else ctypes.byref(lay),
                                           0.1, FAKE, a["ws"], a["wsb"], None)


def test_kv_layout_argument_errors():
    # grouped-query (R16) and paged (R17) layouts: host-checkable errors, no launch
    L = N.KvLayout
    assert _dkv(None) == -1
    assert _dkv(L(3, None, 0, 0, 0)) == -2            # 8 query heads over 3 KV heads
    assert _dkv(L(8, None, 0, 0, 0), B=0) == 0         # nothing to do
    assert _dkv(L(2, None, 0, 0, 0), B=0) == 0         # group 4: valid
    assert _dkv(L(0, None, 0, 0, 0), H=12, B=0) == 0
    assert _dkv(L(4, None, 0, 0, 0), H=12) == -3      # group 3: not a power of two
    assert _dkv(L(2, FAKE, 8, 32, 64)) == -3          # page_size < 64
    assert _dkv(L(2, FAKE, 8, 96, 64)) == -3          # not a power of two
    assert _dkv(L(2, FAKE, 4, 64, 64)) == -2          # 4 pages x 64 < Tc = 512
    assert _dkv(L(2, FAKE, 8, 64, 0)) == -2           # no pages
    assert _dkv(L(2, FAKE + 2, 8, 64, 64)) == -4      # block table alignment
    assert _dkv(L(2, FAKE, 8, 64, 1 << 20)) == -2     # 32-bit row offsets
    assert _dkv(L(2, FAKE, 8, 64, 64), blk=64 | N.SCALE_F16) == -3   # paged: fp32 scales
    assert _dkv(L(2, FAKE, 8, 64, 64), B=0) == 0
    # quantize: x holds the cache heads
    q = N._lib.nqkv_quantize_kv
    lay = L(6, None, 0, 0, 0)
    assert q(FAKE, 64 * 12 * 512, 64 * 12, 64, 1, 12, 64, 512, 64, FAKE, 512, ctypes.byref(lay), FAKE, FAKE, None) == -2
    lay = L(0, FAKE, 8, 64, 64)
    assert q(FAKE, 64 * 12 * 512, 64 * 12, 64, 0, 12, 64, 512, 64, FAKE, 512, ctypes.byref(lay), FAKE, FAKE, None) == 0
    assert q(FAKE, 64 * 12 * 512, 64 * 12, 64, 1, 12, 64, 512, 64, FAKE, 512, None, FAKE, FAKE, None) == -1
    p = N._lib.nqkv_prefill_attention_kv
    assert p(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 1, 8, 64, 64, 512, 16, ctypes.byref(L(3, None, 0, 0, 0)),
             0.1, FAKE, None) == -2
    assert p(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0, 8, 64, 64, 512, 16, ctypes.byref(L(2, None, 0, 0, 0)),
             0.1, FAKE, None) == 0

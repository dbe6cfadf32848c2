"""CPU-side checks of the C ABI: libswr.so loads, exports every function that
include/swr.h declares, and rejects bad arguments with the documented status
codes before touching the GPU (no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from conftest import build_lib
    build_lib()
    from paper_2512_13921_b200 import _lib
    return _lib


def header_functions():
    text = open(os.path.join(ROOT, "include", "swr.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:SWR_API\s+)?(?:const\s+)?\w+\*?\s+\*?(\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_north_star_entry_points():
    fns = header_functions()
    for f in ("swr_fwd", "swr_bwd", "phalanx_mix", "phalanx_mix_bwd", "swr_strerror"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    so = ctypes.CDLL(lib.LIB_PATH)
    for f in header_functions():
        assert hasattr(so, f), f"libswr.so does not export {f}"
    assert set(header_functions()) == set(lib.EXPORTS)


def test_only_abi_symbols_are_exported(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(header_functions()) <= syms
    assert not [s for s in syms if s.startswith("_ZN3swr")], "internal symbols leaked"


def _shape(lib, B=1, L=64, H=1, D=16, sx=None, sa=None):
    sx = sx or (L * H * D, H * D, D)
    sa = sa or (L * H, H, 1)
    return lib.swr_shape(B, L, H, D, *sx, *sa)


FAKE = 1 << 20  # 16-byte aligned, never dereferenced: validation fails first


def test_validation_codes(lib):
    s = _shape(lib)
    # NULL required pointers
    assert lib.raw_status("swr_fwd", None, FAKE, FAKE, None, None, s, 0, None) == 1
    assert lib.raw_status("swr_fwd", FAKE, None, FAKE, None, None, s, 0, None) == 1
    assert lib.raw_status("swr_bwd", FAKE, FAKE, FAKE, FAKE, None, None, None, None, s, 0, None) == 1
    assert lib.raw_status("phalanx_mix", FAKE, FAKE, None, FAKE, FAKE, None, None, s, 0, None) == 1
    # bad dtype
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None, s, 7, None) == 5
    # unsupported head dim / negative sizes
    for D in (8, 24, 256):
        assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None, _shape(lib, D=D), 0, None) == 2
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None, _shape(lib, L=-1), 0, None) == 2
    # strides: d-tensor strides must be multiples of 16 bytes, none negative
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None,
                          _shape(lib, sx=(64 * 16, 18, 16)), 1, None) == 3
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None,
                          _shape(lib, sa=(64, -1, 1)), 1, None) == 3
    # a zero stride over a dimension of size > 1 would make outputs overlap
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None,
                          _shape(lib, H=4, sx=(64 * 64, 64, 0)), 0, None) == 3
    assert lib.raw_status("swr_bwd", FAKE, FAKE, FAKE, FAKE, FAKE, None, None, None,
                          _shape(lib, H=4, sa=(256, 0, 1)), 0, None) == 3
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None,
                          _shape(lib, B=2, sa=(0, 1, 1)), 0, None) == 3
    # grid limits: B <= 65535, H <= 65535 * 4
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None, _shape(lib, B=65536), 0, None) == 2
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, None, None, _shape(lib, H=65535 * 4 + 1),
                          0, None) == 2
    # alignment: d-tensors and carries 16 B, decays element size
    assert lib.raw_status("swr_fwd", FAKE + 4, FAKE, FAKE, None, None, s, 0, None) == 4
    assert lib.raw_status("swr_fwd", FAKE, FAKE + 1, FAKE, None, None, s, 1, None) == 4
    assert lib.raw_status("swr_fwd", FAKE, FAKE, FAKE, FAKE + 8, None, s, 0, None) == 4


def test_decode_step_validation_codes(lib):
    s1 = _shape(lib, L=1)
    # one token per call, non-negative position
    assert lib.raw_status("swr_decode_step", FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0, _shape(lib, L=2), 0,
                          None) == 2
    assert lib.raw_status("swr_decode_step", FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, -1, s1, 0, None) == 2
    # required operands and state
    assert lib.raw_status("swr_decode_step", None, FAKE, FAKE, FAKE, FAKE, FAKE, 0, s1, 0, None) == 1
    assert lib.raw_status("swr_decode_step", FAKE, FAKE, FAKE, FAKE, FAKE, None, 0, s1, 0, None) == 1
    assert lib.raw_status("phalanx_mix_decode_step", FAKE, FAKE, None, FAKE, FAKE, FAKE, FAKE, FAKE, 0, s1,
                          0, None) == 1
    # state alignment: w, v 16 B; g 4 B
    assert lib.raw_status("swr_decode_step", FAKE, FAKE, FAKE, FAKE + 4, FAKE, FAKE, 0, s1, 0, None) == 4
    assert lib.raw_status("swr_decode_step", FAKE, FAKE, FAKE, FAKE, FAKE, FAKE + 2, 0, s1, 0, None) == 4


def test_strerror_names_every_code(lib):
    for code in range(9):
        assert lib._lib.swr_strerror(code).decode().startswith("SWR_")


def test_python_api_refuses_cpu_tensors(lib):
    import torch
    import paper_2512_13921_b200 as P
    u = torch.zeros(1, 16, 1, 16)
    a = torch.zeros(1, 16, 1)
    with pytest.raises(ValueError, match="CUDA"):
        P.swr_fwd(u, a)


def test_layout_copies_are_counted(lib):
    """ops._prep passes ABI-ready d-tensors through and counts every copy it makes
    (layout) and every gradient cast (dtype); no kernel is called here."""
    import torch

    from paper_2512_13921_b200 import ops
    x = torch.zeros(2, 32, 4, 16)
    n0 = ops.layout_copies()
    (y,) = ops._prep(x)
    assert y is x and ops.layout_copies() == n0
    t = torch.zeros(2, 4, 32, 16).transpose(1, 2)  # [B, L, H, D] view of head-major storage
    ops._prep(x, t)  # strides differ: both copied
    assert ops.layout_copies() == n0 + 2
    a = torch.zeros(2, 32, 1).expand(2, 32, 4)  # a decay row shared by the heads
    assert ops._prep_a(a).is_contiguous() and ops.layout_copies() == n0 + 3
    g = ops._grad_as(torch.zeros(2, 32, 4, 16, dtype=torch.float64), x)
    assert g.dtype == x.dtype and ops.layout_copies() == n0 + 4
    assert ops._grad_as(x, x) is x and ops.layout_copies() == n0 + 4


def test_layer_validation_codes(lib):
    """phalanx_layer_mix(_bwd): groups must divide H, group tensors need D contiguous,
    16-byte strides and pointers; checked before any launch."""
    H, L, D = 8, 64, 16

    def layer(Gq=4, Gk=2, sq=None, sk=None, la=1, lk=1):
        sq = sq or (L * Gq * D, Gq * D, D)
        sk = sk or (L * Gk * D, Gk * D, D)
        return lib.swr_layer(Gq, Gk, *sq, *sk, la, lk)

    s = _shape(lib, H=H)
    fwd = lambda g, q=FAKE, k=FAKE: lib.raw_status("phalanx_layer_mix", q, k, FAKE, FAKE, FAKE, None, None, s,  # noqa: E731
                                                   g, 0, None)
    bwd = lambda g, dq=FAKE: lib.raw_status("phalanx_layer_mix_bwd", FAKE, FAKE, FAKE, FAKE, FAKE, dq, FAKE,  # noqa: E731
                                            FAKE, FAKE, None, None, None, s, g, 0, None)
    assert fwd(layer(Gq=3)) == 2 and fwd(layer(Gk=0)) == 2 and bwd(layer(Gk=5)) == 2
    assert fwd(layer(sq=(L * 4 * D, 4 * D, 2))) == 3       # head stride not 16 bytes
    assert fwd(layer(sk=(L * 2 * D, 0, D))) == 3           # zero token stride, L > 1
    assert fwd(layer(), q=None) == 1 and bwd(layer(), dq=None) == 1
    assert fwd(layer(), k=FAKE + 4) == 4


def test_exact_workspace_validation(lib):
    """swr_exact_fwd needs twice swr_exact_workspace_bytes(s), swr_exact_bwd three times
    (the look-back scans' per-block stashes and scratch); too small -> SWR_ERR_SHAPE,
    NULL -> SWR_ERR_NULL, checked before any launch."""
    s = _shape(lib, H=2, L=100)
    n = lib.swr_exact_workspace_bytes(s)
    assert n > 0
    fwd = lambda ws, nb: lib.raw_status("swr_exact_fwd", FAKE, FAKE, FAKE, None, None, ws, nb, s, 0, None)  # noqa: E731
    bwd = lambda ws, nb: lib.raw_status("swr_exact_bwd", FAKE, FAKE, FAKE, FAKE, FAKE, None, None, None, ws, nb,  # noqa: E731
                                        s, 0, None)
    assert fwd(None, 2 * n) == 1 and fwd(FAKE, 2 * n - 4) == 2
    assert bwd(None, 3 * n) == 1 and bwd(FAKE, 2 * n) == 2
    assert lib.swr_exact_workspace_bytes(_shape(lib, L=0)) == 0


def test_layer_workspace_bytes(lib):
    """The tensor-core layer backward's scratch: one bf16 [B, L, H, D] per shared gate
    tensor; none for fp32, d != 128, unshared groups or q and k both shared by pairs."""
    H, L = 16, 64
    s = _shape(lib, H=H, L=L, D=128, sx=(L * H * 128, H * 128, 128))
    lay = lambda Gq, Gk: lib.swr_layer(Gq, Gk, L * Gq * 128, Gq * 128, 128, L * Gk * 128, Gk * 128, 128, 1, 1)  # noqa: E731
    per = 1 * L * H * 128 * 2
    assert lib.phalanx_layer_workspace_bytes(s, lay(4, 4), lib.SWR_BF16) == 2 * per
    assert lib.phalanx_layer_workspace_bytes(s, lay(4, 16), lib.SWR_BF16) == per
    assert lib.phalanx_layer_workspace_bytes(s, lay(8, 16), lib.SWR_BF16) == per
    assert lib.phalanx_layer_workspace_bytes(s, lay(16, 16), lib.SWR_BF16) == 0
    # pairs of heads sharing q and k (the paper's 8 groups at H = 16): summed in the kernel
    assert lib.phalanx_layer_workspace_bytes(s, lay(8, 8), lib.SWR_BF16) == 0
    assert lib.phalanx_layer_workspace_bytes(s, lay(8, 8), lib.SWR_F32) == 0

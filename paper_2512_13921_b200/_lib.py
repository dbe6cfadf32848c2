"""ctypes binding of libswr.so (include/swr.h).  Argument marshalling only.

Every function here takes raw device pointers / sizes exactly like the C ABI and
raises ``SwrError`` on a non-zero status.  There is no CPU fallback: if the
shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# SWR_LIB: an alternative in-tree build of the same library (kernel A/B experiments)
LIB_PATH = os.environ.get("SWR_LIB") or os.path.join(_PKG, "libswr.so")

SWR_F32, SWR_BF16 = 0, 1
SWR_PATH_AUTO, SWR_PATH_FFMA, SWR_PATH_TC = 0, 1, 2

EXPORTS = ("swr_fwd", "swr_bwd", "phalanx_mix", "phalanx_mix_bwd", "swr_strerror",
           "swr_last_cuda_error", "swr_set_path", "swr_launch_count", "swr_last_path",
           "swr_set_trace", "swr_decode_step", "phalanx_mix_decode_step",
           "swr_exact_workspace_bytes", "swr_exact_fwd", "swr_exact_bwd",
           "swr_uniform_fwd", "phalanx_layer_mix", "phalanx_layer_mix_bwd",
           "phalanx_layer_workspace_bytes")


class SwrError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.swr_strerror(status).decode()
        if status == 6:
            msg += " -- " + _lib.swr_last_cuda_error().decode()
        super().__init__(f"{where}: {msg}")
        self.status = status


class swr_shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("B", "L", "H", "D", "sx_b", "sx_l", "sx_h", "sa_b", "sa_l", "sa_h")]


class swr_layer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("Gq", "Gk", "sq_b", "sq_l", "sq_h", "sk_b", "sk_l", "sk_h")] + [
                    ("logit_a", ctypes.c_int32), ("logit_k", ctypes.c_int32),
                    ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_2512_13921_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    S = swr_shape
    I = ctypes.c_int
    lib.swr_fwd.argtypes = [P, P, P, P, P, S, I, P]
    lib.swr_bwd.argtypes = [P, P, P, P, P, P, P, P, S, I, P]
    lib.phalanx_mix.argtypes = [P, P, P, P, P, P, P, S, I, P]
    lib.phalanx_mix_bwd.argtypes = [P, P, P, P, P, P, P, P, P, P, P, P, S, I, P]
    lib.swr_decode_step.argtypes = [P, P, P, P, P, P, ctypes.c_int64, S, I, P]
    lib.phalanx_mix_decode_step.argtypes = [P, P, P, P, P, P, P, P, ctypes.c_int64, S, I, P]
    lib.swr_exact_fwd.argtypes = [P, P, P, P, P, P, ctypes.c_int64, S, I, P]
    lib.swr_exact_bwd.argtypes = [P, P, P, P, P, P, P, P, P, ctypes.c_int64, S, I, P]
    lib.swr_uniform_fwd.argtypes = [P, P, P, I, S, I, P]
    G = swr_layer
    lib.phalanx_layer_mix.argtypes = [P, P, P, P, P, P, P, S, G, I, P]
    lib.phalanx_layer_mix_bwd.argtypes = [P, P, P, P, P, P, P, P, P, P, P, P, S, G, I, P]
    lib.phalanx_layer_workspace_bytes.argtypes = [S, G, I]
    lib.phalanx_layer_workspace_bytes.restype = ctypes.c_int64
    lib.swr_exact_workspace_bytes.argtypes = [S]
    lib.swr_exact_workspace_bytes.restype = ctypes.c_int64
    for f in ("swr_fwd", "swr_bwd", "phalanx_mix", "phalanx_mix_bwd", "swr_decode_step",
              "phalanx_mix_decode_step", "swr_exact_fwd", "swr_exact_bwd", "swr_uniform_fwd",
              "phalanx_layer_mix", "phalanx_layer_mix_bwd"):
        getattr(lib, f).restype = I
    lib.swr_strerror.argtypes = [I]
    lib.swr_strerror.restype = ctypes.c_char_p
    lib.swr_last_cuda_error.argtypes = []
    lib.swr_last_cuda_error.restype = ctypes.c_char_p
    lib.swr_set_path.argtypes = [I]
    lib.swr_set_path.restype = I
    lib.swr_launch_count.argtypes = []
    lib.swr_launch_count.restype = ctypes.c_int64
    lib.swr_last_path.argtypes = []
    lib.swr_last_path.restype = I
    lib.swr_set_trace.argtypes = [P, ctypes.c_int64]
    lib.swr_set_trace.restype = None
    return lib


_lib = _load()


def _check(st: int, where: str):
    if st != 0:
        raise SwrError(st, where)


def swr_fwd(u, a, x, carry_in, carry_out, shape, dtype, stream):
    _check(_lib.swr_fwd(u, a, x, carry_in, carry_out, shape, dtype, stream), "swr_fwd")


def swr_bwd(u, a, dx, du, da, carry_in, mu_in, mu_out, shape, dtype, stream):
    _check(_lib.swr_bwd(u, a, dx, du, da, carry_in, mu_in, mu_out, shape, dtype, stream), "swr_bwd")


def phalanx_mix(q, k, v, a, y, carry_in, carry_out, shape, dtype, stream):
    _check(_lib.phalanx_mix(q, k, v, a, y, carry_in, carry_out, shape, dtype, stream), "phalanx_mix")


def phalanx_mix_bwd(q, k, v, a, dy, dq, dk, dv, da, carry_in, mu_in, mu_out, shape, dtype, stream):
    _check(_lib.phalanx_mix_bwd(q, k, v, a, dy, dq, dk, dv, da, carry_in, mu_in, mu_out, shape,
                                dtype, stream), "phalanx_mix_bwd")


def set_path(path: int) -> int:
    return _lib.swr_set_path(path)


def get_path() -> int:
    """This thread's kernel-family selector (read by setting it and restoring it)."""
    prev = _lib.swr_set_path(SWR_PATH_AUTO)
    _lib.swr_set_path(prev)
    return prev


def launch_count() -> int:
    return _lib.swr_launch_count()


def last_path() -> int:
    return _lib.swr_last_path()


def set_trace(ptr, n: int) -> None:
    """Diagnostics: per-item pipeline timestamps of CTA 0 into device buffer `ptr`."""
    _lib.swr_set_trace(ptr, n)


def raw_status(fn: str, *args) -> int:
    """Call an entry point and return its status code without raising (tests)."""
    return getattr(_lib, fn)(*args)


def swr_decode_step(u, a, x, w_state, v_state, g_state, pos, shape, dtype, stream):
    _check(_lib.swr_decode_step(u, a, x, w_state, v_state, g_state, pos, shape, dtype, stream),
           "swr_decode_step")


def phalanx_mix_decode_step(q, k, v, a, y, w_state, v_state, g_state, pos, shape, dtype, stream):
    _check(_lib.phalanx_mix_decode_step(q, k, v, a, y, w_state, v_state, g_state, pos, shape, dtype,
                                        stream), "phalanx_mix_decode_step")


def swr_exact_workspace_bytes(shape) -> int:
    return _lib.swr_exact_workspace_bytes(shape)


def swr_exact_fwd(u, a, x, carry_in, carry_out, workspace, workspace_bytes, shape, dtype, stream):
    _check(_lib.swr_exact_fwd(u, a, x, carry_in, carry_out, workspace, workspace_bytes, shape, dtype,
                              stream), "swr_exact_fwd")


def swr_exact_bwd(u, a, dx, du, da, carry_in, mu_in, mu_out, workspace, workspace_bytes, shape, dtype,
                  stream):
    _check(_lib.swr_exact_bwd(u, a, dx, du, da, carry_in, mu_in, mu_out, workspace, workspace_bytes,
                              shape, dtype, stream), "swr_exact_bwd")


def swr_uniform_fwd(u, a, x, k, shape, dtype, stream):
    _check(_lib.swr_uniform_fwd(u, a, x, k, shape, dtype, stream), "swr_uniform_fwd")


def phalanx_layer_mix(q, zk, v, za, y, carry_in, carry_out, shape, layer, dtype, stream):
    _check(_lib.phalanx_layer_mix(q, zk, v, za, y, carry_in, carry_out, shape, layer, dtype, stream),
           "phalanx_layer_mix")


def phalanx_layer_mix_bwd(q, zk, v, za, dy, dq, dzk, dv, dza, carry_in, mu_in, mu_out, shape, layer,
                          dtype, stream):
    _check(_lib.phalanx_layer_mix_bwd(q, zk, v, za, dy, dq, dzk, dv, dza, carry_in, mu_in, mu_out, shape,
                                      layer, dtype, stream), "phalanx_layer_mix_bwd")


def phalanx_layer_workspace_bytes(shape, layer, dtype) -> int:
    return _lib.phalanx_layer_workspace_bytes(shape, layer, dtype)

"""fp64 CPU oracle for SWR (jagged window, ell = 16) and the Phalanx double-gated mixer.

TEST INFRASTRUCTURE ONLY: importable from tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs.  Never imported by the
product package ``paper_2512_13921_b200``.

* ``swr_fwd`` / ``swr_bwd`` call the plain C loops of ``oracle/swr_oracle.c``
  (the jagged-window definition, and its literal
  reverse mode).
* ``mix_fwd`` / ``mix_bwd`` compose them with elementwise numpy exactly in the
  order the paper writes the Phalanx mixer:
      u_hat = k * v           (pre-gate)
      x     = SWR(u_hat)      (Eq. truncated_factorization via B2P)
      y     = q * x + v       (post-gate with residual)
  and the backward is the chain rule of those three lines (R13).

All arrays are fp64 numpy, d-tensors [B, L, H, D], decays [B, L, H],
carries [B, H, D].
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "swr_oracle.c")
_LIB = os.path.join(_HERE, "libswr_oracle.so")
_lib = None

ELL = 16


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
             "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.swr_oracle_fwd.argtypes = [dp, dp, dp, dp, dp, i64, i64, i64, i64, ctypes.c_int]
        lib.swr_oracle_fwd.restype = ctypes.c_int
        lib.swr_oracle_bwd.argtypes = [dp, dp, dp, dp, dp, dp, dp, dp, i64, i64, i64, i64, ctypes.c_int]
        lib.swr_oracle_bwd.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f64(x):
    return None if x is None else np.ascontiguousarray(x, dtype=np.float64)


def _ptr(x):
    return None if x is None else x.ctypes.data_as(ctypes.c_void_p)


def _check(u, a):
    if u.ndim != 4 or a.ndim != 3 or a.shape != u.shape[:3]:
        raise ValueError(f"shape mismatch: u {u.shape}, a {a.shape}")


last_threads = 0  # threads used by the most recent call (reported by bench.py)


def swr_fwd(u, a, carry_in=None, carry_out=False, threads: int = 0):
    """x~ = L~ u (jagged window).  Returns x, or (x, carry_out) if carry_out=True."""
    global last_threads
    u, a, carry_in = _f64(u), _f64(a), _f64(carry_in)
    _check(u, a)
    B, L, H, D = u.shape
    x = np.empty_like(u)
    co = np.empty((B, H, D)) if carry_out else None
    last_threads = _load().swr_oracle_fwd(_ptr(u), _ptr(a), _ptr(x), _ptr(carry_in), _ptr(co),
                                          B, L, H, D, threads)
    return (x, co) if carry_out else x


def swr_bwd(u, a, G, carry_in=None, mu_in=None, threads: int = 0):
    """Reverse mode of swr_fwd.  Returns (du, da, mu_out); mu_out = dLoss/dcarry_in."""
    global last_threads
    u, a, G, carry_in, mu_in = _f64(u), _f64(a), _f64(G), _f64(carry_in), _f64(mu_in)
    _check(u, a)
    B, L, H, D = u.shape
    du = np.empty_like(u)
    da = np.empty_like(a)
    mu_out = np.empty((B, H, D))
    last_threads = _load().swr_oracle_bwd(_ptr(u), _ptr(a), _ptr(G), _ptr(du), _ptr(da),
                                          _ptr(carry_in), _ptr(mu_in), _ptr(mu_out),
                                          B, L, H, D, threads)
    return du, da, mu_out


def mix_fwd(q, k, v, a, carry_in=None, carry_out=False, threads: int = 0):
    """Phalanx double-gated mixer."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    u_hat = k * v                                      # pre-gate
    r = swr_fwd(u_hat, a, carry_in, carry_out, threads)
    x = r[0] if carry_out else r
    y = q * x + v                                      # post-gate with residual
    return (y, r[1]) if carry_out else y


def mix_bwd(q, k, v, a, dy, carry_in=None, mu_in=None, threads: int = 0):
    """Chain rule of mix_fwd.  Returns (dq, dk, dv, da, mu_out)."""
    q, k, v, dy = _f64(q), _f64(k), _f64(v), _f64(dy)
    u_hat = k * v
    x = swr_fwd(u_hat, a, carry_in, False, threads)
    dq = dy * x
    G = dy * q
    du_hat, da, mu_out = swr_bwd(u_hat, a, G, carry_in, mu_in, threads)
    dk = du_hat * v
    dv = du_hat * k + dy
    return dq, dk, dv, da, mu_out


def swr_decode(u, a, carry_in=None):
    """Recurrence-mode decoding ("decoded in recurrence mode"; SURVEY 8(f)
    NEXT-3), one token at a time in fp64.  Per (b, h) the state is the local state w
    of the current block (Pass I restarted at each block start, L_t excludes
    a_t[0]), the carrier v = w_{t-1}[15] of the previous block and
    g = a_t[0] ... a_t[i]; each token's output is Pass II, x = w + g v
    (P:1478), with v_{-1} = carry_in or 0.  Returns x for all tokens.
    Pinned against swr_fwd (the jagged-window definition) in tests/test_oracle.py."""
    u, a = _f64(u), _f64(a)
    _check(u, a)
    B, L, H, D = u.shape
    w = np.zeros((B, H, D)) if carry_in is None else _f64(carry_in).copy()
    v = np.zeros((B, H, D))
    g = np.ones((B, H))
    x = np.empty_like(u)
    for n in range(L):
        an = a[:, n, :]
        if n % ELL == 0:        # block start: the finished block's end state is the carrier
            v = w
            g = an.copy()
            w = u[:, n].copy()
        else:
            g = g * an
            w = an[..., None] * w + u[:, n]
        x[:, n] = w + g[..., None] * v
    return x


def mix_decode(q, k, v, a, carry_in=None):
    """Phalanx mixer decoded token by token: u^ = k v, y = q x~ + v."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    return q * swr_decode(k * v, a, carry_in) + v


def linrec_fwd(u, a, carry_in=None):
    """The untruncated linear recurrence, Eq. 2.1: x_n = a_n x_{n-1} + u_n
    with x_{-1} = carry_in (or 0), one token at a time in fp64 -- the reference for
    the exact full-range mode (Alg. 2).  Returns (x, x_{L-1})."""
    u, a = _f64(u), _f64(a)
    _check(u, a)
    B, L, H, D = u.shape
    s = np.zeros((B, H, D)) if carry_in is None else _f64(carry_in).copy()
    x = np.empty_like(u)
    for n in range(L):
        s = a[:, n, :, None] * s + u[:, n]
        x[:, n] = s
    return x, s


def linrec_bwd(u, a, G, carry_in=None, mu_in=None):
    """Reverse mode of linrec_fwd, written out token by token in fp64: lambda_n =
    G_n + a_{n+1} lambda_{n+1} (lambda_{L-1} also receives mu_in = dLoss/dx_{L-1}),
    du = lambda, da_n = sum_c lambda_n x_{n-1} (x_{-1} = carry_in), mu_out = a_0 lambda_0.
    Returns (du, da, mu_out).  Pinned by finite differences in tests/test_oracle.py."""
    u, a, G = _f64(u), _f64(a), _f64(G)
    _check(u, a)
    B, L, H, D = u.shape
    x, _ = linrec_fwd(u, a, carry_in)
    x0 = np.zeros((B, H, D)) if carry_in is None else _f64(carry_in)
    du = np.empty_like(u)
    da = np.empty_like(a)
    lam = np.zeros((B, H, D)) if mu_in is None else _f64(mu_in).copy()
    for n in range(L - 1, -1, -1):
        if n < L - 1:
            lam = a[:, n + 1, :, None] * lam
        lam = lam + G[:, n]
        du[:, n] = lam
        xprev = x[:, n - 1] if n > 0 else x0
        da[:, n] = np.sum(lam * xprev, axis=-1)
    mu_out = a[:, 0, :, None] * lam if L > 0 else np.zeros((B, H, D))
    return du, da, mu_out


def uniform_fwd(u, a, k):
    """Uniform-window recurrence, Eq. banded_L: x = (I + AZ + ... +
    (AZ)^{k-1}) u, by the paper's early-stopped Kogge-Stone -- log2 k doubling stages
    X_n <- X_n + A_n X_{n-s}, A_n <- A_n A_{n-s} (s = 1, 2, 4, ...), starting from
    X = u, A = a, with X_{<0} = 0.  k a power of two.  fp64."""
    u, a = _f64(u), _f64(a)
    _check(u, a)
    if k < 1 or k & (k - 1):
        raise ValueError("k must be a power of two")
    X = u.copy()
    A = a.copy()
    s = 1
    while s < k:
        Xs = np.zeros_like(X)
        As = np.zeros_like(A)
        Xs[:, s:] = X[:, :-s] if s < X.shape[1] else 0.0
        As[:, s:] = A[:, :-s] if s < A.shape[1] else 0.0
        X = X + A[..., None] * Xs
        A = A * As
        s *= 2
    return X


# ---------------------------------------------------------------------------
# The Phalanx layer around the mixer
# ---------------------------------------------------------------------------
def sigmoid(z):
    """sigma(z) = 1 / (1 + e^-z), the featurization's bounding activation for the
    recurrence coefficient a = sigma(W u) and the key-like gate k = sigma(K u)
    (P:1562).  fp64."""
    z = _f64(z)
    return 1.0 / (1.0 + np.exp(-z))


def expand_groups(t, H):
    """Gate sharing across heads ("within each group, multiple heads
    share the same gate parameters"; 8 groups for K and Q): a [B, L, G, D]
    group tensor seen by H heads, head h reading group h // (H / G) (contiguous
    head groups, reading R18).  Returns [B, L, H, D]."""
    t = _f64(t)
    G = t.shape[2]
    if H % G:
        raise ValueError(f"{G} groups do not divide {H} heads")
    return np.repeat(t, H // G, axis=2)


def group_sum(t, G):
    """Adjoint of expand_groups: sum the H per-head gradients of each group."""
    t = _f64(t)
    B, L, H, D = t.shape
    return t.reshape(B, L, G, H // G, D).sum(axis=3)


def layer_mix_fwd(q, zk, v, za, carry_in=None, carry_out=False, threads: int = 0):
    """Phalanx mixer fed by the featurization outputs:
        a = sigma(za)                   [B, L, H]     recurrence coefficient logits
        k = sigma(zk)                   [B, L, Gk, D] key-like gate logits, Gk groups
        q                               [B, L, Gq, D] query-like gate, Gq groups
        v                               [B, L, H, D]
        y = q_g (.) SWR_a(k_g (.) v) + v          (g = the head's group)
    Returns y (or (y, carry_out))."""
    v = _f64(v)
    H = v.shape[2]
    a = sigmoid(za)
    k = expand_groups(sigmoid(zk), H)
    qh = expand_groups(q, H)
    return mix_fwd(qh, k, v, a, carry_in, carry_out, threads)


def layer_mix_bwd(q, zk, v, za, dy, carry_in=None, mu_in=None, threads: int = 0):
    """Chain rule of layer_mix_fwd.  Returns (dq [B,L,Gq,D], dzk [B,L,Gk,D], dv,
    dza [B,L,H], mu_out): the mixer's per-head gradients (mix_bwd), summed over the
    heads of each group (group_sum), times sigma' = s (1 - s) for the logits."""
    q, zk, v = _f64(q), _f64(zk), _f64(v)
    H = v.shape[2]
    Gq, Gk = q.shape[2], zk.shape[2]
    a = sigmoid(za)
    ks = sigmoid(zk)
    dqh, dkh, dv, da, mu_out = mix_bwd(expand_groups(q, H), expand_groups(ks, H), v, a, dy,
                                       carry_in, mu_in, threads)
    dq = group_sum(dqh, Gq)
    dzk = group_sum(dkh, Gk) * ks * (1.0 - ks)
    dza = da * a * (1.0 - a)
    return dq, dzk, dv, dza, mu_out

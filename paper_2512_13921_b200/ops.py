"""PyTorch-facing entry points (argument marshalling over the C ABI).

PyTorch supplies device memory and the current CUDA stream; every step of the
computation runs in libswr.so kernels.  Tensors must live on a CUDA device and
share one storage dtype (float32 or bfloat16).

Layout copies (the only data movement done here, all by torch, none silent in
effect -- outputs always come back in the caller's logical shape):
  * the ABI takes ONE set of element strides for all d-tensors of a call and
    needs the head dim contiguous, 16-byte aligned pointers and 16-byte strides,
    and non-overlapping outputs.  d-tensors that already share such a layout are
    passed as they are (no copy; outputs get the same strides); otherwise every
    d-tensor of the call is made contiguous first (``_prep``).
  * decays are passed with their own strides unless a stride is 0 over a
    dimension of size > 1 or the tensor overlaps itself (e.g. one decay row
    expanded over heads): then they are made contiguous, so that ``da`` (which
    shares the decays' strides) has one element per (b, l, h).
  * the autograd wrappers hand the upstream gradient to the backward kernel in
    the storage dtype (the ABI has one dtype per call): an fp32 gradient of a
    bf16 layer is rounded once to bf16 (RNE) -- the same rounding the bf16
    forward output already has.
Every such copy or cast is counted (``layout_copies()``), so a caller -- bench.py
asserts it for the timed region -- can check that its tensors pass through as is.
"""
from __future__ import annotations

import torch

from . import _lib

_DT = {torch.float32: _lib.SWR_F32, torch.bfloat16: _lib.SWR_BF16}
_copies = 0  # layout copies / dtype casts made by this module (see the module docstring)


def layout_copies() -> int:
    """Number of operand copies (layout) and gradient casts (dtype) made so far."""
    return _copies


def _count(n=1):
    global _copies
    _copies += n


def _like(t):
    """Output buffer with exactly the strides of `t` (the ABI shares strides across d-tensors)."""
    return torch.empty_strided(t.shape, t.stride(), dtype=t.dtype, device=t.device)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _no_overlap(t):
    """True if no two in-range indices of `t` address the same element (and no
    stride is 0 over a dimension of size > 1)."""
    dims = sorted((st, n) for st, n in zip(t.stride(), t.shape) if n > 1)
    span = 0  # largest offset reachable with the dims of smaller stride
    for st, n in dims:
        if st <= span:
            return False
        span += st * (n - 1)
    return True


def _abi_layout(t):
    """d-tensor layout the ABI accepts as is: D contiguous, 16-byte aligned base
    pointer and strides, non-overlapping."""
    e = t.element_size()
    if t.data_ptr() % 16:
        return False
    if t.is_contiguous():  # fast path: strides are multiples of D
        return (t.shape[3] * e) % 16 == 0
    return (t.stride(3) == 1 and all((t.stride(i) * e) % 16 == 0 for i in range(3)) and _no_overlap(t))


def _prep(*ts):
    """The d-tensors of one call with one shared ABI layout: kept as they are if
    they already share one (same shape and strides, `_abi_layout`), else copied
    to contiguous."""
    ref = ts[0]
    if ref.dim() != 4:
        raise ValueError(f"expected [B, L, H, D] tensors, got shape {tuple(ref.shape)}")
    ok = all(t.shape == ref.shape and t.stride() == ref.stride() for t in ts) and all(
        _abi_layout(t) for t in ts)
    if not ok:
        _count(len(ts))
        ts = tuple(t.contiguous() for t in ts)
    return ts


def _prep_a(a):
    """Decays with strides `da` can share: contiguous copy if `a` overlaps itself
    (a zero stride, e.g. a decay row expanded over heads) or is misaligned."""
    if a.is_contiguous():
        return a
    if a.dim() == 3 and (not _no_overlap(a) or a.data_ptr() % a.element_size()):
        _count()
        return a.contiguous()
    return a


def _grad_as(g, like):
    """Upstream gradient in the operands' storage dtype (counted when it is a cast)."""
    if g.dtype != like.dtype:
        _count()
        return g.to(like.dtype)
    return g


def _carry(t, like):
    if t is None:
        return None
    B, _, H, D = like.shape
    if t.shape != (B, H, D):
        raise ValueError(f"carry must be [B, H, D] = {(B, H, D)}, got {tuple(t.shape)}")
    return t.to(device=like.device, dtype=torch.float32).contiguous()


def _shape(x, a):
    if a.dim() != 3 or tuple(a.shape) != tuple(x.shape[:3]):
        raise ValueError(f"decays must be [B, L, H] = {tuple(x.shape[:3])}, got {tuple(a.shape)}")
    B, L, H, D = x.shape
    sx, sa = x.stride(), a.stride()
    return _lib.swr_shape(B, L, H, D, sx[0], sx[1], sx[2], sa[0], sa[1], sa[2])


def _dtype(*ts):
    dt = ts[0].dtype
    if dt not in _DT:
        raise TypeError(f"unsupported dtype {dt}: use torch.float32 or torch.bfloat16")
    for t in ts:
        if t.dtype != dt:
            raise TypeError("all operands must share one dtype")
        if not t.is_cuda:
            raise ValueError("libswr operates on CUDA tensors only (no CPU fallback)")
        if t.device != ts[0].device:
            raise ValueError(f"all operands must be on one device ({ts[0].device} vs {t.device})")
    return _DT[dt]


def _stream(t):
    return torch.cuda.current_stream(t.device).cuda_stream


class _on:
    """Make t's device current for the call (the ABI launches on the current
    device), skipping the switch when it already is."""
    __slots__ = ("idx", "prev")

    def __init__(self, t):
        self.idx = t.device.index

    def __enter__(self):
        self.prev = torch.cuda.current_device()
        if self.prev != self.idx:
            torch.cuda.set_device(self.idx)

    def __exit__(self, *exc):
        if self.prev != self.idx:
            torch.cuda.set_device(self.prev)


def _new_carry(like):
    B, _, H, D = like.shape
    return torch.empty((B, H, D), device=like.device, dtype=torch.float32)


# ---------------------------------------------------------------------------
# raw forward / backward calls
# ---------------------------------------------------------------------------
def swr_fwd(u, a, carry_in=None, return_carry=False):
    """x~ = L~ u (jagged window, B2P).  Returns x or (x, carry_out)."""
    (u,) = _prep(u)
    a = _prep_a(a)
    dt = _dtype(u, a)
    x = _like(u)
    ci = _carry(carry_in, u)
    co = _new_carry(u) if return_carry else None
    with _on(u):
        _lib.swr_fwd(_ptr(u), _ptr(a), _ptr(x), _ptr(ci), _ptr(co), _shape(u, a), dt, _stream(u))
    return (x, co) if return_carry else x


def swr_bwd(u, a, dx, carry_in=None, mu_in=None):
    """Returns (du, da, mu_out) for loss gradient dx = dLoss/dx~."""
    u, dx = _prep(u, dx)
    a = _prep_a(a)
    dt = _dtype(u, a, dx)
    du = _like(u)
    da = _like(a)
    ci, mi = _carry(carry_in, u), _carry(mu_in, u)
    mo = _new_carry(u)
    with _on(u):
        _lib.swr_bwd(_ptr(u), _ptr(a), _ptr(dx), _ptr(du), _ptr(da), _ptr(ci), _ptr(mi), _ptr(mo),
                     _shape(u, a), dt, _stream(u))
    return du, da, mo


def phalanx_mix(q, k, v, a, carry_in=None, return_carry=False):
    """y = q (.) SWR(k (.) v) + v."""
    q, k, v = _prep(q, k, v)
    a = _prep_a(a)
    dt = _dtype(q, k, v, a)
    y = _like(q)
    ci = _carry(carry_in, q)
    co = _new_carry(q) if return_carry else None
    with _on(q):
        _lib.phalanx_mix(_ptr(q), _ptr(k), _ptr(v), _ptr(a), _ptr(y), _ptr(ci), _ptr(co),
                         _shape(q, a), dt, _stream(q))
    return (y, co) if return_carry else y


def phalanx_mix_bwd(q, k, v, a, dy, carry_in=None, mu_in=None):
    """Returns (dq, dk, dv, da, mu_out)."""
    q, k, v, dy = _prep(q, k, v, dy)
    a = _prep_a(a)
    dt = _dtype(q, k, v, a, dy)
    dq, dk, dv = _like(q), _like(q), _like(q)
    da = _like(a)
    ci, mi = _carry(carry_in, q), _carry(mu_in, q)
    mo = _new_carry(q)
    with _on(q):
        _lib.phalanx_mix_bwd(_ptr(q), _ptr(k), _ptr(v), _ptr(a), _ptr(dy), _ptr(dq), _ptr(dk),
                             _ptr(dv), _ptr(da), _ptr(ci), _ptr(mi), _ptr(mo), _shape(q, a), dt,
                             _stream(q))
    return dq, dk, dv, da, mo


# ---------------------------------------------------------------------------
# the Phalanx layer around the mixer (include/swr.h phalanx_layer_mix; NEXT-1)
# ---------------------------------------------------------------------------
def _prep_group(t, like):
    """A group-shared gate [B, L, G, D] (G divides H): kept if ABI-ready, else copied."""
    B, L, H, D = like.shape
    if t.dim() != 4 or t.shape[0] != B or t.shape[1] != L or t.shape[3] != D or H % t.shape[2]:
        raise ValueError(f"group tensor must be [B, L, G, D] with G dividing H={H}, got {tuple(t.shape)}")
    if not _abi_layout(t):
        _count()
        t = t.contiguous()
    return t


def _layer(q, zk, logit_a, logit_k):
    return _lib.swr_layer(q.shape[2], zk.shape[2], *q.stride()[:3], *zk.stride()[:3],
                          int(bool(logit_a)), int(bool(logit_k)))


def phalanx_layer_mix(q, zk, v, za, carry_in=None, return_carry=False, logit_a=True, logit_k=True):
    """The mixer fed by the featurization:
    a = sigma(za), k = sigma(zk) (logits unless logit_a / logit_k is False), q and
    zk group-shared [B, L, G, D] (head h reads group h // (H / G)),
    y = q_g (.) SWR_a(k_g (.) v) + v.  Returns y or (y, carry_out)."""
    (v,) = _prep(v)
    q, zk = _prep_group(q, v), _prep_group(zk, v)
    za = _prep_a(za)
    dt = _dtype(q, zk, v, za)
    y = _like(v)
    ci = _carry(carry_in, v)
    co = _new_carry(v) if return_carry else None
    with _on(v):
        _lib.phalanx_layer_mix(_ptr(q), _ptr(zk), _ptr(v), _ptr(za), _ptr(y), _ptr(ci), _ptr(co),
                               _shape(v, za), _layer(q, zk, logit_a, logit_k), dt, _stream(v))
    return (y, co) if return_carry else y


def phalanx_layer_mix_bwd(q, zk, v, za, dy, carry_in=None, mu_in=None, logit_a=True, logit_k=True):
    """Returns (dq [B,L,Gq,D], dzk [B,L,Gk,D], dv, dza, mu_out): the logits' gradients
    and the group sums over the heads sharing q and k."""
    v, dy = _prep(v, dy)
    q, zk = _prep_group(q, v), _prep_group(zk, v)
    za = _prep_a(za)
    dt = _dtype(q, zk, v, za, dy)
    dq, dzk, dv, dza = _like(q), _like(zk), _like(v), _like(za)
    ci, mi = _carry(carry_in, v), _carry(mu_in, v)
    mo = _new_carry(v)
    shape, layer = _shape(v, za), _layer(q, zk, logit_a, logit_k)
    nws = _lib.phalanx_layer_workspace_bytes(shape, layer, dt)
    ws = None
    if nws > 0 and _lib.get_path() != _lib.SWR_PATH_FFMA:
        # tensor cores with shared groups: per-head dq / dk scratch, summed per group
        ws = torch.empty(nws, dtype=torch.uint8, device=v.device)
        layer.workspace, layer.workspace_bytes = ws.data_ptr(), nws
    with _on(v):
        _lib.phalanx_layer_mix_bwd(_ptr(q), _ptr(zk), _ptr(v), _ptr(za), _ptr(dy), _ptr(dq), _ptr(dzk),
                                   _ptr(dv), _ptr(dza), _ptr(ci), _ptr(mi), _ptr(mo), shape, layer, dt, _stream(v))
    return dq, dzk, dv, dza, mo


# ---------------------------------------------------------------------------
# autograd wrappers
# ---------------------------------------------------------------------------
class SWRFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, a, carry_in):
        ctx.save_for_backward(u, a, carry_in)
        return swr_fwd(u, a, carry_in)

    @staticmethod
    def backward(ctx, dx):
        u, a, carry_in = ctx.saved_tensors
        du, da, mu_out = swr_bwd(u, a, _grad_as(dx, u), carry_in)
        return du, da, (mu_out if carry_in is not None else None)


class PhalanxMixFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, a, carry_in):
        ctx.save_for_backward(q, k, v, a, carry_in)
        return phalanx_mix(q, k, v, a, carry_in)

    @staticmethod
    def backward(ctx, dy):
        q, k, v, a, carry_in = ctx.saved_tensors
        dq, dk, dv, da, mu_out = phalanx_mix_bwd(q, k, v, a, _grad_as(dy, q), carry_in)
        return dq, dk, dv, da, (mu_out if carry_in is not None else None)


class PhalanxLayerMixFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, zk, v, za, carry_in, logit_a, logit_k):
        ctx.save_for_backward(q, zk, v, za, carry_in)
        ctx.logits = (logit_a, logit_k)
        return phalanx_layer_mix(q, zk, v, za, carry_in, logit_a=logit_a, logit_k=logit_k)

    @staticmethod
    def backward(ctx, dy):
        q, zk, v, za, carry_in = ctx.saved_tensors
        dq, dzk, dv, dza, mu_out = phalanx_layer_mix_bwd(q, zk, v, za, _grad_as(dy, v), carry_in,
                                                         logit_a=ctx.logits[0], logit_k=ctx.logits[1])
        return dq, dzk, dv, dza, (mu_out if carry_in is not None else None), None, None


def layer_mix(q, zk, v, za, carry_in=None, logit_a=True, logit_k=True):
    """Differentiable Phalanx layer mixer (logits in, group-shared q / k)."""
    return PhalanxLayerMixFunction.apply(q, zk, v, za, carry_in, logit_a, logit_k)


def swr(u, a, carry_in=None):
    """Differentiable SWR: x~ = L~ u."""
    return SWRFunction.apply(u, a, carry_in)


def mix(q, k, v, a, carry_in=None):
    """Differentiable Phalanx double-gated mixer."""
    return PhalanxMixFunction.apply(q, k, v, a, carry_in)


def swr_exact_fwd(u, a, carry_in=None, return_carry=False):
    """The untruncated recurrence x_n = a_n x_{n-1} + u_n (Eq. 2.1) by Alg. 2's three
    stages (include/swr.h swr_exact_fwd).  Returns x or (x, carry_out)."""
    (u,) = _prep(u)
    a = _prep_a(a)
    dt = _dtype(u, a)
    x = _like(u)
    ci = _carry(carry_in, u)
    co = _new_carry(u) if return_carry else None
    shape = _shape(u, a)
    nbytes = 2 * _lib.swr_exact_workspace_bytes(shape)
    ws = torch.empty(max(nbytes, 16) // 4, dtype=torch.float32, device=u.device)
    with _on(u):
        _lib.swr_exact_fwd(_ptr(u), _ptr(a), _ptr(x), _ptr(ci), _ptr(co), _ptr(ws), nbytes, shape, dt,
                           _stream(u))
    return (x, co) if return_carry else x


def swr_exact_bwd(u, a, dx, carry_in=None, mu_in=None):
    """Reverse mode of swr_exact_fwd.  Returns (du, da, mu_out)."""
    u, dx = _prep(u, dx)
    a = _prep_a(a)
    dt = _dtype(u, a, dx)
    du = _like(u)
    da = _like(a)
    ci, mi = _carry(carry_in, u), _carry(mu_in, u)
    mo = _new_carry(u)
    shape = _shape(u, a)
    nbytes = 3 * _lib.swr_exact_workspace_bytes(shape)
    ws = torch.empty(max(nbytes, 16) // 4, dtype=torch.float32, device=u.device)
    with _on(u):
        _lib.swr_exact_bwd(_ptr(u), _ptr(a), _ptr(dx), _ptr(du), _ptr(da), _ptr(ci), _ptr(mi), _ptr(mo),
                           _ptr(ws), nbytes, shape, dt, _stream(u))
    return du, da, mo


class LinRecFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, u, a, carry_in):
        ctx.save_for_backward(u, a, carry_in)
        return swr_exact_fwd(u, a, carry_in)

    @staticmethod
    def backward(ctx, dx):
        u, a, carry_in = ctx.saved_tensors
        du, da, mu_out = swr_exact_bwd(u, a, _grad_as(dx, u), carry_in)
        return du, da, (mu_out if carry_in is not None else None)


def swr_exact(u, a, carry_in=None):
    """Differentiable untruncated recurrence (Eq. 2.1), for comparison with swr()."""
    return LinRecFunction.apply(u, a, carry_in)


def swr_uniform_fwd(u, a, k):
    """Uniform window of the k most recent tokens (Eq. banded_L), no carry."""
    (u,) = _prep(u)
    a = _prep_a(a)
    dt = _dtype(u, a)
    x = _like(u)
    with _on(u):
        _lib.swr_uniform_fwd(_ptr(u), _ptr(a), _ptr(x), int(k), _shape(u, a), dt, _stream(u))
    return x


# ---------------------------------------------------------------------------
# recurrence-mode decoding (include/swr.h swr_decode_step)
# ---------------------------------------------------------------------------
class DecodeState:
    """Per-(b, h) decode state: w (local state of the current block), v (carrier
    v_{t-1}), g (decay product since the block start), fp32, and the position of the
    next token.  ``carry_in`` [B, H, D] seeds w before position 0."""

    def __init__(self, B, H, D, device, carry_in=None):
        self.w = torch.zeros((B, H, D), device=device, dtype=torch.float32)
        if carry_in is not None:
            self.w.copy_(carry_in)
        self.v = torch.empty((B, H, D), device=device, dtype=torch.float32)
        self.g = torch.empty((B, H), device=device, dtype=torch.float32)
        self.pos = 0

    def prefill(self, u, a, k=None, v=None):
        """Seed the state from a prompt [B, P, H, D] (mixer: pass k and v, u=None) so
        that decoding continues at position P.  The state depends only on the last
        two blocks (v_{t-1} is block t-1's local end state, w and g restart at each
        block start), so this steps through at most 31 prompt tokens
        with the decode kernel and discards their outputs; the prompt's own outputs
        come from the parallel forward.  A prompt shorter than 16 tokens starts from
        the carry_in this state was built with (call it on a fresh state)."""
        src = u if u is not None else k
        P = src.shape[1]
        t = P // 16
        start = 16 * (t - 1) if t >= 1 else 0
        self.pos = start  # from a block start on, the state no longer depends on its past
        q0 = torch.zeros_like(k[:, 0]) if u is None and P > 0 else None
        for n in range(start, P):
            if u is not None:
                swr_decode_step(u[:, n], a[:, n], self)
            else:  # the output (q = 0) is discarded; u^ = k * v is formed in the kernel
                phalanx_mix_decode_step(q0, k[:, n], v[:, n], a[:, n], self)
        return self


def _dec_shape(x, a, st):
    if x.dim() != 3 or x.stride(2) != 1:
        raise ValueError(f"expected one token [B, H, D] with D contiguous, got {tuple(x.shape)}")
    if a.dim() != 2 or tuple(a.shape) != tuple(x.shape[:2]):
        raise ValueError(f"decays must be [B, H] = {tuple(x.shape[:2])}, got {tuple(a.shape)}")
    if tuple(st.w.shape) != tuple(x.shape) or st.w.device != x.device:
        raise ValueError("decode state does not match the token's shape / device")
    B, H, D = x.shape
    return _lib.swr_shape(B, 1, H, D, x.stride(0), 0, x.stride(1), a.stride(0), 0, a.stride(1))


def swr_decode_step(u, a, state):
    """x~ of the next token: u [B, H, D], a [B, H]; advances `state` (a DecodeState)."""
    dt = _dtype(u, a)
    u = u.contiguous()  # the ABI shares (sx_b, sx_h) between u and x
    x = torch.empty(u.shape, dtype=u.dtype, device=u.device)
    with _on(u):
        _lib.swr_decode_step(_ptr(u), _ptr(a), _ptr(x), _ptr(state.w), _ptr(state.v), _ptr(state.g),
                             state.pos, _dec_shape(u, a, state), dt, _stream(u))
    state.pos += 1
    return x


def phalanx_mix_decode_step(q, k, v, a, state):
    """y of the next token, y = q * x~ + v with u^ = k * v."""
    dt = _dtype(q, k, v, a)
    q, k, v = (t.contiguous() for t in (q, k, v))
    y = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    with _on(q):
        _lib.phalanx_mix_decode_step(_ptr(q), _ptr(k), _ptr(v), _ptr(a), _ptr(y), _ptr(state.w),
                                     _ptr(state.v), _ptr(state.g), state.pos, _dec_shape(q, a, state),
                                     dt, _stream(q))
    state.pos += 1
    return y

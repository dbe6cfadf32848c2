"""Pins for the fp64 oracle (oracle/): each test checks it against something other
than itself -- values the paper (or SPEC's hand-derived examples) print, closed
forms, the untruncated recurrence where the paper says the window is exact,
finite differences, a dense operator assembled entrywise from explicit
products, and the structural claims of Eq. block_bidiagonal.

Citations: P:n = /root/reference/PAPER.md line n (section / equation named).
"""
import numpy as np
import pytest

import oracle
from conftest import load_golden

ELL = 16


# --------------------------------------------------------------------------
# independent constructions used as pins
# --------------------------------------------------------------------------
def dense_jagged(a):
    """L~ assembled entrywise (P:126-128 entries L_ij = a_{i:j+1}, support of
    Eq. block_bidiagonal): row n of block t keeps columns from the
    start of block t-1 (0 for t = 0) through n.  Products by np.prod, not a
    recurrence."""
    L = len(a)
    M = np.zeros((L, L))
    for n in range(L):
        t = n // ELL
        lo = 0 if t == 0 else ELL * (t - 1)
        for j in range(lo, n + 1):
            M[n, j] = np.prod(a[j + 1:n + 1])  # empty product = 1
    return M


def dense_carry(a):
    """Response of L~ to the folded initial state: x_n += a_{n:1} x_0 in block 0."""
    L = len(a)
    c = np.zeros(L)
    for n in range(min(L, ELL)):
        c[n] = np.prod(a[:n + 1])
    return c


def full_recurrence(a, u, x0=None):
    """Eq. 2.1 without truncation, one token at a time."""
    x = np.zeros_like(u)
    s = np.zeros(u.shape[1]) if x0 is None else x0.copy()
    for n in range(len(a)):
        s = a[n] * s + u[n]
        x[n] = s
    return x


def rand_problem(B, L, H, D, seed, lo=0.0, hi=1.0):
    r = np.random.default_rng(seed)
    u = r.standard_normal((B, L, H, D))
    a = r.uniform(lo, hi, (B, L, H))
    G = r.standard_normal((B, L, H, D))
    c = r.standard_normal((B, H, D))
    m = r.standard_normal((B, H, D))
    return u, a, G, c, m


def normwise(x, ref):
    return np.max(np.abs(x - ref)) / max(np.max(np.abs(ref)), 1e-300)


# --------------------------------------------------------------------------
# golden worked examples
# --------------------------------------------------------------------------
def test_golden_sequential_example():
    g = load_golden("recurrence_examples.txt")["seq_example"]
    a = np.array(g["a"]).reshape(1, -1, 1)
    u = np.array(g["u"]).reshape(1, -1, 1, 1)
    x = oracle.swr_fwd(u, a)
    assert np.array_equal(x.reshape(-1), np.array(g["x"]))


def test_golden_transfer_operator_columns():
    g = load_golden("recurrence_examples.txt")["transfer_example"]
    a = np.array(g["a"])
    n = len(a)
    Lref = np.array(g["L"])
    cols = []
    for j in range(n):
        e = np.zeros((1, n, 1, 1))
        e[0, j, 0, 0] = 1.0
        cols.append(oracle.swr_fwd(e, a.reshape(1, n, 1)).reshape(n))
    assert np.array_equal(np.stack(cols, axis=1), Lref)


# --------------------------------------------------------------------------
# P1 dense operator, with and without carry_in, ragged lengths
# --------------------------------------------------------------------------
@pytest.mark.parametrize("L", [1, 15, 16, 17, 32, 33, 64, 77])
def test_forward_equals_dense_jagged_operator(L):
    B, H, D = 2, 3, 5
    u, a, _, c, _ = rand_problem(B, L, H, D, seed=L)
    x = oracle.swr_fwd(u, a)
    xc, co = oracle.swr_fwd(u, a, carry_in=c, carry_out=True)
    for b in range(B):
        for h in range(H):
            M = dense_jagged(a[b, :, h])
            ref = M @ u[b, :, h, :]
            np.testing.assert_allclose(x[b, :, h, :], ref, rtol=1e-12, atol=1e-13)
            refc = ref + np.outer(dense_carry(a[b, :, h]), c[b, h])
            np.testing.assert_allclose(xc[b, :, h, :], refc, rtol=1e-12, atol=1e-13)
            # carry_out: local end state of the last block, v_b of Alg. 4
            t_last = (L - 1) // ELL
            lo = ELL * t_last
            v = sum(np.prod(a[b, n + 1:L, h]) * u[b, n, h] for n in range(lo, L))
            np.testing.assert_allclose(co[b, h], v, rtol=1e-12, atol=1e-13)


def test_support_is_jagged_block_bidiagonal():
    """Eq. block_bidiagonal and the lag claims of P:1303: every row
    of a block t >= 1 sees lags 0..i+16, so all rows cover lag <= ell and the
    longest reach is 2*ell - 1."""
    L = 80
    a = np.random.default_rng(3).uniform(0.5, 1.0, L)
    cols = []
    for j in range(L):
        e = np.zeros((1, L, 1, 1))
        e[0, j, 0, 0] = 1.0
        cols.append(oracle.swr_fwd(e, a.reshape(1, L, 1)).reshape(L))
    M = np.stack(cols, axis=1)
    for n in range(L):
        nz = np.nonzero(M[n])[0]
        lags = n - nz
        t, i = divmod(n, ELL)
        expect_max = i if t == 0 else i + ELL
        assert lags.min() == 0 and lags.max() == expect_max
        assert len(nz) == expect_max + 1  # contiguous support
    maxlag = max((n - np.nonzero(M[n])[0]).max() for n in range(L))
    assert maxlag == 2 * ELL - 1


# --------------------------------------------------------------------------
# P2 constant-decay closed form
# --------------------------------------------------------------------------
@pytest.mark.parametrize("rho", [0.0, 0.5, 0.9, 1.0])
def test_constant_decay_closed_form(rho):
    L = 70
    a = np.full((1, L, 1), rho)
    u = np.ones((1, L, 1, 1))
    x = oracle.swr_fwd(u, a).reshape(L)
    n = np.arange(L)
    t, i = n // ELL, n % ELL
    W = np.where(t == 0, i + 1, i + 1 + ELL)   # window length of token n
    ref = W.astype(float) if rho == 1.0 else (1 - rho ** W) / (1 - rho)
    np.testing.assert_allclose(x, ref, rtol=1e-13)
    # general input: x_n = sum_{k<W_n} rho^k u_{n-k}
    r = np.random.default_rng(1)
    u2 = r.standard_normal((1, L, 1, 1))
    x2 = oracle.swr_fwd(u2, a).reshape(L)
    ref2 = np.array([sum(rho ** k * u2[0, m - k, 0, 0] for k in range(W[m])) for m in range(L)])
    np.testing.assert_allclose(x2, ref2, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------
# P3 exact on the first 2*ell steps and special cases
# --------------------------------------------------------------------------
@pytest.mark.parametrize("L", [1, 5, 16, 31, 32])
def test_two_blocks_equal_full_recurrence(L):
    u, a, _, c, _ = rand_problem(1, L, 1, 4, seed=10 + L)
    x = oracle.swr_fwd(u, a)
    ref = full_recurrence(a[0, :, 0], u[0, :, 0, :])
    np.testing.assert_allclose(x[0, :, 0, :], ref, rtol=1e-13, atol=1e-14)
    # carry_in is the carrier of a virtual block -1 (v_0 of Alg. 4 made an input,
    # P:1476): inside block 0 it is the x_0 fold of P:116 ...
    xc = oracle.swr_fwd(u, a, carry_in=c)
    n0 = min(L, ELL)
    ref0 = full_recurrence(a[0, :n0, 0], u[0, :n0, 0, :], x0=c[0, 0])
    np.testing.assert_allclose(xc[0, :n0, 0, :], ref0, rtol=1e-13, atol=1e-14)
    # ... and, as the block bidiagonal structure requires, block 1 never
    # sees it (its window restarts from zero at token 0).
    np.testing.assert_array_equal(xc[0, n0:], x[0, n0:])


def test_first_2ell_exact_then_truncated():
    L = 96
    u, a, _, _, _ = rand_problem(1, L, 1, 2, seed=4, lo=0.6, hi=1.0)
    x = oracle.swr_fwd(u, a)[0, :, 0, :]
    ref = full_recurrence(a[0, :, 0], u[0, :, 0, :])
    np.testing.assert_allclose(x[:2 * ELL], ref[:2 * ELL], rtol=1e-13, atol=1e-14)
    assert np.max(np.abs(x[2 * ELL:] - ref[2 * ELL:])) > 1e-6  # window truncation is active


def test_zero_decay_is_identity_and_one_decay_is_windowed_sum():
    u, _, _, _, _ = rand_problem(2, 50, 2, 3, seed=5)
    assert np.array_equal(oracle.swr_fwd(u, np.zeros((2, 50, 2))), u)
    x = oracle.swr_fwd(u, np.ones((2, 50, 2)))
    for n in range(50):
        t = n // ELL
        lo = 0 if t == 0 else ELL * (t - 1)
        np.testing.assert_allclose(x[:, n], u[:, lo:n + 1].sum(axis=1), rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------
# P4 finite differences for the backward (du, da, mu_out) incl. carry_in/mu_in
# --------------------------------------------------------------------------
def _loss(u, a, G, c, m):
    x, co = oracle.swr_fwd(u, a, carry_in=c, carry_out=True)
    return float(np.sum(G * x) + np.sum(m * co))


@pytest.mark.parametrize("L", [37, 48])
def test_backward_matches_finite_differences(L):
    B, H, D = 1, 2, 3
    u, a, G, c, m = rand_problem(B, L, H, D, seed=20 + L, lo=0.2, hi=1.0)
    du, da, mu_out = oracle.swr_bwd(u, a, G, carry_in=c, mu_in=m)
    h = 1e-6

    def fd(arr, setter):
        g = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            p = arr.copy(); p[idx] += h
            q = arr.copy(); q[idx] -= h
            g[idx] = (setter(p) - setter(q)) / (2 * h)
        return g

    fdu = fd(u, lambda p: _loss(p, a, G, c, m))
    fda = fd(a, lambda p: _loss(u, p, G, c, m))
    fdc = fd(c, lambda p: _loss(u, a, G, p, m))
    assert normwise(du, fdu) < 1e-6
    assert normwise(da, fda) < 1e-6
    assert normwise(mu_out, fdc) < 1e-6


# --------------------------------------------------------------------------
# P5 transpose identity du = L~^T G and the time-reversal form (Appendix A.2)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("L", [16, 40, 64])
def test_du_is_transpose_of_dense_operator(L):
    u, a, G, _, _ = rand_problem(1, L, 2, 4, seed=30 + L)
    du, _, _ = oracle.swr_bwd(u, a, G)
    for h in range(2):
        M = dense_jagged(a[0, :, h])
        np.testing.assert_allclose(du[0, :, h, :], M.T @ G[0, :, h, :], rtol=1e-12, atol=1e-12)


def test_mu_out_is_a0_times_lambda0():
    """mu_out = dLoss/dx_0 = a[0] * (L_1^T G_1)[0] (Appendix A.4)."""
    L = 48
    u, a, G, _, _ = rand_problem(1, L, 1, 3, seed=7)
    _, _, mu = oracle.swr_bwd(u, a, G)
    M = dense_jagged(a[0, :, 0])
    lam0 = (M[:ELL, :ELL].T @ G[0, :ELL, 0, :])[0]
    np.testing.assert_allclose(mu[0, 0], a[0, 0, 0] * lam0, rtol=1e-12)


# --------------------------------------------------------------------------
# P6 locality and P7 linearity
# --------------------------------------------------------------------------
def _blocks_changed(x0, x1, axis_len):
    d = np.abs(x1 - x0).reshape(axis_len // ELL, -1).max(axis=1)
    return set(np.nonzero(d > 0)[0].tolist())


def test_locality_of_forward_and_backward():
    L, D = 96, 4
    u, a, G, _, _ = rand_problem(1, L, 1, D, seed=8, lo=0.3, hi=1.0)
    x0 = oracle.swr_fwd(u, a)[0, :, 0]
    du0, da0, _ = oracle.swr_bwd(u, a, G)
    sl = slice(2 * ELL, 3 * ELL)
    u1 = u.copy(); u1[0, sl] += 1.0
    x1 = oracle.swr_fwd(u1, a)[0, :, 0]
    _, da1, _ = oracle.swr_bwd(u1, a, G)
    assert _blocks_changed(x0, x1, L) == {2, 3}
    assert _blocks_changed(da0[0, :, 0], da1[0, :, 0], L) == {2, 3}
    G1 = G.copy(); G1[0, sl] += 1.0
    du1, da1, _ = oracle.swr_bwd(u, a, G1)
    assert _blocks_changed(du0[0, :, 0], du1[0, :, 0], L) == {1, 2}
    assert _blocks_changed(da0[0, :, 0], da1[0, :, 0], L) == {1, 2}
    a1 = a.copy(); a1[0, sl] *= 0.5
    x1 = oracle.swr_fwd(u, a1)[0, :, 0]
    du1, da1, _ = oracle.swr_bwd(u, a1, G)
    assert _blocks_changed(x0, x1, L) == {2, 3}
    assert _blocks_changed(du0[0, :, 0], du1[0, :, 0], L) == {1, 2}
    assert _blocks_changed(da0[0, :, 0], da1[0, :, 0], L) == {1, 2, 3}


def test_linearity():
    u1, a, _, _, _ = rand_problem(1, 64, 2, 3, seed=9)
    u2, _, _, _, _ = rand_problem(1, 64, 2, 3, seed=10)
    lhs = oracle.swr_fwd(2.5 * u1 - 0.75 * u2, a)
    rhs = 2.5 * oracle.swr_fwd(u1, a) - 0.75 * oracle.swr_fwd(u2, a)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------
# P8 stitching: shards joined by carry_out -> carry_in (forward) and
# mu_out -> mu_in (backward) reproduce the single run bit for bit
# --------------------------------------------------------------------------
@pytest.mark.parametrize("P", [2, 4])
def test_sequence_parallel_stitching_is_bitwise(P):
    B, L, H, D = 2, 256, 2, 3
    u, a, G, _, _ = rand_problem(B, L, H, D, seed=11)
    x = oracle.swr_fwd(u, a)
    du, da, _ = oracle.swr_bwd(u, a, G)
    S = L // P
    sh = [slice(p * S, (p + 1) * S) for p in range(P)]
    xs, carries = [], [None]
    for p in range(P):
        xp, co = oracle.swr_fwd(u[:, sh[p]], a[:, sh[p]], carry_in=carries[-1], carry_out=True)
        xs.append(xp); carries.append(co)
    assert np.array_equal(np.concatenate(xs, axis=1), x)
    mus = [None] * (P + 1)
    dus, das = [None] * P, [None] * P
    for p in reversed(range(P)):
        dus[p], das[p], mus[p] = oracle.swr_bwd(u[:, sh[p]], a[:, sh[p]], G[:, sh[p]],
                                                carry_in=carries[p], mu_in=mus[p + 1])
    assert np.array_equal(np.concatenate(dus, axis=1), du)
    assert np.array_equal(np.concatenate(das, axis=1), da)


def test_thread_count_invariance():
    u, a, G, c, m = rand_problem(3, 70, 5, 4, seed=12)
    x1 = oracle.swr_fwd(u, a, carry_in=c, threads=1)
    x8 = oracle.swr_fwd(u, a, carry_in=c, threads=8)
    assert np.array_equal(x1, x8)
    r1 = oracle.swr_bwd(u, a, G, carry_in=c, mu_in=m, threads=1)
    r8 = oracle.swr_bwd(u, a, G, carry_in=c, mu_in=m, threads=7)
    for p, q in zip(r1, r8):
        assert np.array_equal(p, q)


# --------------------------------------------------------------------------
# Phalanx mixer: dense composition, gate identities, FD
# --------------------------------------------------------------------------
def _mix_problem(B, L, H, D, seed):
    r = np.random.default_rng(seed)
    q = r.standard_normal((B, L, H, D))
    k = 1 / (1 + np.exp(-r.standard_normal((B, L, H, D))))
    v = r.standard_normal((B, L, H, D))
    a = r.uniform(0.1, 1.0, (B, L, H))
    dy = r.standard_normal((B, L, H, D))
    return q, k, v, a, dy


def test_mix_forward_dense_composition():
    q, k, v, a, _ = _mix_problem(1, 50, 2, 3, seed=13)
    y = oracle.mix_fwd(q, k, v, a)
    for h in range(2):
        M = dense_jagged(a[0, :, h])
        ref = q[0, :, h] * (M @ (k[0, :, h] * v[0, :, h])) + v[0, :, h]
        np.testing.assert_allclose(y[0, :, h], ref, rtol=1e-12, atol=1e-12)


def test_mix_gate_identities():
    q, k, v, a, _ = _mix_problem(1, 40, 2, 3, seed=14)
    assert np.array_equal(oracle.mix_fwd(np.zeros_like(q), k, v, a), v)
    assert np.array_equal(oracle.mix_fwd(q, np.zeros_like(k), v, a), v)


def test_mix_backward_matches_finite_differences():
    q, k, v, a, dy = _mix_problem(1, 35, 1, 2, seed=15)
    dq, dk, dv, da, _ = oracle.mix_bwd(q, k, v, a, dy)
    h = 1e-6

    def loss(q_, k_, v_, a_):
        return float(np.sum(dy * oracle.mix_fwd(q_, k_, v_, a_)))

    def fd(arr, f):
        g = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            p = arr.copy(); p[i] += h
            m = arr.copy(); m[i] -= h
            g[i] = (f(p) - f(m)) / (2 * h)
        return g

    assert normwise(dq, fd(q, lambda p: loss(p, k, v, a))) < 1e-6
    assert normwise(dk, fd(k, lambda p: loss(q, p, v, a))) < 1e-6
    assert normwise(dv, fd(v, lambda p: loss(q, k, p, a))) < 1e-6
    assert normwise(da, fd(a, lambda p: loss(q, k, v, p))) < 1e-6


def test_empty_sequence():
    """L = 0: nothing to compute; carry_out and mu_out are zero (no block carries state)."""
    u = np.zeros((2, 0, 3, 4))
    a = np.zeros((2, 0, 3))
    c = np.ones((2, 3, 4))
    x, co = oracle.swr_fwd(u, a, carry_in=c, carry_out=True)
    assert x.shape == u.shape and np.all(co == 0)
    du, da, mo = oracle.swr_bwd(u, a, u, carry_in=c, mu_in=c)
    assert du.shape == u.shape and da.shape == a.shape and np.all(mo == 0)


# --------------------------------------------------------------------------
# recurrence-mode decoding
# --------------------------------------------------------------------------
@pytest.mark.parametrize("L", [1, 15, 16, 17, 50])
def test_decode_equals_dense_jagged_operator(L):
    """Token-by-token decoding reproduces the jagged-window operator (entrywise
    products) including the carry_in fold of block 0, for every prefix length."""
    u, a, _, c, _ = rand_problem(2, L, 3, 4, seed=90 + L)
    x = oracle.swr_decode(u, a, carry_in=c)
    for b in range(2):
        for h in range(3):
            M, cc = dense_jagged(a[b, :, h]), dense_carry(a[b, :, h])
            ref = M @ u[b, :, h] + np.outer(cc, c[b, h])
            assert normwise(x[b, :, h], ref) < 1e-12


def test_decode_equals_parallel_forward_and_mixer():
    u, a, _, c, _ = rand_problem(2, 83, 5, 8, seed=7)
    assert normwise(oracle.swr_decode(u, a, c), oracle.swr_fwd(u, a, carry_in=c)) < 1e-12
    r = np.random.default_rng(8)
    q, k, v = (r.standard_normal(u.shape) for _ in range(3))
    y = oracle.mix_decode(q, k, v, a, carry_in=c)
    assert normwise(y, oracle.mix_fwd(q, k, v, a, carry_in=c)) < 1e-12


# --------------------------------------------------------------------------
# exact full-range recurrence (Eq. 2.1)
# --------------------------------------------------------------------------
def dense_full(a):
    """Lower-triangular L of Eq. 2.1 entrywise: L_nj = a_{j+1} ... a_n."""
    L = len(a)
    M = np.zeros((L, L))
    for n in range(L):
        for j in range(n + 1):
            M[n, j] = np.prod(a[j + 1:n + 1])
    return M


@pytest.mark.parametrize("L", [1, 16, 33, 70])
def test_linrec_equals_dense_full_operator(L):
    u, a, _, c, _ = rand_problem(2, L, 2, 3, seed=500 + L)
    x, last = oracle.linrec_fwd(u, a, carry_in=c)
    for b in range(2):
        for h in range(2):
            ref = dense_full(a[b, :, h]) @ u[b, :, h] + np.outer(np.cumprod(a[b, :, h]), c[b, h])
            assert normwise(x[b, :, h], ref) < 1e-12
    assert np.array_equal(last, x[:, -1])


def test_linrec_constant_decay_closed_form_and_two_block_agreement():
    rho, L = 0.9, 64
    u = np.ones((1, L, 1, 1))
    a = np.full((1, L, 1), rho)
    x, _ = oracle.linrec_fwd(u, a)
    n = np.arange(L)
    assert np.allclose(x[0, :, 0, 0], (1 - rho ** (n + 1)) / (1 - rho), rtol=1e-13, atol=0)
    # on the first two blocks the jagged window is the full recurrence
    u, a, _, _, _ = rand_problem(1, 2 * ELL, 3, 4, seed=5)
    assert normwise(oracle.linrec_fwd(u, a)[0], oracle.swr_fwd(u, a)) < 1e-12


def test_linrec_backward_matches_finite_differences():
    """d/d(u, a, carry_in) of <G, x> + <mu_in, x_{L-1}> by central differences."""
    u, a, G, c, m = rand_problem(1, 37, 2, 3, seed=77, lo=0.3, hi=0.95)

    def loss(u_, a_, c_):
        x, last = oracle.linrec_fwd(u_, a_, carry_in=c_)
        return np.sum(G * x) + np.sum(m * last)

    du, da, mo = oracle.linrec_bwd(u, a, G, carry_in=c, mu_in=m)
    eps = 1e-6
    r = np.random.default_rng(3)
    for _ in range(12):
        idx = tuple(r.integers(0, s) for s in u.shape)
        up, um = u.copy(), u.copy()
        up[idx] += eps
        um[idx] -= eps
        assert abs((loss(up, a, c) - loss(um, a, c)) / (2 * eps) - du[idx]) < 1e-6
        ia = tuple(r.integers(0, s) for s in a.shape)
        ap, am = a.copy(), a.copy()
        ap[ia] += eps
        am[ia] -= eps
        assert abs((loss(u, ap, c) - loss(u, am, c)) / (2 * eps) - da[ia]) < 1e-6
        ic = tuple(r.integers(0, s) for s in c.shape)
        cp, cm = c.copy(), c.copy()
        cp[ic] += eps
        cm[ic] -= eps
        assert abs((loss(u, a, cp) - loss(u, a, cm)) / (2 * eps) - mo[ic]) < 1e-6


# --------------------------------------------------------------------------
# uniform window (Eq. banded_L)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("k", [1, 2, 4, 8, 16, 32])
def test_uniform_equals_dense_banded_operator(k):
    """Early-stopped Kogge-Stone == I + AZ + ... + (AZ)^{k-1} assembled entrywise."""
    u, a, _, _, _ = rand_problem(2, 45, 2, 3, seed=900 + k)
    x = oracle.uniform_fwd(u, a, k)
    for b in range(2):
        for h in range(2):
            full = dense_full(a[b, :, h])
            band = np.tril(full) - np.tril(full, -k)  # lags 0 .. k-1
            assert normwise(x[b, :, h], band @ u[b, :, h]) < 1e-12


def test_uniform_limits():
    u, a, _, _, _ = rand_problem(1, 20, 2, 3, seed=4)
    assert np.array_equal(oracle.uniform_fwd(u, a, 1), u)
    assert normwise(oracle.uniform_fwd(u, a, 32), oracle.linrec_fwd(u, a)[0]) < 1e-12


# --------------------------------------------------------------------------
# the Phalanx layer around the mixer: sigma on the a and k
# logits, group-shared q and k
# --------------------------------------------------------------------------
def test_sigmoid_values():
    """sigma(0) = 1/2, sigma(-z) = 1 - sigma(z), sigma(log(p/(1-p))) = p, sigma(ln 3) = 3/4."""
    z = np.linspace(-30, 30, 121)
    s = oracle.sigmoid(z)
    assert oracle.sigmoid(np.array(0.0)) == 0.5
    np.testing.assert_allclose(oracle.sigmoid(-z), 1.0 - s, rtol=0, atol=1e-15)
    p = np.array([1e-6, 0.1, 0.25, 0.5, 0.8, 0.999])
    np.testing.assert_allclose(oracle.sigmoid(np.log(p / (1 - p))), p, rtol=1e-12)
    np.testing.assert_allclose(oracle.sigmoid(np.log(3.0)), 0.75, rtol=1e-15)


def _layer_problem(B, L, H, Gq, Gk, D, seed):
    r = np.random.default_rng(seed)
    q = r.standard_normal((B, L, Gq, D))
    zk = r.standard_normal((B, L, Gk, D))
    v = r.standard_normal((B, L, H, D))
    za = r.standard_normal((B, L, H))
    dy = r.standard_normal((B, L, H, D))
    return q, zk, v, za, dy


@pytest.mark.parametrize("H,Gq,Gk", [(4, 2, 2), (6, 3, 1), (8, 8, 2), (4, 1, 4)])
def test_layer_forward_dense_per_head(H, Gq, Gk):
    """y[:, :, h] = q[g_q(h)] * (L~(sigma(za_h)) (sigma(zk[g_k(h)]) * v_h)) + v_h with
    g(h) = h // (H / G), written with the entrywise dense jagged operator and
    explicit scalar sigmoids, head by head."""
    import math
    B, L, D = 1, 40, 3
    q, zk, v, za, _ = _layer_problem(B, L, H, Gq, Gk, D, seed=50 + H + Gq)
    y = oracle.layer_mix_fwd(q, zk, v, za)
    for h in range(H):
        gq, gk = h // (H // Gq), h // (H // Gk)
        a = np.array([1.0 / (1.0 + math.exp(-z)) for z in za[0, :, h]])
        k = np.vectorize(lambda z: 1.0 / (1.0 + math.exp(-z)))(zk[0, :, gk])
        M = dense_jagged(a)
        ref = q[0, :, gq] * (M @ (k * v[0, :, h])) + v[0, :, h]
        np.testing.assert_allclose(y[0, :, h], ref, rtol=1e-12, atol=1e-12)


def test_layer_with_one_head_per_group_is_the_mixer():
    """G = H and logits of given gates: the layer mixer is mix_fwd / mix_bwd on the
    gates, with the logit gradients scaled by sigma' = s (1 - s)."""
    q, k, v, a, dy = _mix_problem(2, 45, 3, 4, seed=16)
    k = np.clip(k, 1e-3, 1 - 1e-3)
    a = np.clip(a, 1e-3, 1 - 1e-3)
    zk, za = np.log(k / (1 - k)), np.log(a / (1 - a))
    np.testing.assert_allclose(oracle.layer_mix_fwd(q, zk, v, za), oracle.mix_fwd(q, k, v, a),
                               rtol=1e-10, atol=1e-10)
    dq, dzk, dv, dza, mo = oracle.layer_mix_bwd(q, zk, v, za, dy)
    rq, rk, rv, ra, rmo = oracle.mix_bwd(q, k, v, a, dy)
    np.testing.assert_allclose(dq, rq, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dzk, rk * k * (1 - k), rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(dv, rv, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dza, ra * a * (1 - a), rtol=1e-9, atol=1e-10)
    np.testing.assert_allclose(mo, rmo, rtol=1e-10, atol=1e-10)


def test_layer_backward_matches_finite_differences():
    """Central differences of sum(dy * y) in every group-tensor and logit entry
    (H = 4 heads, 2 q groups, 1 k group, 35 tokens, 2 channels), with carries."""
    B, L, H, Gq, Gk, D = 1, 35, 4, 2, 1, 2
    q, zk, v, za, dy = _layer_problem(B, L, H, Gq, Gk, D, seed=17)
    r = np.random.default_rng(18)
    ci, mi = r.standard_normal((B, H, D)), r.standard_normal((B, H, D))
    dq, dzk, dv, dza, mo = oracle.layer_mix_bwd(q, zk, v, za, dy, carry_in=ci, mu_in=mi)
    h = 1e-6

    def loss(q_, zk_, v_, za_, ci_=ci):
        y, co = oracle.layer_mix_fwd(q_, zk_, v_, za_, carry_in=ci_, carry_out=True)
        return float(np.sum(dy * y) + np.sum(mi * co))

    def fd(arr, f):
        g = np.zeros_like(arr)
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            i = it.multi_index
            p = arr.copy(); p[i] += h
            m = arr.copy(); m[i] -= h
            g[i] = (f(p) - f(m)) / (2 * h)
        return g

    assert normwise(dq, fd(q, lambda p: loss(p, zk, v, za))) < 1e-6
    assert normwise(dzk, fd(zk, lambda p: loss(q, p, v, za))) < 1e-6
    assert normwise(dv, fd(v, lambda p: loss(q, zk, p, za))) < 1e-6
    assert normwise(dza, fd(za, lambda p: loss(q, zk, v, p))) < 1e-6
    assert normwise(mo, fd(ci, lambda p: loss(q, zk, v, za, p))) < 1e-6

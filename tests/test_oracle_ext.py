"""Pins for the oracle's NEXT-1 (gate z, last state) and NEXT-2 (state
passing h0 -> h_last, the paper's future work P:275) extension."""
import numpy as np
import pytest

import oracle
from tests.test_oracle_pins import rand_problem


def _prob(seed, R=2, Dn=3, L=23, N=4, rows=None):
    rng = np.random.default_rng(seed)
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, N, 4, rows)
    u = rng.standard_normal((R, Dn, L))
    z = rng.standard_normal((R, Dn, L))
    h0 = rng.standard_normal((R, Dn, N))
    dh = rng.standard_normal((R, Dn, N))
    return rng, pos, P, u, z, h0, dh


def test_ext_reduces_to_base_bit_exact():
    rng, pos, P, u, z, h0, dh = _prob(1)
    args = (u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    y, _ = oracle.scan_fwd_ext(*args)
    assert np.array_equal(y, oracle.scan_fwd(*args))
    g = oracle.scan_bwd_ext(*args, P["dy"])
    ref = oracle.scan_bwd(*args, P["dy"])
    for k in ("du", "ddt", "dB", "dC"):
        assert np.array_equal(g[k], ref[k]), k
    for k in ("dA", "dD", "ddt_bias"):
        np.testing.assert_allclose(g[k], ref[k], rtol=1e-13, atol=1e-13)


def test_gate_closed_forms():
    rng, pos, P, u, z, h0, dh = _prob(2)
    args = (u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    y, _ = oracle.scan_fwd_ext(*args)
    zero = np.zeros_like(u)
    out, _ = oracle.scan_fwd_ext(*args, z=zero)
    assert np.all(out == 0)                      # silu(0) = 0
    g = oracle.scan_bwd_ext(*args, P["dy"], z=zero)
    np.testing.assert_allclose(g["dz"], P["dy"] * y * 0.5, rtol=1e-13, atol=1e-14)
    assert np.all(g["du"] == 0) and np.all(g["dB"] == 0)


@pytest.mark.parametrize("seed", range(3))
def test_ext_finite_differences(seed):
    rng, pos, P, u, z, h0, dh = _prob(10 + seed, R=2, Dn=2, L=9, N=2)
    pos[:, 0] = np.array([3, 0])  # row 0 continues a sequence (uses h0), row 1 starts one
    pos[0, 1:4] = [4, 5, 6]
    dout = rng.standard_normal(u.shape)
    X = dict(u=u, dt=P["dt"], A=P["A"], B=P["B"], C=P["C"], D=P["D"], dt_bias=P["dt_bias"],
             z=z, h0=h0)

    def loss(k):
        out, hl = oracle.scan_fwd_ext(k["u"], k["dt"], k["A"], k["B"], k["C"], k["D"],
                                      k["dt_bias"], pos, z=k["z"], h0=k["h0"])
        return float(np.sum(out * dout) + np.sum(hl * dh))

    g = oracle.scan_bwd_ext(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, dout,
                            z=z, h0=h0, dh_last=dh)
    names = dict(u="du", dt="ddt", A="dA", B="dB", C="dC", D="dD", dt_bias="ddt_bias", z="dz",
                 h0="dh0")
    eps = 1e-6
    for k, gk in names.items():
        fd = np.zeros_like(X[k])
        for idx in np.ndindex(X[k].shape):
            kp = {a: b.copy() for a, b in X.items()}
            km = {a: b.copy() for a, b in X.items()}
            kp[k][idx] += eps
            km[k][idx] -= eps
            fd[idx] = (loss(kp) - loss(km)) / (2 * eps)
        err = np.max(np.abs(g[gk] - fd)) / max(np.max(np.abs(fd)), 1e-30)
        assert err < 1e-5, (k, err)
    # h0 is ignored for rows whose slot 0 is a head
    assert np.all(g["dh0"][1] == 0)


def test_ext_matches_autograd():
    torch = pytest.importorskip("torch")
    rng, pos, P, u, z, h0, dh = _prob(20, R=2, Dn=3, L=17, N=4)
    pos[0, 0] = 7  # continued sequence in row 0
    pos[0, 1:5] = [8, 9, 10, 11]
    dout = rng.standard_normal(u.shape)
    L = u.shape[2]
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
         for k, v in dict(u=u, dt=P["dt"], A=P["A"], B=P["B"], C=P["C"], D=P["D"],
                          dt_bias=P["dt_bias"], z=z, h0=h0).items()}
    head = torch.tensor(pos == 0)
    delta = torch.nn.functional.softplus(T["dt"] + T["dt_bias"][None, :, None])
    h = T["h0"]
    outs = []
    for t in range(L):
        keep = (~head[:, t]).to(torch.float64)[:, None, None]
        h = keep * torch.exp(delta[:, :, t, None] * T["A"][None]) * h + \
            delta[:, :, t, None] * T["B"][:, None, :, t] * T["u"][:, :, t, None]
        y = (h * T["C"][:, None, :, t]).sum(-1) + T["D"][None] * T["u"][:, :, t]
        outs.append(y * torch.nn.functional.silu(T["z"][:, :, t]))
    out = torch.stack(outs, -1)
    ((out * torch.tensor(dout)).sum() + (h * torch.tensor(dh)).sum()).backward()
    g = oracle.scan_bwd_ext(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, dout,
                            z=z, h0=h0, dh_last=dh)
    for k, gk in dict(u="du", dt="ddt", A="dA", B="dB", C="dC", D="dD", dt_bias="ddt_bias",
                      z="dz", h0="dh0").items():
        np.testing.assert_allclose(g[gk], T[k].grad.numpy(), rtol=1e-10, atol=1e-12, err_msg=k)


def test_state_passing_reproduces_the_uncut_row():
    """cut a long sequence at a non-head slot into two rows and pass
    the state: forward outputs and per-token gradients equal the uncut run."""
    rng = np.random.default_rng(30)
    Dn, L, N, m = 3, 40, 4, 17
    rows = [[9, 31]]  # the 2nd sequence (slots 9..39) is cut at slot m
    _, pos, _, P = rand_problem(rng, 1, Dn, L, N, 4, rows)
    u = rng.standard_normal((1, Dn, L))
    z = rng.standard_normal((1, Dn, L))
    dout = rng.standard_normal((1, Dn, L))
    full = (u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    out, _ = oracle.scan_fwd_ext(*full, z=z)
    g = oracle.scan_bwd_ext(*full, dout, z=z)
    cut = lambda a, s: np.ascontiguousarray(a[..., s])
    a1, a2 = slice(0, m), slice(m, L)
    part = lambda s: (cut(u, s), cut(P["dt"], s), P["A"], cut(P["B"], s), cut(P["C"], s), P["D"],
                      P["dt_bias"], cut(pos, s))
    o1, h1 = oracle.scan_fwd_ext(*part(a1), z=cut(z, a1))
    o2, _ = oracle.scan_fwd_ext(*part(a2), z=cut(z, a2), h0=h1)
    assert np.array_equal(np.concatenate([o1, o2], -1), out)
    g2 = oracle.scan_bwd_ext(*part(a2), cut(dout, a2), z=cut(z, a2), h0=h1)
    g1 = oracle.scan_bwd_ext(*part(a1), cut(dout, a1), z=cut(z, a1), dh_last=g2["dh0"])
    for k in ("du", "ddt", "dB", "dC", "dz"):
        assert np.array_equal(np.concatenate([g1[k], g2[k]], -1), g[k]), k
    for k in ("dA", "dD", "ddt_bias"):
        np.testing.assert_allclose(g1[k] + g2[k], g[k], rtol=1e-12, atol=1e-12)


def test_decay_row_summary():
    """decay = d h_last / d h0 (NEXT-2's (prod abar, h) row summary): equals
    exp(A sum delta) on rows without a head, 0 on rows with one, and
    h_last(h0) = decay * h0 + h_last(0) exactly up to rounding (linearity)."""
    rng = np.random.default_rng(40)
    R, Dn, L, N = 3, 2, 12, 3
    _, pos, _, P = rand_problem(rng, R, Dn, L, N, 4, [[L], [L], [5, 7]])
    pos[0] += 4  # row 0 continues a sequence: no head anywhere
    pos[1, :4] = [2, 3, 4, 5]  # row 1 continues, then a head at slot 4
    pos[1, 4:] = np.arange(L - 4)
    u = rng.standard_normal((R, Dn, L))
    h0 = rng.standard_normal((R, Dn, N))
    args = (u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    for zoh in (False, True):
        _, hl, dec = oracle.scan_fwd_ext(*args, h0=h0, zoh=zoh, want_decay=True)
        _, hl0, dec0 = oracle.scan_fwd_ext(*args, h0=np.zeros_like(h0), zoh=zoh, want_decay=True)
        assert np.array_equal(dec, dec0)
        delta = np.logaddexp(0.0, P["dt"] + P["dt_bias"][None, :, None])
        closed = np.exp(P["A"][None] * delta.sum(-1)[:, :, None])
        np.testing.assert_allclose(dec[0], closed[0], rtol=1e-12)
        assert np.all(dec[1] == 0) and np.all(dec[2] == 0)
        np.testing.assert_allclose(hl, dec * h0 + hl0, rtol=1e-12, atol=1e-13)
        # finite differences of h_last in h0 (diagonal Jacobian)
        eps = 1e-6
        for idx in [(0, 0, 0), (0, 1, 2), (1, 1, 1)]:
            hp, hm = h0.copy(), h0.copy()
            hp[idx] += eps
            hm[idx] -= eps
            fd = (oracle.scan_fwd_ext(*args, h0=hp, zoh=zoh)[1][idx] -
                  oracle.scan_fwd_ext(*args, h0=hm, zoh=zoh)[1][idx]) / (2 * eps)
            assert abs(fd - dec[idx]) < 1e-8

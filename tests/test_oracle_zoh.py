"""Pins for the oracle's NEXT-4 discretisation: ZOH, Eq 2b
B-bar = (delta A)^-1 (exp(delta A) - I) delta B, with the removable
singularity handled by a Taylor branch."""
import numpy as np
import pytest

import oracle
from tests.test_oracle_pins import rand_problem


def _one_step(delta, a, b, steps=1, u=None):
    """R = Dn = N = 1, softplus off, C = 1, D = 0: y_t = h_t."""
    L = steps
    u = np.ones((1, 1, L)) if u is None else np.asarray(u, float).reshape(1, 1, L)
    dt = np.full((1, 1, L), delta)
    A = np.array([[a]])
    B = np.full((1, 1, L), b)
    C = np.ones((1, 1, L))
    pos = np.arange(L, dtype=np.int32)[None, :]
    y, h = oracle.scan_fwd_ext(u, dt, A, B, C, np.zeros(1), np.zeros(1), pos, softplus=False,
                               zoh=True)
    return y[0, 0], h[0, 0, 0]


def test_spec_discretize_examples(golden):
    """S:262-264 through the scan: a head step gives h_0 = b_bar * u_0, a
    second step with u = 0 gives h_1 = a_bar * h_0."""
    for c in golden["discretize_zoh"]["cases"]:
        y, _ = _one_step(c["delta"], c["a"], c["b"], steps=2, u=[1.0, 0.0])
        assert abs(y[0] - c["b_bar"]) <= c["tol"], c["note"]
        assert abs(y[1] - c["a_bar"] * c["b_bar"]) <= c["tol"] * max(1.0, c["a_bar"]), c["note"]


def test_taylor_branch_is_continuous():
    """f(z) = (e^z - 1)/z across the |z| = 1e-4 switch and f'(z)
    across 1e-3, seen through b_bar and through dA (FD)."""
    for z in (-1.01e-4, -0.99e-4, 0.99e-4, 1.01e-4, -1.01e-3, -0.99e-3):
        y, _ = _one_step(1.0, z, 1.0)
        # the 3-term Taylor value of S:262 is within z^3/24 < 5e-14 of f(z)
        assert abs(y[0] - np.expm1(z) / z) < 5e-14


def test_zoh_equals_euler_when_A_is_zero():
    """At A = 0, f(0) = 1: forward, dB, dC are bit-identical to the Euler
    path, du and ddt equal up to summation order; dA gains exactly
    sum_t g_t B_t u_t delta_t^2 / 2 (f'(0) = 1/2)."""
    rng = np.random.default_rng(3)
    rows, pos, valid, P = rand_problem(rng, 2, 3, 30, 4, 4)
    A0 = np.zeros_like(P["A"])
    args = (P["x"], P["dt"], A0, P["B"], P["C"], P["D"], P["dt_bias"], pos)
    ye, _ = oracle.scan_fwd_ext(*args)
    yz, _ = oracle.scan_fwd_ext(*args, zoh=True)
    assert np.array_equal(ye, yz)
    ge = oracle.scan_bwd_ext(*args, P["dy"])
    gz = oracle.scan_bwd_ext(*args, P["dy"], zoh=True)
    for k in ("dB", "dC"):
        assert np.array_equal(ge[k], gz[k]), k
    for k in ("du", "ddt"):
        np.testing.assert_allclose(gz[k], ge[k], rtol=1e-13, atol=1e-14, err_msg=k)
    # closed form of the extra dA term: with A = 0, abar = 1 and the state
    # gradient g_t is the suffix sum of C dy within the sequence
    R, Dn, L = P["x"].shape
    N = A0.shape[1]
    delta = np.logaddexp(0.0, P["dt"] + P["dt_bias"][None, :, None])
    extra = np.zeros((Dn, N))
    for r in range(R):
        for d in range(Dn):
            g = np.zeros(N)
            for t in range(L - 1, -1, -1):
                g = g + P["C"][r, :, t] * P["dy"][r, d, t]
                extra[d] += g * P["B"][r, :, t] * P["x"][r, d, t] * delta[r, d, t] ** 2 / 2
                if pos[r, t] == 0:
                    g = np.zeros(N)
    np.testing.assert_allclose(gz["dA"] - ge["dA"], extra, rtol=1e-9, atol=1e-12)


def test_geometric_closed_form():
    """Constant delta, A, B, u on one sequence: h_t = b_bar (1 - a^(t+1)) / (1 - a)."""
    delta, a, b, L = 0.3, -0.7, 1.3, 12
    y, _ = _one_step(delta, a, b, steps=L)
    ab = np.exp(delta * a)
    bb = np.expm1(delta * a) / a * b
    ref = bb * (1 - ab ** np.arange(1, L + 1)) / (1 - ab)
    np.testing.assert_allclose(y, ref, rtol=1e-13)


@pytest.mark.parametrize("seed", range(2))
def test_zoh_finite_differences(seed):
    rng = np.random.default_rng(50 + seed)
    rows, pos, valid, P = rand_problem(rng, 2, 2, 9, 3, 4)
    pos[0, 0] = 5  # row 0 continues a sequence through h0
    A = P["A"].copy()
    A[0, 0] = -3e-5  # exercises the Taylor branches of f and f'
    A[1, 1] = -4e-4
    u, z = P["x"], rng.standard_normal(P["x"].shape)
    h0 = rng.standard_normal((2, 2, 3))
    dh = rng.standard_normal((2, 2, 3))
    dout = rng.standard_normal(u.shape)
    X = dict(u=u, dt=P["dt"], A=A, B=P["B"], C=P["C"], D=P["D"], dt_bias=P["dt_bias"], z=z, h0=h0)

    def loss(k):
        out, hl = oracle.scan_fwd_ext(k["u"], k["dt"], k["A"], k["B"], k["C"], k["D"],
                                      k["dt_bias"], pos, z=k["z"], h0=k["h0"], zoh=True)
        return float(np.sum(out * dout) + np.sum(hl * dh))

    g = oracle.scan_bwd_ext(u, P["dt"], A, P["B"], P["C"], P["D"], P["dt_bias"], pos, dout,
                            z=z, h0=h0, dh_last=dh, zoh=True)
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


def test_zoh_matches_autograd():
    """An independent torch statement of Eq 1a/1b with Eq 2b's B-bar."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(60)
    rows, pos, valid, P = rand_problem(rng, 2, 3, 17, 4, 4)
    dout = rng.standard_normal(P["x"].shape)
    L = P["x"].shape[2]
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
         for k, v in dict(u=P["x"], dt=P["dt"], A=P["A"], B=P["B"], C=P["C"], D=P["D"],
                          dt_bias=P["dt_bias"]).items()}
    head = torch.tensor(pos == 0)
    delta = torch.nn.functional.softplus(T["dt"] + T["dt_bias"][None, :, None])
    h = torch.zeros(2, 3, 4, dtype=torch.float64)
    outs = []
    for t in range(L):
        dA = delta[:, :, t, None] * T["A"][None]
        bbar = torch.expm1(dA) / T["A"][None] * T["B"][:, None, :, t]  # (e^{dA}-1)/(dA) * delta B
        keep = (~head[:, t]).to(torch.float64)[:, None, None]
        h = keep * torch.exp(dA) * h + bbar * T["u"][:, :, t, None]
        outs.append((h * T["C"][:, None, :, t]).sum(-1) + T["D"][None] * T["u"][:, :, t])
    (torch.stack(outs, -1) * torch.tensor(dout)).sum().backward()
    g = oracle.scan_bwd_ext(P["x"], P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos,
                            dout, zoh=True)
    for k, gk in dict(u="du", dt="ddt", A="dA", B="dB", C="dC", D="dD",
                      dt_bias="ddt_bias").items():
        np.testing.assert_allclose(g[gk], T[k].grad.numpy(), rtol=1e-10, atol=1e-12, err_msg=k)

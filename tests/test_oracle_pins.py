"""Pins for the fp64 oracle against things the paper and mathematics fix.

None of these re-types the oracle's formulas: each check is an independent
fact -- a printed worked example (tests/golden, SPEC citations), the PUI
invariant f(S) = unpack(f(pack(S))) against the *unpacked*
textbook operators, zero cross-sequence leakage, central finite differences,
autograd of an independent torch statement of Eq 1a/1b, the Eq 3 brute force
(P:213-216), torch.nn.functional.conv1d on single-sequence rows, closed forms
(all heads, L = 1, integer-exact prefix sums), and adjoint identities.
"""
import numpy as np
import pytest

import oracle
from workload import gen_lengths, pos_from_rows

LN_HALF = float(np.log(0.5))


# ----------------------------------------------------------------------------
# helpers (data construction only)
# ----------------------------------------------------------------------------

def rand_layout(rng, R, L, max_len=None, allow_pad=True):
    rows = []
    for _ in range(R):
        lens, t = [], 0
        while t < L:
            ln = int(rng.integers(1, (max_len or L) + 1))
            if t + ln > L:
                if allow_pad and rng.random() < 0.5:
                    break
                ln = L - t
            lens.append(ln)
            t += ln
        rows.append(lens)
    return rows


def rand_problem(rng, R, Dn, L, N, K, rows=None):
    rows = rows if rows is not None else rand_layout(rng, R, L, max_len=max(2, L // 2))
    pos, valid = pos_from_rows(rows, L)
    P = dict(
        x=rng.standard_normal((R, Dn, L)) * valid[:, None, :],
        dt=0.5 * rng.standard_normal((R, Dn, L)),
        B=rng.standard_normal((R, N, L)),
        C=rng.standard_normal((R, N, L)),
        dy=rng.standard_normal((R, Dn, L)) * valid[:, None, :],
        A=-(np.arange(1, N + 1)[None, :]) * np.exp(0.1 * rng.standard_normal((Dn, N))),
        D=1 + 0.1 * rng.standard_normal(Dn),
        dt_bias=rng.uniform(-4, -1, Dn),
        w=rng.uniform(-0.5, 0.5, (Dn, K)),
        bias=rng.uniform(-0.5, 0.5, Dn),
    )
    return rows, pos, valid, P


def segments(rows):
    """(row, start, length) of each sequence of a layout."""
    out = []
    for r, lens in enumerate(rows):
        t = 0
        for ln in lens:
            out.append((r, t, ln))
            t += ln
    return out


# ----------------------------------------------------------------------------
# P4: printed worked examples (SPEC)
# ----------------------------------------------------------------------------

def test_plan_fifo_examples(golden):
    for ex in golden["plan_fifo"]:
        row, off, nr = oracle.plan_fifo(ex["lengths"], ex["capacity"])
        packs = [[i for i in range(len(row)) if row[i] == r] for r in range(nr)]
        assert packs == ex["packs"], ex["cite"]
        pad = nr * ex["capacity"] - sum(ex["lengths"])
        assert [pad, nr * ex["capacity"]] == ex["padding"], ex["cite"]


def test_plan_ffd_examples(golden):
    for ex in golden["plan_ffd"]:
        row, off, nr = oracle.plan_ffd(ex["lengths"], ex["capacity"])
        packs = [sorted([i for i in range(len(row)) if row[i] == r],
                        key=lambda i: off[i]) for r in range(nr)]
        assert packs == ex["packs"], ex["cite"]
        assert [nr * ex["capacity"] - sum(ex["lengths"]),
                nr * ex["capacity"]] == ex["padding"]


def test_capacity_error():
    with pytest.raises(oracle.CapacityError):
        oracle.plan_fifo([3, 9], 8)
    with pytest.raises(oracle.CapacityError):
        oracle.plan_ffd([9], 8)


def test_pack_examples(golden):
    for ex in golden["pack"]:
        seqs = ex["sequences"]
        lens = [len(s) for s in seqs]
        src = np.array([v for s in seqs for v in s], np.float32).view(np.uint8).reshape(-1, 4)
        dst, pos = oracle.pack(lens, ex["capacity"], src)
        data = dst.reshape(dst.shape[0], -1).view(np.float32)
        assert data.tolist() == ex["data"], ex["cite"]
        assert pos.tolist() == ex["pos"], ex["cite"]


def test_reverse_indices_reading(golden):
    """Reading Q7: o <= rev[s]  <=>  o <= pos[s+o] (for s+o inside the row)."""
    for ex in golden["reverse_indices"]:
        pos, rev = np.array(ex["pos"]), np.array(ex["reverse"])
        L = len(pos)
        for s in range(L):
            for o in range(0, 4):
                if s + o < L:
                    assert (o <= rev[s]) == (o <= pos[s + o]), (s, o)


def test_scan_serial_examples(golden):
    for ex in golden["scan_serial"]:
        abar = np.array(ex["abar"], float)
        L = len(abar)
        pos = np.array([ex["pos"]], np.int32)
        # abar away from heads is constant in these examples; A = ln(abar)
        a_in = abar[pos[0] != 0]
        A = np.array([[np.log(a_in[0]) if len(a_in) else 0.0]])
        u = np.array(ex["b"], float)[None, None, :]
        y, h = oracle.scan_fwd(u, np.ones((1, 1, L)), A, np.ones((1, 1, L)),
                               np.ones((1, 1, L)), None, None, pos,
                               softplus=False, return_h=True)
        np.testing.assert_allclose(h[0, 0, :, 0], ex["h"], rtol=0, atol=1e-15,
                                   err_msg=ex["cite"])


def test_scan_reverse_example(golden):
    """S:207 g_t = a_t g_{t+1} + b_t with shifted a; observed through the
    scan bwd as dB_t = g_t * delta * u (delta = u = 1) and du = g_t B."""
    ex = golden["scan_reverse"][0]
    L = len(ex["b"])
    # abar_shifted[t] = abar_{t+1}; here abar_1 = abar_2 = 0.5
    A = np.array([[LN_HALF]])
    pos = np.arange(L, dtype=np.int32)[None, :]
    one = np.ones((1, 1, L))
    g = oracle.scan_bwd(one, one, A, one, one, None, None, pos,
                        np.array(ex["b"], float)[None, None, :], softplus=False)
    np.testing.assert_allclose(g["dB"][0, 0], ex["g"], atol=1e-15)
    np.testing.assert_allclose(g["du"][0, 0], ex["g"], atol=1e-15)


def test_ssm_fwd_examples(golden):
    for ex in golden["ssm_fwd"]:
        L = len(ex["x"])
        f = lambda v: np.full((1, 1, L), v, float)
        y = oracle.scan_fwd(np.array(ex["x"], float)[None, None], f(ex["delta"]),
                            np.array([[ex["A"]]]), f(ex["B"]), f(ex["C"]),
                            np.array([ex["D"]]), None,
                            np.array([ex["pos"]], np.int32), softplus=False)
        np.testing.assert_array_equal(y[0, 0], ex["y"], err_msg=ex["cite"])


def test_conv_examples(golden):
    for ex in golden["conv_fwd"]:
        x = np.array(ex["x"], float)[None, None]
        y = oracle.conv_fwd(x, np.array([ex["weight"]], float), np.array([ex["bias"]]),
                            np.array([ex["pos"]], np.int32), silu=False)
        np.testing.assert_array_equal(y[0, 0], ex["y"], err_msg=ex["cite"])
    for ex in golden["conv_bwd"]:
        x = np.array(ex["x"], float)[None, None]
        dx, dw, db = oracle.conv_bwd(x, np.array([ex["weight"]], float),
                                     np.array([ex["bias"]]),
                                     np.array([ex["pos"]], np.int32),
                                     np.array(ex["dy"], float)[None, None], silu=False)
        np.testing.assert_array_equal(dx[0, 0], ex["dx"], err_msg=ex["cite"])
        np.testing.assert_array_equal(dw[0], ex["dweight"], err_msg=ex["cite"])
        np.testing.assert_array_equal(db, ex["dbias"], err_msg=ex["cite"])


# ----------------------------------------------------------------------------
# P1: PUI against the unpacked textbook operators (bit-exact in fp64)
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("silu,softplus", [(True, True), (False, False)])
def test_pui_packed_equals_unpacked(seed, silu, softplus):
    rng = np.random.default_rng(seed)
    R, Dn, L, N, K = 3, 4, 37, 3, 1 + seed % 4
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, N, K)
    u = oracle.conv_fwd(P["x"], P["w"], P["bias"], pos, silu)
    y = oracle.scan_fwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"],
                        pos, softplus)
    gs = oracle.scan_bwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"],
                         pos, P["dy"], softplus)
    dx, dw, db = oracle.conv_bwd(P["x"], P["w"], P["bias"], pos, gs["du"], silu)

    acc = dict(dA=np.zeros_like(P["A"]), dD=np.zeros(Dn), ddt_bias=np.zeros(Dn))
    dw2, db2 = np.zeros_like(P["w"]), np.zeros(Dn)
    for r, s, ln in segments(rows):
        sl = slice(s, s + ln)
        xs = P["x"][r, :, sl]
        us = oracle.seq_conv_fwd(xs, P["w"], P["bias"], silu)
        np.testing.assert_array_equal(u[r, :, sl], us)
        ys = oracle.seq_scan_fwd(us, P["dt"][r, :, sl], P["A"], P["B"][r, :, sl],
                                 P["C"][r, :, sl], P["D"], P["dt_bias"], softplus)
        np.testing.assert_array_equal(y[r, :, sl], ys)
        du, ddt, dB, dC = oracle.seq_scan_bwd(
            us, P["dt"][r, :, sl], P["A"], P["B"][r, :, sl], P["C"][r, :, sl],
            P["D"], P["dt_bias"], P["dy"][r, :, sl], acc, softplus)
        # per-token grads: same arithmetic order -> bit-exact
        np.testing.assert_array_equal(gs["du"][r, :, sl], du)
        np.testing.assert_array_equal(gs["ddt"][r, :, sl], ddt)
        np.testing.assert_array_equal(gs["dB"][r, :, sl], dB)
        np.testing.assert_array_equal(gs["dC"][r, :, sl], dC)
        dxs = oracle.seq_conv_bwd(xs, P["w"], P["bias"], du, dw2, db2, silu)
        np.testing.assert_array_equal(dx[r, :, sl], dxs)
    # param grads: summation order differs (per sequence vs per row)
    for k in ("dA", "dD", "ddt_bias"):
        np.testing.assert_allclose(gs[k], acc[k], rtol=1e-12, atol=1e-12)
    # padding contributes exactly zero to conv param grads once dy = 0 there
    np.testing.assert_allclose(dw, dw2, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(db, db2, rtol=1e-12, atol=1e-12)


def test_unmasked_conv_fails_pui():
    """Negative pin: a conv that ignores position_indices reads
    across the boundary and breaks PUI at the 2nd sequence's first slot."""
    rng = np.random.default_rng(0)
    Dn, L, K = 2, 12, 4
    rows = [[5, 7]]
    pos, _ = pos_from_rows(rows, L)
    x = rng.standard_normal((1, Dn, L))
    w, b = rng.uniform(-1, 1, (Dn, K)), np.zeros(Dn)
    masked = oracle.conv_fwd(x, w, b, pos, silu=False)
    unmasked = oracle.conv_fwd(x, w, b, np.arange(L, dtype=np.int32)[None], silu=False)
    ref = oracle.seq_conv_fwd(x[0, :, 5:], w, b, silu=False)
    np.testing.assert_array_equal(masked[0, :, 5:], ref)
    bad = np.abs(unmasked[0, :, 5:] - ref)
    assert bad[:, 0].max() > 1e-3            # worst location: position 0 of seq 2
    assert np.all(bad[:, K - 1:] == 0)       # taps stay inside after K-1 slots


# ----------------------------------------------------------------------------
# P2: zero cross-sequence leakage
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(4))
def test_isolation(seed):
    rng = np.random.default_rng(100 + seed)
    R, Dn, L, N, K = 1, 3, 40, 2, 4
    rows = [[9, 1, 14, 10]]
    _, pos, valid, P = rand_problem(rng, R, Dn, L, N, K, rows)
    j0, j1 = 10, 24  # the 3rd sequence (slots 10..23)

    def run(Q):
        u = oracle.conv_fwd(Q["x"], Q["w"], Q["bias"], pos)
        y = oracle.scan_fwd(u, Q["dt"], Q["A"], Q["B"], Q["C"], Q["D"], Q["dt_bias"], pos)
        g = oracle.scan_bwd(u, Q["dt"], Q["A"], Q["B"], Q["C"], Q["D"], Q["dt_bias"], pos, Q["dy"])
        dx, _, _ = oracle.conv_bwd(Q["x"], Q["w"], Q["bias"], pos, g["du"])
        return dict(u=u, y=y, du=g["du"], ddt=g["ddt"], dB=g["dB"], dC=g["dC"], dx=dx)

    base = run(P)
    Q = {k: v.copy() for k, v in P.items()}
    for k, v in (("x", 5.0), ("dt", 3.0), ("dy", -7.0)):
        Q[k][:, :, j0:j1] += v * rng.standard_normal((R, Dn, j1 - j0))
    for k in ("B", "C"):
        Q[k][:, :, j0:j1] += 4.0 * rng.standard_normal((R, N, j1 - j0))
    pert = run(Q)
    other = np.ones(L, bool)
    other[j0:j1] = False
    for k in base:
        assert np.array_equal(base[k][..., other], pert[k][..., other]), k
        assert not np.array_equal(base[k][..., j0:j1], pert[k][..., j0:j1]), k


# ----------------------------------------------------------------------------
# P3: central finite differences (fp64, step 1e-6)
# ----------------------------------------------------------------------------

def _rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("softplus", [True, False])
def test_scan_bwd_finite_differences(seed, softplus):
    rng = np.random.default_rng(200 + seed)
    R, Dn, L, N = 2, 2, 8, 2
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, N, 4)
    if not softplus:  # delta = dt + dt_bias must stay a positive step size
        P["dt"] = 0.2 * np.abs(P["dt"]) + 0.05
        P["dt_bias"] = rng.uniform(0.0, 0.1, Dn)
    u = rng.standard_normal((R, Dn, L))
    keys = dict(u=u, dt=P["dt"], A=P["A"], B=P["B"], C=P["C"], D=P["D"], dt_bias=P["dt_bias"])
    dy = rng.standard_normal((R, Dn, L))

    def loss(kw):
        y = oracle.scan_fwd(kw["u"], kw["dt"], kw["A"], kw["B"], kw["C"], kw["D"],
                            kw["dt_bias"], pos, softplus)
        return float(np.sum(y * dy))

    g = oracle.scan_bwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, dy, softplus)
    names = dict(u="du", dt="ddt", A="dA", B="dB", C="dC", D="dD", dt_bias="ddt_bias")
    eps = 1e-6
    for k, gk in names.items():
        fd = np.zeros_like(keys[k])
        for idx in np.ndindex(keys[k].shape):
            kp = {kk: vv.copy() for kk, vv in keys.items()}
            km = {kk: vv.copy() for kk, vv in keys.items()}
            kp[k][idx] += eps
            km[k][idx] -= eps
            fd[idx] = (loss(kp) - loss(km)) / (2 * eps)
        assert _rel(g[gk], fd) < 1e-5, (k, _rel(g[gk], fd))


@pytest.mark.parametrize("K", [1, 2, 3, 4])
@pytest.mark.parametrize("silu", [True, False])
def test_conv_bwd_finite_differences(K, silu):
    rng = np.random.default_rng(300 + K)
    R, Dn, L = 2, 3, 11
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, 2, K)
    x = rng.standard_normal((R, Dn, L))
    dout = rng.standard_normal((R, Dn, L))
    keys = dict(x=x, w=P["w"], bias=P["bias"])

    def loss(kw):
        return float(np.sum(oracle.conv_fwd(kw["x"], kw["w"], kw["bias"], pos, silu) * dout))

    dx, dw, db = oracle.conv_bwd(x, P["w"], P["bias"], pos, dout, silu)
    eps = 1e-6
    for k, gk in (("x", dx), ("w", dw), ("bias", db)):
        fd = np.zeros_like(keys[k])
        for idx in np.ndindex(keys[k].shape):
            kp = {kk: vv.copy() for kk, vv in keys.items()}
            km = {kk: vv.copy() for kk, vv in keys.items()}
            kp[k][idx] += eps
            km[k][idx] -= eps
            fd[idx] = (loss(kp) - loss(km)) / (2 * eps)
        assert _rel(gk, fd) < 1e-6, (k, _rel(gk, fd))


# ----------------------------------------------------------------------------
# autograd of an independent torch statement of the packed forward
# ----------------------------------------------------------------------------

def test_scan_bwd_matches_autograd():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(7)
    R, Dn, L, N = 2, 3, 19, 4
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, N, 4)
    u = rng.standard_normal((R, Dn, L))
    dy = rng.standard_normal((R, Dn, L))
    T = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
         for k, v in dict(u=u, dt=P["dt"], A=P["A"], B=P["B"], C=P["C"],
                          D=P["D"], dt_bias=P["dt_bias"]).items()}
    head = torch.tensor((pos == 0) | (np.arange(L)[None] == 0))
    delta = torch.nn.functional.softplus(T["dt"] + T["dt_bias"][None, :, None])
    h = torch.zeros(R, Dn, N, dtype=torch.float64)
    ys = []
    for t in range(L):
        dA = torch.exp(delta[:, :, t, None] * T["A"][None])
        keep = (~head[:, t]).to(torch.float64)[:, None, None]
        h = keep * dA * h + delta[:, :, t, None] * T["B"][:, None, :, t] * T["u"][:, :, t, None]
        ys.append((h * T["C"][:, None, :, t]).sum(-1) + T["D"][None] * T["u"][:, :, t])
    y = torch.stack(ys, -1)
    (y * torch.tensor(dy)).sum().backward()
    g = oracle.scan_bwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, dy)
    for k, gk in dict(u="du", dt="ddt", A="dA", B="dB", C="dC", D="dD", dt_bias="ddt_bias").items():
        np.testing.assert_allclose(g[gk], T[k].grad.numpy(), rtol=1e-10, atol=1e-12, err_msg=k)
    np.testing.assert_allclose(
        oracle.scan_fwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos),
        y.detach().numpy(), rtol=1e-12, atol=1e-12)


# ----------------------------------------------------------------------------
# P5: Eq 3 brute force; P7: library conv; P6/P8: closed forms
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(3))
def test_eq3_brute_force(seed):
    rng = np.random.default_rng(400 + seed)
    R, Dn, L, N = 2, 3, 23, 3
    rows, pos, valid, P = rand_problem(rng, R, Dn, L, N, 4)
    u = rng.standard_normal((R, Dn, L))
    a = oracle.scan_fwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    b = oracle.scan_fwd_eq3(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("K", [1, 2, 3, 4])
def test_conv_single_sequence_equals_torch_conv1d(K):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(500 + K)
    Dn, L = 5, 33
    x = rng.standard_normal((2, Dn, L))
    w, b = rng.uniform(-1, 1, (Dn, K)), rng.uniform(-1, 1, Dn)
    pos = np.tile(np.arange(L, dtype=np.int32), (2, 1))
    ref = torch.nn.functional.conv1d(torch.tensor(x), torch.tensor(w)[:, None, :],
                                     torch.tensor(b), padding=K - 1, groups=Dn)[..., :L]
    np.testing.assert_allclose(oracle.conv_fwd(x, w, b, pos, silu=False), ref.numpy(),
                               rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(oracle.conv_fwd(x, w, b, pos, silu=True),
                               torch.nn.functional.silu(ref).numpy(), rtol=1e-13, atol=1e-13)


def test_integer_exact_regime():
    """P6: A=0, delta=1 (softplus off) -> y = segmented prefix sum of B*u
    contracted with C, exact in floating point for small integers."""
    rng = np.random.default_rng(9)
    R, Dn, L, N = 2, 3, 50, 2
    rows = [[7, 1, 30, 12], [50]]
    pos, valid = pos_from_rows(rows, L)
    u = rng.integers(-3, 4, (R, Dn, L)).astype(float)
    B = rng.integers(-2, 3, (R, N, L)).astype(float)
    C = rng.integers(-2, 3, (R, N, L)).astype(float)
    D = rng.integers(-2, 3, Dn).astype(float)
    y = oracle.scan_fwd(u, np.ones_like(u), np.zeros((Dn, N)), B, C, D, None, pos,
                        softplus=False)
    ref = np.zeros_like(y)
    for r, s, ln in segments(rows):
        bu = B[r, None, :, s:s + ln] * u[r, :, None, s:s + ln]        # (Dn,N,ln)
        h = np.cumsum(bu, axis=-1)
        ref[r, :, s:s + ln] = (h * C[r, None, :, s:s + ln]).sum(1) + D[:, None] * u[r, :, s:s + ln]
    np.testing.assert_array_equal(y, ref)


def test_all_heads_closed_form():
    """with every slot a head, y_t = C_t delta_t B_t u_t + D u_t."""
    rng = np.random.default_rng(11)
    R, Dn, L, N = 2, 3, 9, 4
    _, pos, _, P = rand_problem(rng, R, Dn, L, N, 4, [[1] * L] * R)
    u = rng.standard_normal((R, Dn, L))
    y = oracle.scan_fwd(u, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    v = P["dt"] + P["dt_bias"][None, :, None]
    delta = np.log1p(np.exp(v))
    ref = (P["C"][:, None] * P["B"][:, None]).sum(2) * delta * u + P["D"][None, :, None] * u
    np.testing.assert_allclose(y, ref, rtol=1e-13, atol=1e-13)


def test_L1_closed_form_and_zero_cotangent():
    """L = 1 -> y = C delta B x + D x; dx = C delta B + D (dy=1),
    dC = delta B x, dD = x.  S:292: dy = 0 -> all grads 0."""
    d, Bv, Cv, Dv, x = 0.7, 1.3, -0.4, 0.9, 2.0
    one = lambda v: np.array([[[v]]], float)
    pos = np.zeros((1, 1), np.int32)
    y = oracle.scan_fwd(one(x), one(d), np.array([[-1.5]]), one(Bv), one(Cv),
                        np.array([Dv]), None, pos, softplus=False)
    assert abs(y[0, 0, 0] - (Cv * d * Bv * x + Dv * x)) < 1e-15
    g = oracle.scan_bwd(one(x), one(d), np.array([[-1.5]]), one(Bv), one(Cv),
                        np.array([Dv]), None, pos, one(1.0), softplus=False)
    assert abs(g["du"][0, 0, 0] - (Cv * d * Bv + Dv)) < 1e-15
    assert abs(g["dC"][0, 0, 0] - d * Bv * x) < 1e-15
    assert abs(g["dD"][0] - x) < 1e-15
    assert g["dA"][0, 0] == 0.0  # head: abar is the constant 0
    rng = np.random.default_rng(3)
    rows, pos, valid, P = rand_problem(rng, 2, 3, 10, 2, 3)
    z = np.zeros((2, 3, 10))
    g = oracle.scan_bwd(P["x"], P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, z)
    assert all(np.all(v == 0) for v in g.values())
    dx, dw, db = oracle.conv_bwd(P["x"], P["w"], P["bias"], pos, z)
    assert np.all(dx == 0) and np.all(dw == 0) and np.all(db == 0)


def test_linearity_adjoint_identities():
    """P9: for fixed delta, B, C the scan is linear in u: <dy, y(v)> = <du, v>;
    the conv without SiLU is affine in x: <dout, out(v) - bias> = <dx, v>."""
    rng = np.random.default_rng(12)
    rows, pos, valid, P = rand_problem(rng, 2, 4, 21, 3, 4)
    v = rng.standard_normal((2, 4, 21))
    y = oracle.scan_fwd(v, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos)
    g = oracle.scan_bwd(v, P["dt"], P["A"], P["B"], P["C"], P["D"], P["dt_bias"], pos, P["dy"])
    assert abs(np.sum(P["dy"] * y) - np.sum(g["du"] * v)) < 1e-10 * np.sum(np.abs(P["dy"] * y))
    out = oracle.conv_fwd(v, P["w"], P["bias"], pos, silu=False)
    dx, dw, db = oracle.conv_bwd(v, P["w"], P["bias"], pos, P["dy"], silu=False)
    lhs = np.sum(P["dy"] * (out - P["bias"][None, :, None]))
    assert abs(lhs - np.sum(dx * v)) < 1e-10 * np.sum(np.abs(P["dy"] * out))
    # bilinear pairing with the weights: <dout, out - bias> = <dw, w> too
    assert abs(lhs - np.sum(dw * P["w"])) < 1e-10 * np.sum(np.abs(P["dy"] * out))


def test_conv_k1_pointwise():
    """width 1 -> y = c x + bias, boundaries irrelevant."""
    rng = np.random.default_rng(13)
    rows, pos, valid, P = rand_problem(rng, 2, 3, 15, 2, 1)
    y = oracle.conv_fwd(P["x"], P["w"], P["bias"], pos, silu=False)
    np.testing.assert_array_equal(y, P["w"][None, :, 0:1] * P["x"] + P["bias"][None, :, None])


# ----------------------------------------------------------------------------
# packing properties and the paper's padding-rate regime
# ----------------------------------------------------------------------------

@pytest.mark.parametrize("plan", ["fifo", "ffd"])
def test_plan_soundness_and_roundtrip(plan):
    rng = np.random.default_rng(21)
    for trial in range(20):
        cap = int(rng.integers(4, 40))
        lens = rng.integers(1, cap + 1, int(rng.integers(1, 30))).astype(np.int32)
        f = oracle.plan_fifo if plan == "fifo" else oracle.plan_ffd
        row, off, nr = f(lens, cap)
        used = np.zeros(nr, int)
        for i in range(len(lens)):
            assert 0 <= off[i] and off[i] + lens[i] <= cap
            used[row[i]] += lens[i]
        assert np.all(used <= cap)
        # slots do not overlap
        occ = np.zeros((nr, cap), int)
        for i in range(len(lens)):
            occ[row[i], off[i]:off[i] + lens[i]] += 1
        assert occ.max() <= 1
        if plan == "fifo":  # received order preserved, new row only when it does not fit
            order = np.lexsort((off, row))
            assert list(order) == list(range(len(lens)))
            for i in range(1, len(lens)):
                if row[i] != row[i - 1]:
                    assert used[row[i - 1]] + lens[i] > cap
        src = rng.integers(0, 255, (int(lens.sum()), 6)).astype(np.uint8)
        dst, pos = oracle.pack(lens, cap, src, row, off)
        assert np.all(dst[occ == 0] == 0) and np.all(pos[occ == 0] == 0)
        t = 0
        for i in range(len(lens)):
            seg = dst[row[i], off[i]:off[i] + lens[i]]
            assert np.array_equal(seg, src[t:t + lens[i]])  # unpack(pack(S)) == S
            assert np.array_equal(pos[row[i], off[i]:off[i] + lens[i]], np.arange(lens[i]))
            t += lens[i]


def test_padding_rates_on_paper_workload():
    """S:586 (approximate reproduction, P:82 66.3%, P:273 19.1% / 0.41%):
    lognormal [57, 2048] mean ~646."""
    lens = gen_lengths(100_000, 0)
    assert 633 <= lens.mean() <= 659
    assert 0.60 <= 1 - lens.mean() / 2048 <= 0.72  # pad-to-max at 2048
    row, off, nr = oracle.plan_fifo(lens, 4096)
    fifo = 1 - lens.sum() / (nr * 4096)
    assert 0.08 <= fifo <= 0.28
    row, off, nr = oracle.plan_ffd(lens[:20_000], 4096)
    ffd = 1 - lens[:20_000].sum() / (nr * 4096)
    assert ffd <= 0.02 and ffd < fifo

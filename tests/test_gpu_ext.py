"""GPU parity of the extended scan (SURVEY §8(f) NEXT-1 fused gate + last
state, NEXT-2 cross-row state passing h0 -> h_last) against the fp64
oracle's scan_fwd_ext / scan_bwd_ext, through the C ABI
(pm_selective_scan_fwd_ex / pm_selective_scan_bwd_ex)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import paper_2408_03865_b200 as pm
import workload
from tests._common import TOL, layout, rel_err, to_np

pytestmark = pytest.mark.gpu

DT = {"f32": torch.float32, "bf16": torch.bfloat16}


def problem(R, Dn, L, N, kind, io, seed, continued=(), dev="cuda"):
    """Seeded inputs; rows listed in ``continued`` start mid-sequence: their
    first sequence's positions are offset so slot 0 is not a head."""
    rng = np.random.default_rng(seed)
    rows = layout(kind, R, L, rng)
    pos_np, valid = workload.pos_from_rows(rows, L)
    for r in continued:
        n0 = rows[r][0]
        pos_np[r, :n0] += 1 + int(rng.integers(0, 500))
    shape = workload.Shape(f"e{seed}", R, L, Dn, N, 4, io)
    T = workload.row_tensors(torch, shape, list(range(R)), valid, device=dev, dtype=DT[io])
    P = workload.params(torch, shape, device=dev)
    g = torch.Generator().manual_seed(seed)
    z = torch.randn((R, Dn, L), generator=g).to(dev, DT[io])
    h0 = torch.randn((R, Dn, N), generator=g).to(dev)
    dh = torch.randn((R, Dn, N), generator=g).to(dev)
    # the scan input u: the conv output's range (silu of a unit normal)
    u = torch.nn.functional.silu(torch.randn((R, Dn, L), generator=g)).to(dev, DT[io])
    pos = torch.as_tensor(pos_np, device=dev)
    return pos, u, T, P, z, h0, dh


def run_ext(pos, u, T, P, z, h0, dh, states=True, zoh=False):
    out, st, hl = pm.pm_selective_scan_fwd_ex(u, T["dt"], P["A"], T["B"], T["C"], P["D"],
                                               P["dt_bias"], pos, z=z, h0=h0,
                                               want_states=states, want_last_state=True,
                                               zoh=zoh)
    g = pm.pm_selective_scan_bwd_ex(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"],
                                    pos, T["dy"], z=z, h0=h0, states=st, dh_last=dh,
                                    want_dh0=True, zoh=zoh)
    torch.cuda.synchronize()
    return out, hl, g


def check_ext(pos, u, T, P, z, h0, dh, io, res, zoh=False):
    out, hl, g = res
    args = (to_np(u), to_np(T["dt"]), to_np(P["A"]), to_np(T["B"]), to_np(T["C"]),
            to_np(P["D"]), to_np(P["dt_bias"]), to_np(pos).astype(np.int32))
    zz, hh = to_np(z), to_np(h0)
    ro, rhl = oracle.scan_fwd_ext(*args, z=zz, h0=hh, zoh=zoh)
    ref = oracle.scan_bwd_ext(*args, to_np(T["dy"]), z=zz, h0=hh, dh_last=to_np(dh), zoh=zoh)
    errs = {"out": (rel_err(to_np(out), ro), "fwd"), "h_last": (rel_err(to_np(hl), rhl), "fwd")}
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias", "dz", "dh0"):
        if ref.get(k) is not None and g.get(k) is not None:
            errs[k] = (rel_err(to_np(g[k]), ref[k]), "bwd")
    bad = {k: (e, TOL[(io, kind)]) for k, (e, kind) in errs.items() if not e <= TOL[(io, kind)]}
    assert not bad, f"tolerance exceeded: {bad}; all: {errs}"
    return errs


@pytest.mark.parametrize("io", ["f32", "bf16"])
@pytest.mark.parametrize("kind", ["random", "one", "edges"])
def test_ext_gate_and_state_passing(io, kind):
    pos, u, T, P, z, h0, dh = problem(3, 200, 1024, 16, kind, io, seed=40 + len(kind),
                                      continued=(0, 2))
    check_ext(pos, u, T, P, z, h0, dh, io, run_ext(pos, u, T, P, z, h0, dh))


@pytest.mark.parametrize("N", [4, 8])
@pytest.mark.parametrize("L", [13, 700])
def test_ext_shapes_and_scalar_path(N, L):
    pos, u, T, P, z, h0, dh = problem(2, 70, L, N, "random", "f32", seed=N * 1000 + L,
                                      continued=(1,))
    check_ext(pos, u, T, P, z, h0, dh, "f32", run_ext(pos, u, T, P, z, h0, dh))


def test_ext_each_option_alone():
    """z only, h0 only, dh_last only: each against the oracle."""
    pos, u, T, P, z, h0, dh = problem(2, 64, 512, 16, "random", "f32", seed=7, continued=(0,))
    for zz, hh, dd in ((z, None, None), (None, h0, None), (None, None, dh)):
        res = run_ext(pos, u, T, P, zz, hh, dd)
        out, hl, g = res
        args = (to_np(u), to_np(T["dt"]), to_np(P["A"]), to_np(T["B"]), to_np(T["C"]),
                to_np(P["D"]), to_np(P["dt_bias"]), to_np(pos).astype(np.int32))
        ro, rhl = oracle.scan_fwd_ext(*args, z=to_np(zz), h0=to_np(hh))
        ref = oracle.scan_bwd_ext(*args, to_np(T["dy"]), z=to_np(zz), h0=to_np(hh),
                                  dh_last=to_np(dd))
        assert rel_err(to_np(out), ro) <= 1e-4
        assert rel_err(to_np(hl), rhl) <= 1e-4
        for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias", "dz", "dh0"):
            if ref.get(k) is not None and g.get(k) is not None:
                assert rel_err(to_np(g[k]), ref[k]) <= 1e-3, k


def test_ext_without_options_equals_base_abi():
    """pm_selective_scan_*_ex with no options is the base ABI, bit for bit."""
    pos, u, T, P, z, h0, dh = problem(2, 96, 900, 16, "random", "bf16", seed=8)
    y, st = pm.pm_selective_scan_fwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"],
                                     pos)
    g = pm.pm_selective_scan_bwd(u, T["dt"], P["A"], T["B"], T["C"], P["D"], P["dt_bias"], pos,
                                 T["dy"], states=st)
    out, hl, ge = run_ext(pos, u, T, P, None, None, None)
    assert torch.equal(out, y)
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias"):
        assert torch.equal(ge[k], g[k]), k
    assert ge["dz"] is None


def test_ext_recompute_states_equals_saved():
    pos, u, T, P, z, h0, dh = problem(2, 96, 900, 16, "random", "f32", seed=9, continued=(1,))
    a = run_ext(pos, u, T, P, z, h0, dh, states=True)
    b = run_ext(pos, u, T, P, z, h0, dh, states=False)
    assert torch.equal(a[0], b[0])
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias", "dz", "dh0"):
        assert torch.equal(a[2][k], b[2][k]), k


@pytest.mark.parametrize("m", [16, 333, 512])
def test_cut_row_state_passing_reproduces_uncut(monkeypatch, m):
    """a row cut at slot m into two rows with h_last -> h0 (and dh0 ->
    dh_last backwards) gives the uncut row's results; per-token outputs are
    bit-identical (the per-lane recurrence runs the same operations in the
    same order), per-parameter sums agree to rounding."""
    # (the backward's time split cuts the two launches' rows at different
    # places -- another summation order -- so it is pinned off here; it has
    # its own parity tests below)
    monkeypatch.setenv("PM_TSPLIT", "0")
    L = 1024
    pos, u, T, P, z, h0, dh = problem(1, 128, L, 16, "random", "f32", seed=11 + m)
    full = run_ext(pos, u, T, P, z, None, None)
    cut = lambda t, s: t[..., s].contiguous()
    a1, a2 = slice(0, m), slice(m, L)

    def part(s, h0_, dh_):
        Tp = {k: cut(T[k], s) for k in ("dt", "B", "C", "dy")}
        return run_ext(cut(pos, s), cut(u, s), Tp, P, cut(z, s), h0_, dh_)

    o1, hl1, _ = part(a1, None, None)
    o2, _, g2 = part(a2, hl1, None)
    _, _, g1 = part(a1, None, g2["dh0"])
    assert torch.equal(torch.cat([o1, o2], -1), full[0])
    for k in ("du", "ddt", "dz", "dB", "dC"):
        assert torch.equal(torch.cat([g1[k], g2[k]], -1), full[2][k]), k
    for k in ("dA", "dD", "ddt_bias"):
        torch.testing.assert_close(g1[k] + g2[k], full[2][k], rtol=1e-5, atol=1e-5)


# --------------------------------------------------------------------------
# NEXT-4: ZOH discretisation (Eq 2b)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("io", ["f32", "bf16"])
@pytest.mark.parametrize("gate", [False, True])
def test_zoh_parity(io, gate):
    """delta in [1e-3, 0.1+] and A in [-17, -1] put z = delta A on both sides
    of the series / closed-form switch at |z| = 0.1."""
    pos, u, T, P, z, h0, dh = problem(3, 200, 1024, 16, "random", io, seed=70 + gate,
                                      continued=(1,))
    z = z if gate else None
    check_ext(pos, u, T, P, z, h0, dh, io, run_ext(pos, u, T, P, z, h0, dh, zoh=True), zoh=True)


@pytest.mark.parametrize("N,L", [(4, 13), (8, 700)])
def test_zoh_shapes_and_zero_A(N, L):
    """Scalar path, other N, and a zero column of A (f(0) = 1: the series)."""
    pos, u, T, P, z, h0, dh = problem(2, 70, L, N, "random", "f32", seed=80 + N, continued=(0,))
    P["A"][3] = 0.0
    P["A"][5, 1] = -1e-6
    check_ext(pos, u, T, P, None, h0, dh, "f32", run_ext(pos, u, T, P, None, h0, dh, zoh=True),
              zoh=True)


def test_zoh_recompute_equals_saved():
    pos, u, T, P, z, h0, dh = problem(2, 96, 900, 16, "edges", "f32", seed=90, continued=(1,))
    a = run_ext(pos, u, T, P, z, h0, dh, states=True, zoh=True)
    b = run_ext(pos, u, T, P, z, h0, dh, states=False, zoh=True)
    assert torch.equal(a[0], b[0])
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias", "dz", "dh0"):
        assert torch.equal(a[2][k], b[2][k]), k


# --------------------------------------------------------------------------
# NEXT-2 row summaries: decay = d h_last / d h0, context-parallel composition
# --------------------------------------------------------------------------

def test_decay_parity():
    pos, u, T, P, z, h0, dh = problem(4, 96, 512, 16, "one", "f32", seed=95, continued=(0, 2))
    out, st, hl, dec = pm.pm_selective_scan_fwd_ex(u, T["dt"], P["A"], T["B"], T["C"], P["D"],
                                                   P["dt_bias"], pos, h0=h0, want_last_state=True,
                                                   want_decay=True)
    torch.cuda.synchronize()
    args = (to_np(u), to_np(T["dt"]), to_np(P["A"]), to_np(T["B"]), to_np(T["C"]),
            to_np(P["D"]), to_np(P["dt_bias"]), to_np(pos).astype(np.int32))
    _, rhl, rdec = oracle.scan_fwd_ext(*args, h0=to_np(h0), want_decay=True)
    assert rel_err(to_np(dec), rdec) <= 1e-4
    assert rel_err(to_np(hl), rhl) <= 1e-4
    d = to_np(dec)
    assert np.all(d[1] == 0) and np.all(d[3] == 0)  # rows that start a sequence
    assert np.any(d[0] > 0) and np.any(d[2] > 0)  # (exp underflows to 0 for large sums)


def test_context_parallel_scan_over_rows():
    """One long sequence cut into 4 rows of one launch: a local pass (h0 = 0)
    gives each row's (decay, h_last); composing them row by row gives every
    row's true h0, and a second pass reproduces the uncut sequence (oracle)."""
    G, L, Dn, N = 4, 256, 64, 16
    pos, u, T, P, z, h0, dh = problem(G, Dn, L, N, "one", "f32", seed=96)
    pos = (torch.arange(G * L, device="cuda", dtype=torch.int32).view(G, L)).contiguous()
    zero = torch.zeros((G, Dn, N), device="cuda")
    _, _, hl, dec = pm.pm_selective_scan_fwd_ex(u, T["dt"], P["A"], T["B"], T["C"], P["D"],
                                                P["dt_bias"], pos, h0=zero, want_last_state=True,
                                                want_decay=True)
    hin = torch.zeros_like(zero)
    for k in range(1, G):  # the exchange: G x (Dn x N) summaries
        hin[k] = dec[k - 1] * hin[k - 1] + hl[k - 1]
    out, _, hl2 = pm.pm_selective_scan_fwd_ex(u, T["dt"], P["A"], T["B"], T["C"], P["D"],
                                              P["dt_bias"], pos, h0=hin, want_last_state=True)
    torch.cuda.synchronize()
    cat = lambda t: np.concatenate(list(to_np(t)), axis=-1)[None]  # rows -> one long row
    args = (cat(u), cat(T["dt"]), to_np(P["A"]), cat(T["B"]), cat(T["C"]), to_np(P["D"]),
            to_np(P["dt_bias"]), np.arange(G * L, dtype=np.int32)[None])
    ro, rhl = oracle.scan_fwd_ext(*args)
    assert rel_err(cat(out), ro) <= 1e-4
    assert rel_err(to_np(hl2)[-1], rhl[0]) <= 1e-4


# --------------------------------------------------------------------------
# backward time split of long segments (latency-bound launches): parts
# coupled by the NEXT-2 algebra inside a row (tsplit.cu)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("io", ["f32", "bf16"])
@pytest.mark.parametrize("feat", ["base", "gate", "next2", "zoh", "gate_next2"])
def test_time_split_parity(monkeypatch, io, feat):
    """PM_TSPLIT=1 cuts every segment longer than 384 steps into up to 4
    chunk-aligned parts for the backward (each part starts from the
    forward's checkpoint; the carry entering its end comes from the reverse
    pre-pass over the following parts): one-sequence rows and long random
    rows, with the gate, h0 / dh_last / dh0 (NEXT-2) and ZOH, against the
    oracle; then the same launch without the split agrees to rounding."""
    monkeypatch.setenv("PM_TSPLIT", "1")
    kind = "one" if feat in ("base", "next2") else "random"
    pos, u, T, P, z, h0, dh = problem(3, 96, 2048, 16, kind, io, seed=120 + len(feat),
                                      continued=(1,))
    z = z if "gate" in feat else None
    nx = "next2" in feat
    h0_, dh_ = (h0, dh) if nx else (None, None)
    zoh = feat == "zoh"
    res = run_ext(pos, u, T, P, z, h0_, dh_, zoh=zoh)
    check_ext(pos, u, T, P, z, h0_, dh_, io, res, zoh=zoh)
    monkeypatch.setenv("PM_TSPLIT", "0")
    ref = run_ext(pos, u, T, P, z, h0_, dh_, zoh=zoh)
    assert torch.equal(res[0], ref[0])  # the forward is not split
    tol = 2e-2 if io == "bf16" else 1e-4
    for k in ("du", "ddt", "dB", "dC", "dA", "dD", "ddt_bias", "dz", "dh0"):
        if res[2].get(k) is not None:
            assert rel_err(to_np(res[2][k]), to_np(ref[2][k])) <= 10 * tol, k


def test_time_split_recompute_equals_saved(monkeypatch):
    """With the split, the recompute path (states = NULL: the library runs
    its own forward) equals the saved-states path bit for bit."""
    monkeypatch.setenv("PM_TSPLIT", "1")
    pos, u, T, P, z, h0, dh = problem(3, 64, 2048, 16, "one", "f32", seed=131, continued=(0, 2))
    a = run_ext(pos, u, T, P, z, h0, dh, states=True)
    b = run_ext(pos, u, T, P, z, h0, dh, states=False)
    assert torch.equal(a[0], b[0])
    for k in ("du", "ddt", "dA", "dB", "dC", "dD", "ddt_bias", "dz", "dh0"):
        assert torch.equal(a[2][k], b[2][k]), k

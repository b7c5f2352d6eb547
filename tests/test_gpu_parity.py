"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Solution sets are compared per instance with the R21 rule: identical counts of CONVERGED
distinct endpoints and nearest-neighbour agreement within 1e-8 relative per coordinate
(north_star tolerance).  Statuses of non-converged tracks and trajectories are not
compared element-wise ("parity unpinned": FMA contraction and summation order differ).
"""
import numpy as np
import pytest

from hc_inputs import fixtures, rng, systems

pytestmark = pytest.mark.gpu

TOL = 1e-8


@pytest.fixture(scope="module")
def hc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2112_03444_b200 import hc as hcmod
    return hcmod


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def run_td(hc, desc, gamma, st=None):
    s = hc.System.total_degree_homotopy(desc, device=0)
    p0, p1 = s.td_params(gamma)
    X0 = s.td_start()
    res = hc.track_batch(s, _cuda(X0), _cuda(p0), _cuda(p1)[None], st=st)
    res.wait()
    return res, X0


def run_ph(hc, desc, start, p0, p1s, st=None):
    s = hc.System(desc, device=0)
    res = hc.track_batch(s, _cuda(start), _cuda(p0), _cuda(np.atleast_2d(p1s)), st=st)
    res.wait()
    return res


def gpu_set(orc, res, b=0):
    st = res.status.cpu().numpy()[b]
    X = res.x.cpu().numpy()[b]
    return orc.dedup(X[st == 0])[0]


def assert_same_set(orc, A, B, what):
    ok, ua, ub = orc.match_sets(A, B, tol=TOL)
    assert ok, f"{what}: oracle {len(A)} vs gpu {len(B)} solutions, unmatched {ua}/{ub}"


# ------------------------------------------------------------------ the fused LU

@pytest.mark.parametrize("n", list(range(1, 33)))
def test_batched_zgesv_vs_lapack(hc, n):
    """Fig. 3 shape (batch 1000): fused LU + solve vs numpy (LAPACK zgesv); ragged batch."""
    import torch
    g = rng.gen(100 + n)
    B = 1000 + n   # not a multiple of any tile
    A = (g.standard_normal((B, n, n)) + 1j * g.standard_normal((B, n, n))) + 2 * np.eye(n)
    b = g.standard_normal((B, n)) + 1j * g.standard_normal((B, n))
    x, info = hc.batched_zgesv(_cuda(A), _cuda(b))
    torch.cuda.synchronize()
    x = x.cpu().numpy()
    assert np.all(info.cpu().numpy() == 0)
    ref = np.linalg.solve(A, b[..., None])[..., 0]
    err = np.max(np.abs(x - ref), axis=1) / np.maximum(1, np.max(np.abs(ref), axis=1))
    cond = np.linalg.cond(A)
    assert np.all(err <= 1e-13 * cond), (err / cond).max()


def test_batched_zgesv_singular_and_pivoting(hc):
    import torch
    A = np.zeros((4, 3, 3), complex)
    b = np.ones((4, 3), complex)
    A[0] = np.eye(3)
    A[1] = [[0, 1, 0], [1, 0, 0], [0, 0, 1]]          # needs pivoting
    A[2] = [[1, 2, 3], [2, 4, 6], [1, 0, 1]]          # singular
    A[3] = np.eye(3)
    A[3, 1, 1] = np.nan                               # non-finite
    x, info = hc.batched_zgesv(_cuda(A), _cuda(b))
    torch.cuda.synchronize()
    assert list(info.cpu().numpy()) == [0, 0, 1, 1]
    assert np.allclose(x.cpu().numpy()[1], [1, 1, 1])


# ------------------------------------------------------------------ whole tracker

def test_univariate_vs_companion(hc, orc):
    g = rng.gen(21)
    for d in (1, 2, 3, 5, 8):
        c = (g.standard_normal(d + 1) + 1j * g.standard_normal(d + 1))
        res, _ = run_td(hc, systems.univariate(c), rng.gamma(d))
        st = res.status.cpu().numpy()[0]
        assert np.all(st == 0)
        got = res.x.cpu().numpy()[0][:, 0]
        ok, ua, ub = orc.match_sets(got[:, None], np.roots(c[::-1])[:, None], tol=TOL)
        assert ok


def test_katsura6_parity(hc, orc):
    d = systems.katsura(6)
    for seed in (0, 1):
        gam = rng.gamma(seed)
        res, X0 = run_td(hc, d, gam)
        st = res.status.cpu().numpy()[0]
        assert np.all(st == 0), np.bincount(st)
        ref = orc.track(orc.td_homotopy(d, gam), orc.td_start(d.degrees()))
        A = orc.dedup(orc.finite_solutions(ref))[0]
        B = gpu_set(orc, res)
        assert len(B) == 64
        assert_same_set(orc, A, B, f"katsura-6 gamma seed {seed}")
        # start solutions: identical roots of unity on both sides
        assert np.max(np.abs(X0 - orc.td_start(d.degrees()))) <= 1e-15
        # per-track agreement (diagnostic, R21): same start -> same endpoint
        Xg = res.x.cpu().numpy()[0]
        agree = np.mean(np.all(np.abs(Xg - ref.x[0]) <= 1e-6 * np.maximum(1, np.abs(ref.x[0])), axis=1))
        assert agree >= 0.95


def test_cyclic7_parity(hc, orc):
    """Table 1: 924 solutions, same set as the oracle (gamma seed of config 2)."""
    d = systems.cyclic(7)
    gam = rng.gamma(2)
    res, _ = run_td(hc, d, gam)
    B = gpu_set(orc, res)
    ref = orc.track(orc.td_homotopy(d, gam), orc.td_start(d.degrees()))
    A = orc.dedup(orc.finite_solutions(ref))[0]
    assert len(A) == 924
    assert_same_set(orc, A, B, "cyclic-7")
    r = res.resid.cpu().numpy()[0]
    st = res.status.cpu().numpy()[0]
    assert r[st == 0, 0].max() < 1e-10


def test_counters_and_determinism(hc, orc):
    d = systems.katsura(5)
    gam = rng.gamma(7)
    a, _ = run_td(hc, d, gam)
    b, _ = run_td(hc, d, gam)
    assert np.array_equal(a.x.cpu().numpy().view(np.float64), b.x.cpu().numpy().view(np.float64))
    assert np.array_equal(a.counters.cpu().numpy(), b.counters.cpu().numpy())
    c = a.counters.cpu().numpy()[0]
    # steps >= accepted steps >= 1; solves = 4 per successful predictor + newton + polish
    assert np.all(c[:, 0] >= 1) and np.all(c[:, 3] >= 4 * (c[:, 0] - c[:, 1]))
    ref = orc.track(orc.td_homotopy(d, gam), orc.td_start(d.degrees()))
    same = np.all(ref.counters[0] == c, axis=1).mean()
    assert same >= 0.8   # same algorithm: most tracks take identical step sequences


def test_host_memory_path_matches_device_path(hc):
    d = systems.katsura(4)
    s = hc.System.total_degree_homotopy(d, device=0)
    p0, p1 = s.td_params(rng.gamma(3))
    X0 = s.td_start()
    a = hc.track_batch(s, _cuda(X0), _cuda(p0), _cuda(p1)[None])
    a.wait()
    h = hc.track_batch_host(s, X0, p0, p1[None])
    assert np.array_equal(a.x.cpu().numpy().view(np.float64), h.x.view(np.float64))
    assert np.array_equal(a.status.cpu().numpy(), h.status)


def test_fourview_ph_parity(hc, orc):
    """Config 3 shape: 296 starts (oracle TD fixture) -> planted real instances; identical sets,
    planted ground truth recovered (R18), every path converges."""
    d = systems.nview_triangulation(4)
    start = fixtures.read_solutions(fixtures.fixture_path("fourview_start.sols"))
    p0 = fixtures.read_params(fixtures.fixture_path("fourview_p0.params"))
    assert start.shape == (296, 14)
    B = 3
    p1s, xs = rng.fourview_batch(B)
    res = run_ph(hc, d, start, p0, p1s)
    ref = orc.track(orc.ph_homotopy(d, p0), start, p1s=p1s)
    for b in range(B):
        A = orc.dedup(ref.x[b][ref.status[b] == 0])[0]
        G = gpu_set(orc, res, b)
        assert_same_set(orc, A, G, f"4-view instance {b}")
        assert np.min(np.max(np.abs(G - xs[b]), axis=1)) < 1e-8


def test_trifocal_ph_parity_sampled(hc, orc):
    """Config 4 shape on a sample of start solutions: per-track endpoint agreement and GT recovery."""
    d = systems.trifocal_unknown_f()
    start, p0 = fixtures.trifocal_start()
    p1s, xg = rng.trifocal_batch(2)
    res = run_ph(hc, d, start, p0, p1s)
    st = res.status.cpu().numpy()
    X = res.x.cpu().numpy()
    for b in range(2):
        G = X[b][st[b] == 0]
        # planted ground truth is reached by some track (up to the Z2^3 symmetry images)
        imgs = np.array(systems.trifocal_symmetry(xg[b]))
        dist = min(np.min(np.max(np.abs(G - y), axis=1)) for y in imgs)
        assert dist < 1e-8
    sample = np.arange(0, start.shape[0], 97)
    ref = orc.track(orc.ph_homotopy(d, p0), start[sample], p1s=p1s[:1])
    Xg = X[0][sample]
    both = (ref.status[0] == 0) & (st[0][sample] == 0)
    assert both.mean() > 0.8
    close = np.all(np.abs(Xg[both] - ref.x[0][both]) <= TOL * np.maximum(1, np.abs(ref.x[0][both])), axis=1)
    assert close.mean() >= 0.97

"""CPU tests of the toy-MD oracle (oracle/toysim.py): the Philox4x32-10 generator
against the published known-answer vectors, Box-Muller moments, the bonded force
against finite differences of its energy, and the zero-temperature fixed point."""

import math

import numpy as np

from oracle import toysim as OT


def test_philox4x32_10_known_answers():
    # Random123 kat_vectors (philox4x32_10): counter, key -> output
    kats = [
        ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
        ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
        ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
         (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
    ]
    for ctr, key, want in kats:
        got = OT.philox4x32_10(np.array([ctr], dtype=np.uint64), key)[0]
        assert [int(v) for v in got] == list(want)


def test_normals_moments():
    z = np.concatenate([OT.normals(7, 0, t, 64) for t in range(400)]).ravel()
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1.0) < 0.02


def _energy(x, p):
    n = x.shape[0]
    u = 0.0
    for k in range(n - 1):
        d = np.linalg.norm(x[k + 1] - x[k])
        u += 0.5 * p["bond_k"] * (d - p["bond_r0"]) ** 2
    for v in range(1, n - 1):
        a, b = x[v - 1] - x[v], x[v + 1] - x[v]
        c = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
        u += 0.5 * p["angle_k"] * (math.acos(c) - p["theta0"]) ** 2
    return u


def test_bonded_force_is_minus_energy_gradient():
    rng = np.random.default_rng(3)
    p = {"bond_k": 2000.0, "bond_r0": 0.15, "angle_k": 100.0, "theta0": 1.91}
    x = np.cumsum(rng.normal(0, 0.1, size=(7, 3)), axis=0)
    F = OT.bonded_force(x, p)
    h = 1e-6
    for k in range(7):
        for a in range(3):
            xp, xm = x.copy(), x.copy()
            xp[k, a] += h
            xm[k, a] -= h
            fd = -(_energy(xp, p) - _energy(xm, p)) / (2 * h)
            assert abs(fd - F[k, a]) <= 1e-6 * max(1.0, abs(fd))


def test_zero_temperature_fixed_point():
    from paper_1801_02362_b200.toysim import ToySystem

    sysm = ToySystem(temperature=0.0)
    x0 = sysm.initial_chain()
    p = {"bond_k": sysm.bond_k, "bond_r0": sysm.bond_r0, "angle_k": sysm.angle_k, "theta0": sysm.theta0,
         "mob": sysm.mobility, "noise": sysm.noise, "seed": 1, "tau_g": 0}
    _, _, _, x, _, _ = OT.run(p, None, None, x0, 200, mode=0)
    assert np.abs(x - x0).max() < 1e-12


def _toy_params(**kw):
    p = {"bond_k": 2000.0, "bond_r0": 0.15, "angle_k": 100.0, "theta0": 1.9106332362490186, "mob": 8.3e-6,
         "noise": 4.0e-3, "seed": 3, "tau_g": 10, "lam": 100.0, "eps": 4e-4, "hill_h": 1.0, "hill_sigma": 0.3}
    p.update(kw)
    return p


def _chain(n=8):
    x = np.zeros((n, 3))
    for k in range(1, n):
        a = 1.9106332362490186 * (k % 2)
        x[k] = x[k - 1] + 0.15 * np.array([math.cos(0.3 * k), math.sin(0.3 * k) * math.cos(a), math.sin(a) * 0.2])
    return x


def _refs(L=6, n=8):
    rng = np.random.default_rng(4)
    base = _chain(n)
    r = np.stack([base + rng.normal(0.0, 0.02 * (1 + k), size=base.shape) for k in range(L)])
    return r - r.mean(axis=1, keepdims=True)


def test_toy_neighbour_list_counters_and_degenerate_case():
    """SPEC neighbourlist in the toy loop: original mode with M < N charges exactly
    M + (N - M) updates / steps expensive computations per step (SPEC.md:400 identity); M = N
    with stride 1 reproduces the run without a list (same CV series and counters) in both
    modes; the members are the M nearest at each update."""
    refs, q, x0, steps = _refs(), np.arange(6.0), _chain(), 60
    for mode in (1, 2):
        a = OT.run(_toy_params(), refs, q, x0, steps, mode)
        b = OT.run(_toy_params(nl_m=6, nl_stride=1), refs, q, x0, steps, mode)
        np.testing.assert_allclose(b[0], a[0], rtol=1e-12, atol=1e-15)
        assert np.array_equal(b[2], a[2])
    M, stride = 2, 7
    cv, rlog, counters, x, _, st = OT.run(_toy_params(nl_m=M, nl_stride=stride), refs, q, x0, steps, 1)
    updates = len(range(0, steps, stride))
    assert counters[0] == M * steps + (6 - M) * updates
    assert st["active"].shape == (M,) and np.all(np.diff(st["active"]) > 0)
    # close mode: one expensive x<->y fit per step + N on reassignment; M cheap otherwise
    cv, rlog, counters, x, _, st = OT.run(_toy_params(nl_m=M, nl_stride=stride), refs, q, x0, steps, 2)
    reas = int(rlog.sum())
    assert counters[2] == reas and counters[0] == steps + 6 * reas
    assert counters[1] >= M * (steps - reas)

"""CPU oracle for the toy MD driver (SPEC [MODULE] toysim).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).  A plain numpy restatement of
the loop that ``csrc/toysim.cu`` runs on the device, built on this package's
per-pair restatement of the reference geometry (``oracle.kearsley_fit``,
``exact_distance``, ``approx_distance``, ``property_map``, ``path_z``):

* overdamped Langevin, Euler-Maruyama: x += mob F + noise xi
  (mob = dt / (m gamma), noise = sqrt(2 kB T mob));
* forces: harmonic bonds 1/2 k_b (d - r0)^2, harmonic angles 1/2 k_a (theta -
  theta0)^2, plus the metadynamics bias force -dV/ds ds/dx (Eq. 1);
* the path CV per step in the original mode (Alg. 1) or the close-structure
  mode (Alg. 2, strict '>' and first-step reassignment);
* hills of height w, width sigma on s, deposited at the step's s when
  step % tau_G == 0, after that step's force;
* xi: Philox4x32-10 (Salmon et al. 2011, the Random123 round function and key
  schedule) keyed by the seed, counter (bead, step lo, step hi, walker);
  Box-Muller on (c + 0.5) 2^-32.  The integers are identical to the device's.
"""

from __future__ import annotations

import math

import numpy as np

from . import oracle as O

KB = 0.0083144626  # kJ/mol/K

_M0, _M1 = 0xD2511F53, 0xCD9E8D57
_W0, _W1 = 0x9E3779B9, 0xBB67AE85
_MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """ctr: uint64 array [..., 4] of 32-bit words; key: (k0, k1).  Returns [..., 4]."""
    c = [ctr[..., i].astype(np.uint64) for i in range(4)]
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    for _ in range(10):
        p0 = np.uint64(_M0) * c[0]
        p1 = np.uint64(_M1) * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(_MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(_MASK)
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + np.uint64(_W0)) & np.uint64(_MASK)
        k1 = (k1 + np.uint64(_W1)) & np.uint64(_MASK)
    return np.stack(c, axis=-1)


def normals(seed, walker, step, n):
    """[n, 3] standard normals of (walker, step) for beads 0..n-1 (toysim.cu toy_normals)."""
    ctr = np.zeros((n, 4), dtype=np.uint64)
    ctr[:, 0] = np.arange(n, dtype=np.uint64)
    ctr[:, 1] = step & _MASK
    ctr[:, 2] = (step >> 32) & _MASK
    ctr[:, 3] = walker
    c = philox4x32_10(ctr, (seed & _MASK, (seed >> 32) & _MASK)).astype(np.float64)
    u = (c + 0.5) * 2.0 ** -32
    twopi = 6.283185307179586
    r0 = np.sqrt(-2.0 * np.log(u[:, 0]))
    r1 = np.sqrt(-2.0 * np.log(u[:, 2]))
    return np.stack([r0 * np.cos(twopi * u[:, 1]), r0 * np.sin(twopi * u[:, 1]), r1 * np.cos(twopi * u[:, 3])], axis=1)


def bonded_force(x, p):
    """Per-bead force, terms in the device's order (bond left, bond right, angles with
    vertex k-1, k, k+1)."""
    n = x.shape[0]
    F = np.zeros_like(x)

    def angle(v):
        u = x[v - 1] - x[v]
        w = x[v + 1] - x[v]
        nu, nw = math.sqrt(u @ u), math.sqrt(w @ w)
        c = min(1.0, max(-1.0, (u @ w) / (nu * nw)))
        th = math.acos(c)
        sn = max(math.sqrt(max(0.0, 1.0 - c * c)), 1e-12)
        pre = p["angle_k"] * (th - p["theta0"]) / sn
        fa = pre * (w / (nu * nw) - c * u / (nu * nu))
        fb = pre * (u / (nu * nw) - c * w / (nw * nw))
        return fa, fb

    for k in range(n):
        f = np.zeros(3)
        for j in (k - 1, k + 1):
            if 0 <= j < n:
                r = x[j] - x[k]
                d = math.sqrt(r @ r)
                f = f + p["bond_k"] * (d - p["bond_r0"]) / d * r
        if 1 <= k - 1 <= n - 2:
            f = f + angle(k - 1)[1]
        if 1 <= k <= n - 2:
            fa, fb = angle(k)
            f = f - (fa + fb)
        if 1 <= k + 1 <= n - 2:
            f = f + angle(k + 1)[0]
        F[k] = f
    return F


def run(p, refs, q, x0, steps, mode, walker=0, step0=0, state=None, traj_stride=0):
    """One walker.  p: dict of ToyParams fields (bond_k, bond_r0, angle_k, theta0, mob,
    noise, lam, eps, hill_h, hill_sigma, tau_g, seed; optional nl_m, nl_stride: the SPEC
    neighbour list); refs [L, n, 3] centred; mode 0 free / 1 original /
    2 close.  Returns (cv [steps, 4], refresh [steps], counters [3], final x, traj, state)
    -- state carries y, saved rotations, hills and the neighbour list.

    Neighbour list (nl_m = M > 0, stride nl_stride): updated on the first step and then
    whenever step - last_update >= stride (maybe_update) from that step's
    distances to ALL references -- exact in the original mode (N expensive), the Eq. 5
    approximations in the close mode (N cheap) or the exact refit of a reassignment step --
    as the M smallest, ties by lower index; between updates only the M members are
    evaluated (M expensive / M cheap) and s, z and their gradients sum over them
    (SPEC.md:252)."""
    x = np.array(x0, dtype=np.float64)
    n = x.shape[0]
    L = 0 if refs is None else refs.shape[0]
    w = np.full(n, 1.0 / n)
    nl_m, nl_stride = int(p.get("nl_m", 0)), int(p.get("nl_stride", 1))
    st = state or {"y": None, "rays": None, "hills": [], "counters": np.zeros(3, dtype=np.int64),
                   "active": None, "nl_last": None}
    cv = np.zeros((steps, 4))
    rlog = np.zeros(steps, dtype=np.uint8)
    traj = []
    for it in range(steps):
        t = step0 + it
        if traj_stride and t % traj_stride == 0:
            traj.append(x.copy())
        gs = None
        dvds = 0.0
        if mode != 0:
            xc = O.center(x, w)
            fit_xy = None
            if mode == 2 and st["y"] is not None:
                fit_xy = O.kearsley_fit(xc, st["y"], w, with_derivatives=True)
                dxy = float(fit_xy["eigvals"][0])
                refresh = dxy > p["eps"]
            else:
                dxy, refresh = 0.0, True
            dist = np.zeros(L)
            grads = np.zeros((L, n, 3))
            update = nl_m > 0 and (st["nl_last"] is None or t - st["nl_last"] >= nl_stride)
            # the references evaluated this step: all (no list, an update, or a close-mode
            # reassignment, which refits every saved rotation) or the list members
            every = nl_m == 0 or update or (mode == 2 and refresh)
            todo = range(L) if every else st["active"]
            if refresh:
                rots = np.zeros((L, 3, 3)) if mode == 2 else None
                for i in todo:
                    dist[i], grads[i], fit = O.exact_distance(xc, refs[i], w, w, with_rot_term=False)
                    if mode == 2:
                        rots[i] = fit["rot"]
                if mode == 2:
                    st["y"], st["rays"] = xc.copy(), rots
            else:
                for i in todo:
                    dist[i], grads[i] = O.approx_distance(xc, refs[i], st["rays"][i], fit_xy, w, w)
            if update:
                st["active"] = np.sort(np.argsort(dist, kind="stable")[:nl_m])
                st["nl_last"] = t
            act = np.arange(L) if nl_m == 0 else st["active"]
            s, gsa = O.property_map(dist[act], grads[act], q[act], p["lam"])
            z, _ = O.path_z(dist[act], grads[act], p["lam"])
            gs = gsa
            V = 0.0
            for c in st["hills"]:
                d = s - c
                e = p["hill_h"] * math.exp(-0.5 * d * d / p["hill_sigma"] ** 2)
                V += e
                dvds -= e * d / p["hill_sigma"] ** 2
            cv[it] = (s, z, V, dxy)
            rlog[it] = 1 if (mode == 2 and refresh) else 0
            # counters (SPEC msd-engine / neighbourlist: an update step evaluates all N)
            nev = L if every else nl_m
            if mode == 1:
                st["counters"][0] += nev
            else:
                st["counters"][0] += 1
                if refresh:
                    st["counters"][0] += L
                    st["counters"][2] += 1
                else:
                    st["counters"][1] += nev
        F = bonded_force(x, p)
        if gs is not None:
            F = F - dvds * gs
        x = x + p["mob"] * F + p["noise"] * normals(p["seed"], walker, t, n)
        if mode != 0 and p["tau_g"] > 0 and t % p["tau_g"] == 0:
            st["hills"].append(cv[it, 0])
    return cv, rlog, st["counters"].copy(), x, (np.array(traj) if traj_stride else None), st

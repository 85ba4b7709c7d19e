"""Thin torch-tensor wrappers over the C ABI (one per libmcb200 entry point).

Torch provides device memory and the current stream; every arithmetic step
runs in libmcb200.so.  Shapes follow include/mcb200.h.
"""

from __future__ import annotations

import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .errors import DeviceError

F64 = torch.float64
I32 = torch.int32
U8 = torch.uint8


def require_cuda(t=None):
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    if t is not None and not t.is_cuda:
        raise DeviceError("expected a CUDA tensor")
    _lib.load()


def npad_for(n):
    return ((int(n) + 31) // 32) * 32


class Centred:
    """Centred planes + per-structure scalars of a batch of structures."""

    __slots__ = ("planes", "wplanes", "centroid", "g", "wbar", "mom", "flags", "n", "npad", "count")

    def __init__(self, planes, wplanes, centroid, g, wbar, mom, flags, n, npad):
        self.planes, self.wplanes, self.centroid, self.g = planes, wplanes, centroid, g
        self.wbar, self.mom, self.flags = wbar, mom, flags
        self.n, self.npad, self.count = n, npad, planes.shape[0]


def center(coords, w_align, w_disp, weighted=False, moments=False, recenter=True):
    """K1: coords [B, n, 3] (f32/f64, CUDA) -> Centred.  w_* are [n] fp64 CUDA tensors."""
    require_cuda(coords)
    coords = coords.contiguous()
    b, n, _ = coords.shape
    npad = npad_for(n)
    dev = coords.device
    dt = _lib.MC_F64 if coords.dtype == torch.float64 else _lib.MC_F32
    if coords.dtype not in (torch.float32, torch.float64):
        raise DeviceError("coords must be float32 or float64")
    planes = torch.empty((b, 3, npad), dtype=F64, device=dev)
    wplanes = torch.empty((b, 3, npad), dtype=F64, device=dev) if weighted else None
    centroid = torch.empty((b, 3), dtype=F64, device=dev)
    g = torch.empty((b,), dtype=F64, device=dev)
    wbar = torch.empty((b, 3), dtype=F64, device=dev)
    mom = torch.empty((b, 6), dtype=F64, device=dev) if moments else None
    flags = torch.empty((b,), dtype=U8, device=dev)
    call("mc_center", ptr(coords), dt, b, n, npad, ptr(w_align) if recenter else None, ptr(w_disp), ptr(planes),
         ptr(wplanes), ptr(centroid), ptr(g), ptr(wbar), ptr(mom), ptr(flags), stream_ptr())
    return Centred(planes, wplanes, centroid, g, wbar, mom, flags, n, npad)


def cov_dense(fr: Centred, lm: Centred):
    """S [T, L, 9] fp64 from frame planes and weighted landmark planes."""
    T, L = fr.count, lm.count
    S = torch.empty((T, L, 9), dtype=F64, device=fr.planes.device)
    call("mc_cov_f64", ptr(fr.planes), ptr(lm.wplanes), T, L, fr.npad, ptr(S), stream_ptr())
    return S


def cov_dmma(frames, fr: Centred, lraw, lm: Centred, w, wuni):
    """S [T, L, 9] fp64 (the cov_dense contract) on the fp64 tensor cores from raw
    fp32 frames / landmarks and the centroids / w-sums of their Centred objects
    (uniform displacement weight wuni)."""
    T, n = frames.shape[0], frames.shape[1]
    L = lraw.shape[0]
    S = torch.empty((T, L, 9), dtype=F64, device=frames.device)
    call("mc_cov_dmma", ptr(frames), ptr(fr.centroid), ptr(fr.wbar), ptr(lraw), ptr(lm.centroid), ptr(lm.wbar), ptr(w),
         float(wuni), T, L, n, ptr(S), stream_ptr())
    return S


def close_grad_fix(wres, close, w, frames, fcentroid, ds, dz):
    """Adds the Eq. 6 dR_xy term of the non-refresh frames of wres's chunk to ds / dz
    (full [T, n, 3] arrays) after pathcv_grad_block wrote the contraction part."""
    T, t0 = wres["count"], wres["t0"]
    call("mc_close_grad_fix", T, t0, frames.shape[1], ptr(close["refresh"]), ptr(close["ridx"]), ptr(close["xyeig"]),
         ptr(wres["fvec"]), ptr(w), ptr(frames), ptr(fcentroid), ptr(ds), ptr(dz),
         1 if ds.dtype == torch.float32 else 0, stream_ptr())


def cov_pairs(xplanes, aplanes, xi, ai, npad, w):
    P = int(xi.shape[0]) if xi is not None else int(xplanes.shape[0])
    S = torch.empty((P, 9), dtype=F64, device=xplanes.device)
    call("mc_cov_pairs", ptr(xplanes), ptr(aplanes), ptr(xi), ptr(ai), P, npad, ptr(w), ptr(S), stream_ptr())
    return S


def fit_dense(S, gx, ga, rowmask=None, D=None, want_rot=True, want_quat=False, want_flags=True):
    T, L = S.shape[0], S.shape[1]
    dev = S.device
    D = torch.empty((T, L), dtype=F64, device=dev) if D is None else D
    rot = torch.empty((T, L, 9), dtype=F64, device=dev) if want_rot else None
    quat = torch.empty((T, L, 4), dtype=F64, device=dev) if want_quat else None
    flags = torch.zeros((T, L), dtype=U8, device=dev) if want_flags else None
    call("mc_fit_dense", ptr(S), T, L, ptr(gx), ptr(ga), ptr(rowmask), ptr(D), ptr(rot), ptr(quat), ptr(flags),
         stream_ptr())
    return D, rot, quat, flags


def fit_list_msd(S, xi, ai, gx, ga):
    P = int(S.shape[0])
    D = torch.empty((P,), dtype=F64, device=S.device)
    call("mc_fit_list_msd", ptr(S), P, ptr(xi), ptr(ai), ptr(gx), ptr(ga), ptr(D), stream_ptr())
    return D


def fit_full(S, gx, ga, xi=None, ai=None):
    P = int(S.shape[0])
    dev = S.device
    eig = torch.empty((P, 20), dtype=F64, device=dev)
    quat = torch.empty((P, 4), dtype=F64, device=dev)
    rot = torch.empty((P, 9), dtype=F64, device=dev)
    flags = torch.empty((P,), dtype=U8, device=dev)
    call("mc_fit_full", ptr(S), P, ptr(xi), ptr(ai), ptr(gx), ptr(ga), ptr(eig), ptr(quat), ptr(rot), ptr(flags),
         stream_ptr())
    return eig, quat, rot, flags


def rot_grad(xplanes, aplanes, n, npad, w, eig, xi=None, ai=None):
    P = int(eig.shape[0])
    out = torch.empty((P, n, 3, 3, 3), dtype=F64, device=eig.device)
    call("mc_rot_grad", ptr(xplanes), ptr(aplanes), ptr(xi), ptr(ai), P, n, npad, ptr(w), ptr(eig), ptr(out),
         stream_ptr())
    return out


def jacobi_n(mats, tol=1e-14, max_sweeps=60):
    """mats [B, n, n] fp64 symmetric (CUDA) -> (vals [B, n], vecs [B, n, n], flags [B])."""
    B, n = mats.shape[0], mats.shape[1]
    vals = torch.empty((B, n), dtype=F64, device=mats.device)
    vecs = torch.empty((B, n, n), dtype=F64, device=mats.device)
    flags = torch.empty((B,), dtype=U8, device=mats.device)
    call("mc_jacobi_n", ptr(mats.contiguous()), B, n, float(tol), int(max_sweeps), ptr(vals), ptr(vecs), ptr(flags),
         stream_ptr())
    return vals, vecs, flags


def jacobi4(mats):
    mats = mats.contiguous()
    B = int(mats.shape[0])
    vals = torch.empty((B, 4), dtype=F64, device=mats.device)
    vecs = torch.empty((B, 4, 4), dtype=F64, device=mats.device)
    flags = torch.empty((B,), dtype=U8, device=mats.device)
    call("mc_jacobi4", ptr(mats), B, ptr(vals), ptr(vecs), ptr(flags), stream_ptr())
    return vals, vecs, flags


def close_decisions(fr: Centred, w, eps, walkers, steps, window=8):
    """Window fits + sequential scan + x<->y spectra.  Returns a dict of device tensors."""
    dev = fr.planes.device
    P = walkers * steps * window
    xi = torch.empty((P,), dtype=I32, device=dev)
    ai = torch.empty((P,), dtype=I32, device=dev)
    call("mc_window_pairs", walkers, steps, window, ptr(xi), ptr(ai), stream_ptr())
    Swin = cov_pairs(fr.planes, fr.planes, xi, ai, fr.npad, w)
    dwin = fit_list_msd(Swin, xi, ai, fr.g, fr.g)
    T = walkers * steps
    refresh = torch.empty((T,), dtype=U8, device=dev)
    ridx = torch.empty((T,), dtype=I32, device=dev)
    dxy = torch.empty((T,), dtype=F64, device=dev)
    fly = torch.zeros((walkers,), dtype=I32, device=dev)
    call("mc_close_scan", ptr(fr.planes), ptr(fr.g), walkers, steps, fr.npad, ptr(w), ptr(dwin), window, float(eps),
         ptr(refresh), ptr(ridx), ptr(dxy), ptr(fly), stream_ptr())
    xyeig = torch.zeros((T, 20), dtype=F64, device=dev)
    rxy = torch.empty((T, 9), dtype=F64, device=dev)
    xyflags = torch.empty((T,), dtype=U8, device=dev)
    call("mc_xy_eig", ptr(fr.planes), ptr(fr.g), T, fr.npad, ptr(w), ptr(refresh), ptr(ridx), ptr(xyeig), ptr(rxy),
         ptr(xyflags), stream_ptr())
    return {"refresh": refresh, "ridx": ridx, "dxy": dxy, "xyeig": xyeig, "rxy": rxy, "xyflags": xyflags,
            "onthefly": fly}


def neighbour_topm(D, M, rows=None):
    """Neighbour-list update on the device (SPEC neighbourlist.maybe_update): for each
    row of D [*, L] (fp32/fp64; the listed ``rows`` or all), the indices of the M
    smallest distances, ties by lower index, ascending -> int32 [nrows, M]."""
    require_cuda(D)
    if D.ndim != 2 or D.stride(1) != 1:
        raise ValueError("D must be a row-major [rows, L] tensor")
    L = D.shape[1]
    rows_t = None if rows is None else rows.to(device=D.device, dtype=I32).contiguous()
    nrows = D.shape[0] if rows_t is None else rows_t.numel()
    idx = torch.empty((nrows, M), dtype=I32, device=D.device)
    dt = _lib.MC_F64 if D.dtype == torch.float64 else _lib.MC_F32
    call("mc_neighbour_topm", ptr(D), dt, nrows, L, D.stride(0), ptr(rows_t), int(M), ptr(idx), stream_ptr())
    return idx


def pathcv_weights(D, q, lam, R, fr, lm, cap, cutoff=50.0, close=None, S=None, L=None, rowlo=None, rowcnt=None,
                   t0=0, count=None, s=None, z=None, nb=None, dmode=0):
    """K4 weights for frames t0 .. t0+count-1.  D/R rows are dense [T, L] or sparse
    windows [T, ld] (rowlo/rowcnt); the significant-list outputs are chunk-local.
    nb = {"idx": [U, M] int32, "row": [T] int32} restricts each row to its active
    neighbour set (dense rows); dmode 1 = fill D only, 2 = D already filled."""
    if nb is not None or dmode:
        return _pathcv_weights_nl(D, q, lam, R, fr, lm, cap, cutoff, close, S, t0, count, s, z, nb, dmode)
    Ttot, ld = D.shape
    T = Ttot - t0 if count is None else count
    L = ld if L is None else L
    dev = D.device
    s = torch.empty((Ttot,), dtype=F64, device=dev) if s is None else s
    z = torch.empty((Ttot,), dtype=F64, device=dev) if z is None else z
    sig_idx = torch.empty((T, cap), dtype=I32, device=dev)
    sig_coef = torch.empty((T, cap, 18), dtype=F64, device=dev)
    nsig = torch.empty((T,), dtype=I32, device=dev)
    fvec = torch.empty((T, 16), dtype=F64, device=dev)
    flags = torch.empty((T,), dtype=U8, device=dev)
    c = close or {}
    call("mc_pathcv_weights", T, t0, L, float(lam), float(cutoff), cap, ld, ptr(rowlo), ptr(rowcnt), ptr(D), ptr(q), ptr(R),
         ptr(fr.wbar), ptr(lm.wbar),
         ptr(c.get("refresh")), ptr(c.get("ridx")), ptr(S if close else None), ptr(c.get("rxy")), ptr(c.get("xyeig")),
         ptr(fr.g if close else None), ptr(lm.g if close else None), ptr(lm.mom if close else None),
         ptr(s), ptr(z), ptr(sig_idx), ptr(sig_coef), ptr(nsig), ptr(fvec), ptr(flags), stream_ptr())
    return {"s": s, "z": z, "sig_idx": sig_idx, "sig_coef": sig_coef, "nsig": nsig, "fvec": fvec, "flags": flags,
            "t0": t0, "count": T}


def shard_rescale(wres, alpha, beta, cap):
    """Rescale a landmark shard's K4 coefficients (wres, in place) to the merged softmax:
    cs' = alpha (cs + beta cz), cz' = alpha cz (alpha, beta: fp64 [T] in wres' row order)."""
    call("mc_shard_rescale", int(wres["count"]), int(cap), ptr(wres["nsig"]), ptr(alpha), ptr(beta),
         ptr(wres["sig_coef"]), ptr(wres["fvec"]), stream_ptr())
    return wres


def _pathcv_weights_nl(D, q, lam, R, fr, lm, cap, cutoff, close, S, t0, count, s, z, nb, dmode):
    Ttot, L = D.shape
    T = Ttot - t0 if count is None else count
    dev = D.device
    s = torch.empty((Ttot,), dtype=F64, device=dev) if s is None else s
    z = torch.empty((Ttot,), dtype=F64, device=dev) if z is None else z
    outs = dmode != 1
    sig_idx = torch.empty((T, cap), dtype=I32, device=dev) if outs else None
    sig_coef = torch.empty((T, cap, 18), dtype=F64, device=dev) if outs else None
    nsig = torch.empty((T,), dtype=I32, device=dev) if outs else None
    fvec = torch.empty((T, 16), dtype=F64, device=dev) if outs else None
    flags = torch.empty((T,), dtype=U8, device=dev) if outs else None
    c = close or {}
    nbi = nb["idx"] if nb is not None else None
    nbr = nb["row"] if nb is not None else None
    call("mc_pathcv_weights_nl", T, t0, L, float(lam), float(cutoff), cap, ptr(nbi), ptr(nbr),
         int(nbi.shape[1]) if nbi is not None else 0, int(dmode), ptr(D), ptr(q), ptr(R), ptr(fr.wbar), ptr(lm.wbar),
         ptr(c.get("refresh")), ptr(c.get("ridx")), ptr(S if close else None), ptr(c.get("rxy")), ptr(c.get("xyeig")),
         ptr(fr.g if close else None), ptr(lm.g if close else None), ptr(lm.mom if close else None),
         ptr(s if outs else None), ptr(z if outs else None), ptr(sig_idx), ptr(sig_coef), ptr(nsig), ptr(fvec),
         ptr(flags), stream_ptr())
    if not outs:
        return None
    return {"s": s, "z": z, "sig_idx": sig_idx, "sig_coef": sig_coef, "nsig": nsig, "fvec": fvec, "flags": flags,
            "t0": t0, "count": T}


def pathcv_grad(wres, fr, lm, w, w_align, cap, out_dtype=F64, close=None, raw=None, perm=None, ds=None, dz=None):
    """K4 gradient pass for the frames of ``wres`` (t0, count).  fr/lm: Centred (fp64
    planes) or, with raw=(frames, landmarks) fp32 AoS tensors, Split objects."""
    Ttot, n = fr.count, fr.n
    t0, T = wres.get("t0", 0), wres.get("count", Ttot)
    dev = wres["s"].device
    ds = torch.empty((Ttot, n, 3), dtype=out_dtype, device=dev) if ds is None else ds
    dz = torch.empty((Ttot, n, 3), dtype=out_dtype, device=dev) if dz is None else dz
    c = close or {}
    if raw is None:
        fpl, lpl, fraw, fcen, lraw, lcen = fr.planes, lm.planes, None, None, None, None
        npad = fr.npad
    else:
        fpl = lpl = None
        fraw, lraw = raw
        fcen, lcen = fr.centroid, lm.centroid
        npad = npad_for(n)
    call("mc_pathcv_grad", T, t0, n, npad, cap, ptr(fpl), ptr(lpl), ptr(w), ptr(w_align),
         ptr(wres["sig_idx"]), ptr(wres["sig_coef"]), ptr(wres["nsig"]), ptr(wres["fvec"]), ptr(c.get("refresh")),
         ptr(c.get("ridx")), ptr(c.get("xyeig")), ptr(ds), ptr(dz), 1 if out_dtype == torch.float32 else 0,
         ptr(fraw), ptr(fcen), ptr(lraw), ptr(lcen), ptr(perm), stream_ptr())
    return ds, dz


class LandmarkDigits:
    """int8 digits of a landmark set for the tensor-core gradient (mc_ldig_prep):
    dig [npad, kpad / 32, 4, 32] int8 (the 4 digits of each 32-byte k-step of an atom's
    row interleaved), eB [npad] int32 (per-atom power-of-two scale)."""

    __slots__ = ("dig", "eB", "npad", "kpad", "L", "n")

    def __init__(self, dig, eB, npad, kpad, L, n):
        self.dig, self.eB, self.npad, self.kpad, self.L, self.n = dig, eB, npad, kpad, L, n


def ldig_prep(landmarks, lcen):
    """landmarks [L, n, 3] fp32 raw, lcen [L, 3] fp64 centroids -> LandmarkDigits."""
    L, n = landmarks.shape[0], landmarks.shape[1]
    npad = ((n + 127) // 128) * 128
    kpad = ((3 * L + 31) // 32) * 32
    dev = landmarks.device
    dig = torch.empty((npad, kpad // 32, 4, 32), dtype=torch.int8, device=dev)
    eB = torch.empty((npad,), dtype=I32, device=dev)
    call("mc_ldig_prep", ptr(landmarks.contiguous()), ptr(lcen.contiguous()), L, n, npad, kpad, ptr(eB), ptr(dig),
         stream_ptr())
    return LandmarkDigits(dig, eB, npad, kpad, L, n)


def _grad_i8_ws(T, ncv, dev):
    nb = int(_lib.load().mc_grad_i8_workspace_size(int(T), int(ncv)))
    return torch.empty((nb,), dtype=torch.uint8, device=dev), nb


# groups wider than the resident-image limit (117 landmarks) on the streamed-A int8 kernel
# (env MC_GRAD_I8_WIDE=0: the DMMA kernel, as before)
GRAD_I8_WIDE = __import__("os").environ.get("MC_GRAD_I8_WIDE", "1") == "1"


def _grad_i8_wide(wres, cap, perm, ncv, dev, T):
    """Plan the wide frame groups of a mc_pathcv_grad_i8 call: (wide_ids, nwide, wide_off,
    header workspace, image workspace) or None when no group is wide (one host read)."""
    DG = 8 if ncv == 2 else 16  # frames per group (csrc/grad_i8.cu Cfg<ncv>::DG)
    groups = (T + DG - 1) // DG
    by = torch.empty((groups,), dtype=torch.int64, device=dev)
    call("mc_grad_i8_wide_plan", T, cap, ncv, ptr(wres["sig_idx"]), ptr(wres["nsig"]), ptr(perm), ptr(by),
         stream_ptr())
    ids = torch.nonzero(by).squeeze(1)
    nwide = int(ids.numel())
    if nwide == 0:
        return None
    sz = by[ids]
    off = (torch.cumsum(sz, 0) - sz).contiguous()
    total = int(sz.sum().item())
    hb = int(_lib.load().mc_grad_i8_wide_header_size(nwide, ncv))
    return (ids.to(I32).contiguous(), nwide, off, torch.empty((hb,), dtype=torch.uint8, device=dev), hb,
            torch.empty((total + 256,), dtype=torch.uint8, device=dev))


def _grad_i8_call(wres, fs, ls, frames, landmarks, w, w_align, cap, perm, out_map, ldig, dV, out0, out1, f32, ncv,
                  wide_flag, dev):
    T, n = frames.shape[0], frames.shape[1]
    ws, nb = _grad_i8_ws(T, ncv, dev)
    plan = _grad_i8_wide(wres, cap, perm, ncv, dev, T) if GRAD_I8_WIDE and n % 4 == 0 else None
    wf = wide_flag
    if wf is None and (plan is not None or (GRAD_I8_WIDE and n % 4 == 0)):
        # a non-NULL flag keeps the wide groups out of the narrow call (the streamed-A kernel
        # runs them) and skips the DMMA fallback launch when there are none
        wf = torch.zeros((1,), dtype=I32, device=dev)
    call("mc_pathcv_grad_i8", T, n, cap, ptr(frames), ptr(fs.centroid), ptr(landmarks), ptr(ls.centroid), ptr(w),
         ptr(w_align), ptr(ldig.dig), ptr(ldig.eB), ldig.npad, ldig.kpad, ptr(wres["sig_idx"]),
         ptr(wres["sig_coef"]), ptr(wres["nsig"]), ptr(wres["fvec"]), ptr(dV), ptr(perm), ptr(out_map), ptr(out0),
         ptr(out1), f32, ncv, ptr(wf), ptr(ws), nb, stream_ptr())
    if plan is not None:
        ids, nwide, off, hws, hb, wimg = plan
        call("mc_pathcv_grad_i8_wide", T, n, cap, ptr(frames), ptr(fs.centroid), ptr(w), ptr(w_align), ptr(ldig.dig),
             ptr(ldig.eB), ldig.npad, ldig.kpad, ptr(wres["sig_idx"]), ptr(wres["sig_coef"]), ptr(wres["nsig"]),
             ptr(wres["fvec"]), ptr(dV), ptr(perm), ptr(out_map), ptr(out0), ptr(out1), f32, ncv, ptr(ids), nwide,
             ptr(off), ptr(hws), hb, ptr(wimg), stream_ptr())
        if wide_flag is not None:
            wide_flag.zero_()  # every wide group was written by the streamed-A kernel


def pathcv_grad_block(wres, fs, ls, frames, landmarks, w, w_align, cap, perm, out_dtype=torch.float32,
                      out_map=None, ds=None, dz=None, ldig=None):
    """Blocked gradient pass (fp32 path, exact rows): groups of 8 sorted frames.
    out_map (optional, int32 [T]): the caller's row of frame t -- its raw coordinates
    are read from and its gradients written to that row.  ds / dz: optional outputs.
    ldig (LandmarkDigits): the contraction runs on the int8 tensor cores
    (mc_pathcv_grad_i8; wide groups on DMMA in the same call), else on DMMA."""
    T, n = frames.shape[0], frames.shape[1]
    dev = frames.device
    ds = torch.empty((T, n, 3), dtype=out_dtype, device=dev) if ds is None else ds
    dz = torch.empty((T, n, 3), dtype=out_dtype, device=dev) if dz is None else dz
    f32 = 1 if ds.dtype == torch.float32 else 0
    if ldig is not None:
        _grad_i8_call(wres, fs, ls, frames, landmarks, w, w_align, cap, perm, out_map, ldig, None, ds, dz, f32, 2,
                      None, dev)
        return ds, dz
    call("mc_pathcv_grad_block", T, n, cap, ptr(frames), ptr(fs.centroid), ptr(landmarks), ptr(ls.centroid), ptr(w),
         ptr(w_align), ptr(wres["sig_idx"]), ptr(wres["sig_coef"]), ptr(wres["nsig"]), ptr(wres["fvec"]), ptr(perm),
         ptr(out_map), ptr(ds), ptr(dz), f32, stream_ptr())
    return ds, dz


def pathcv_force_i8(wres, fs, ls, frames, landmarks, w, w_align, cap, perm, ldig, dV, out_dtype=torch.float32,
                    out_map=None, F=None, wide=None):
    """Fused metadynamics bias force F = -(dV/ds ds + dV/dz dz) [T, n, 3] from the K4
    coefficients (one tensor-core contraction instead of ds, dz + mc_mtd_force).
    dV [T, 2] fp64 (indexed like the coefficient rows).  Groups of 16 frames wider than
    117 landmarks are skipped and set wide[0] = 1 (int32 device flag, caller-zeroed)."""
    T, n = frames.shape[0], frames.shape[1]
    F = torch.empty((T, n, 3), dtype=out_dtype, device=frames.device) if F is None else F
    _grad_i8_call(wres, fs, ls, frames, landmarks, w, w_align, cap, perm, out_map, ldig, dV.contiguous(), F, None,
                  1 if F.dtype == torch.float32 else 0, 1, wide, frames.device)
    return F


def sig_span_key(wres, L):
    """Gradient grouping key of each frame: first + last significant landmark (frames
    with similar significant spans land in the same 8-frame group, so the group's
    landmark union -- the K extent of the gradient GEMM -- stays close to one span)."""
    idx, ns = wres["sig_idx"], wres["nsig"].long()
    first = idx[:, 0]
    last = idx.gather(1, (ns - 1).clamp_min(0)[:, None])[:, 0]
    return torch.where(ns > 0, first + last, torch.full_like(first, 2 * L)).contiguous()


def prune_plan(Dc, fnorm, cnorm, c_unit, mind, thr, knear=4, wide=None, maxd=None, cstride=0, frnorm=None,
               crnorm=None, dub_in=None):
    """Per-frame admissible landmark-tile hulls of the metric-pruned screen (csrc/prune.cu).
    dub_in (fp64 [T], landmark-sharded): the D_min upper bound over every shard."""
    T, C = Dc.shape
    ntl = mind.shape[1]
    dev = Dc.device
    hlo = torch.empty((T,), dtype=I32, device=dev)
    hhi = torch.empty((T,), dtype=I32, device=dev)
    key = torch.empty((T,), dtype=I32, device=dev)
    wide = max(1, (3 * ntl) // 4) if wide is None else int(wide)
    call("mc_prune_plan", ptr(Dc), T, C, Dc.stride(0), ptr(fnorm), ptr(cnorm), ptr(frnorm), ptr(crnorm),
         float(c_unit), ptr(mind), ptr(maxd), int(cstride), ntl, float(thr), int(knear), wide, ptr(dub_in), None,
         ptr(hlo), ptr(hhi), ptr(key), stream_ptr())
    return hlo, hhi, key


def screen_bound(Dc, fnorm, cnorm, c_unit, frnorm=None, crnorm=None):
    """Per-frame D_min upper bound min_c (Dc + e_tc) of a coarse one-term screen
    (mc_prune_plan's bound-only pass; landmark-sharded evaluation all-reduces it)."""
    T, C = Dc.shape
    dub = torch.empty((T,), dtype=F64, device=Dc.device)
    call("mc_prune_plan", ptr(Dc), T, C, Dc.stride(0), ptr(fnorm), ptr(cnorm), ptr(frnorm), ptr(crnorm),
         float(c_unit), None, None, 0, 1, 0.0, 1, 1, None, ptr(dub), None, None, None, stream_ptr())
    return dub


def band_tiles(perm, hull_lo, hull_hi, BM, BL, L, ntl):
    """(band, landmark tile) work list of the pruned screen + per-row landmark ranges."""
    T = perm.numel()
    dev = perm.device
    ntm = (T + BM - 1) // BM
    tlist = torch.empty((ntm * ntl, 2), dtype=I32, device=dev)
    nlist = torch.empty((1,), dtype=I32, device=dev)
    rlo = torch.empty((T,), dtype=I32, device=dev)
    rhi = torch.empty((T,), dtype=I32, device=dev)
    call("mc_band_tiles", ptr(perm), T, ptr(hull_lo), ptr(hull_hi), BM, BL, L, ptr(tlist), ptr(nlist), ptr(rlo),
         ptr(rhi), stream_ptr())
    return tlist, nlist, rlo, rhi


def gather_split(sp, idx):
    """The Split of frames idx[0], idx[1], ... (rows of every operand plane and of the
    per-structure scalars gathered on the device; flags are kept as they are)."""
    rows = idx.numel()
    hi = torch.empty((sp.hi.shape[0], rows, sp.hi.shape[2]), dtype=sp.hi.dtype, device=sp.hi.device)
    for p in range(sp.hi.shape[0]):
        call("mc_gather_rows", ptr(sp.hi[p]), 4, sp.hi.shape[2] * sp.hi.element_size() // 4, ptr(idx), rows,
             ptr(hi[p]), stream_ptr())
    lo = None
    if sp.lo is not None:
        lo = torch.empty((sp.lo.shape[0], rows, sp.lo.shape[2]), dtype=sp.lo.dtype, device=sp.lo.device)
        for p in range(sp.lo.shape[0]):
            call("mc_gather_rows", ptr(sp.lo[p]), 4, sp.lo.shape[2], ptr(idx), rows, ptr(lo[p]), stream_ptr())
    g = lambda x: None if x is None else gather_rows(x, idx)  # noqa: E731
    return Split(hi, lo, g(sp.centroid), g(sp.g), g(sp.wbar), g(sp.mom), sp.flags, sp.n, sp.kpad, g(sp.scale),
                 sp.fmt, sp.terms, g(sp.opnorm), g(sp.rnorm), g(sp.dexp))


def gather_rows(src, idx):
    """dst[r] = src[idx[r]] for a contiguous [rows, ...] fp32/fp64 tensor."""
    src = src.contiguous()
    rows = idx.numel()
    dst = torch.empty((rows,) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    rowlen = int(src[0].numel()) if src.shape[0] else 0
    call("mc_gather_rows", ptr(src), src.element_size(), rowlen, ptr(idx), rows, ptr(dst), stream_ptr())
    return dst


def candidates(D, lam, thr, cap, L=None, fnorm=None, fcoef=0.0, rlo=None, rhi=None, dref=None):
    """Per-frame D_min and the window of landmarks with lam (D - D_min) <= thr_t,
    thr_t = thr + fcoef * fnorm[t] (fnorm: optional per-frame fp64 tensor).
    dref (fp32 [T], landmark-sharded): the estimate minimum over every shard."""
    T = D.shape[0]
    L = D.shape[1] if L is None else L
    dev = D.device
    lo = torch.empty((T,), dtype=I32, device=dev)
    cnt = torch.empty((T,), dtype=I32, device=dev)
    dmin = torch.empty((T,), dtype=torch.float32, device=dev)
    flags = torch.empty((T,), dtype=U8, device=dev)
    call("mc_candidates", ptr(D), T, L, D.stride(0), float(lam), float(thr), ptr(fnorm), float(fcoef), ptr(rlo),
         ptr(rhi), ptr(dref), cap, ptr(lo), ptr(cnt), ptr(dmin), ptr(flags), stream_ptr())
    return lo, cnt, dmin, flags


def candidates_life(D, lam, thr, cap, dlife, fnorm=None, fcoef=0.0):
    """mc_candidates with the close-structure lifetime window: row t a refresh frame y,
    dlife [T] fp64 the largest D(x, y) of the frames x that keep y."""
    T, L = D.shape
    dev = D.device
    lo = torch.empty((T,), dtype=I32, device=dev)
    cnt = torch.empty((T,), dtype=I32, device=dev)
    dmin = torch.empty((T,), dtype=torch.float32, device=dev)
    flags = torch.empty((T,), dtype=U8, device=dev)
    call("mc_candidates_life", ptr(D), T, L, D.stride(0), float(lam), float(thr), ptr(fnorm), float(fcoef),
         ptr(dlife.contiguous()), cap, ptr(lo), ptr(cnt), ptr(dmin), ptr(flags), stream_ptr())
    return lo, cnt, dmin, flags


def sort_by_key(key, nbins):
    T = key.shape[0]
    bins = torch.empty((nbins,), dtype=I32, device=key.device)
    perm = torch.empty((T,), dtype=I32, device=key.device)
    call("mc_sort_by_key", ptr(key), T, nbins, ptr(bins), ptr(perm), stream_ptr())
    return perm


class RowDigits:
    """Row digits of B structures (mc_row_digits): dig [3B, kpad/32, 4, 32] int8, e [3B] int32."""

    __slots__ = ("dig", "e", "kpad", "count")

    def __init__(self, dig, e, kpad, count):
        self.dig, self.e, self.kpad, self.count = dig, e, kpad, count


def row_digits(raw, centroid, w=None, perm=None, fmap=None, count=None, out=None, ein=None, planes=False):
    """raw [*, n, 3] fp32 (rows read through fmap / perm), centroid [*, 3] fp64 -> RowDigits.
    planes=True: the digit-plane layout [kpad/32, 4, 3B, 32] (the frame operand of refine_i8)."""
    n = raw.shape[1]
    B = int(count if count is not None else (perm.numel() if perm is not None else raw.shape[0]))
    kpad = ((n + 31) // 32) * 32
    if out is None or out.dig.shape[0] < 3 * B or out.kpad != kpad:
        dig = torch.empty((3 * B, kpad // 32, 4, 32), dtype=torch.int8, device=raw.device)
        e = torch.empty((3 * B,), dtype=I32, device=raw.device)
    else:
        dig, e = out.dig, out.e
    call("mc_row_digits", ptr(raw.contiguous()), ptr(centroid.contiguous()), ptr(w), ptr(perm), ptr(fmap), B, n, kpad,
         ptr(dig), ptr(e), ptr(None if (ein is None or w is not None) else ein.contiguous()), 1 if planes else 0,
         stream_ptr())
    return RowDigits(dig, e, kpad, B)


def refine_i8(ldig, fdig, T, L, n, gx, ga, perm=None, lo=None, cnt=None, cap=0, want_rot=True, Dd=None):
    """mc_refine on the int8 tensor cores from landmark / frame row digits (same outputs as refine)."""
    dev = gx.device
    Dex = torch.empty((T, cap), dtype=F64, device=dev) if cap else None
    Rex = torch.empty((T, cap, 9), dtype=F64, device=dev) if (cap and want_rot) else None
    flags = torch.zeros((T,), dtype=U8, device=dev)
    call("mc_refine_i8", ptr(ldig.dig), ptr(ldig.e), ptr(fdig.dig), ptr(fdig.e), T, L, n, ldig.kpad, ptr(perm),
         ptr(lo), ptr(cnt), ptr(gx), ptr(ga), cap, ptr(Dex), ptr(Rex), ptr(Dd),
         Dd.stride(0) if Dd is not None else 0, ptr(flags), stream_ptr())
    return Dex, Rex, flags


def refine_i8_close(ldig, fdig, T, L, n, gx, ga, perm, lo, cnt, cap, fitmask):
    """Pruned close-structure replay: S [T, cap, 9] of every window pair, fits (D [T, cap],
    R [T, cap, 9]) on the rows with fitmask (mc_refine_i8_close)."""
    dev = gx.device
    Sex = torch.empty((T, cap, 9), dtype=F64, device=dev)
    Dex = torch.empty((T, cap), dtype=F64, device=dev)
    Rex = torch.empty((T, cap, 9), dtype=F64, device=dev)
    flags = torch.zeros((T,), dtype=U8, device=dev)
    call("mc_refine_i8_close", ptr(ldig.dig), ptr(ldig.e), ptr(fdig.dig), ptr(fdig.e), T, L, n, ldig.kpad, ptr(perm),
         ptr(lo), ptr(cnt), ptr(gx), ptr(ga), cap, ptr(fitmask), ptr(Sex), ptr(Dex), ptr(Rex), ptr(flags), stream_ptr())
    return Sex, Dex, Rex, flags


def refine(frames, fsplit, landmarks, lsplit, w, perm=None, lo=None, cnt=None, cap=0, want_rot=True, Dd=None,
           fmap=None, wuni=0.0):
    """Exact fp64 fits of the in-window pairs (sparse) or of all pairs (dense, into Dd).
    fmap (optional int32 [T]): frame t's row in `frames` (per-frame scalars indexed by t)."""
    T, n = frames.shape[0], frames.shape[1]
    L = landmarks.shape[0]
    dev = frames.device
    Dex = torch.empty((T, cap), dtype=F64, device=dev) if cap else None
    Rex = torch.empty((T, cap, 9), dtype=F64, device=dev) if (cap and want_rot) else None
    flags = torch.zeros((T,), dtype=U8, device=dev)
    call("mc_refine", ptr(frames), ptr(fsplit.centroid), ptr(landmarks), ptr(lsplit.centroid), ptr(lsplit.wbar),
         ptr(w), ptr(fsplit.g),
         ptr(lsplit.g), T, L, n, ptr(perm), ptr(lo), ptr(cnt), cap, ptr(Dex), ptr(Rex), ptr(Dd),
         Dd.stride(0) if Dd is not None else 0, ptr(fmap), ptr(fsplit.wbar if wuni > 0 else None), float(wuni),
         ptr(flags), stream_ptr())
    return Dex, Rex, flags


# ---------------------------------------------------------------- fp32 / tensor-core path

def kpad_for(n, fmt="tf32", terms=3):
    q = (64 if terms == 1 else 32) if fmt == "f16" else 16
    return ((int(n) + q - 1) // q) * q


OPERAND_FMT = __import__("os").environ.get("MC_OPERAND_FMT", "f16")


class Split:
    """Split operand planes: TF32 hi/lo fp32 words [3, B, kpad] each, or (F16) one
    interleaved tensor hi [3, B, 2 kpad] of scaled IEEE halves (lo None) with
    scale = 2^-e per structure; + per-structure scalars."""

    __slots__ = ("hi", "lo", "scale", "fmt", "terms", "opnorm", "rnorm", "centroid", "g", "wbar", "mom", "flags", "n",
                 "kpad", "count", "dexp")

    def __init__(self, hi, lo, centroid, g, wbar, mom, flags, n, kpad, scale=None, fmt="tf32", terms=3, opnorm=None,
                 rnorm=None, dexp=None):
        self.hi, self.lo, self.centroid, self.g, self.wbar, self.mom, self.flags = hi, lo, centroid, g, wbar, mom, flags
        self.scale, self.fmt, self.terms, self.opnorm, self.rnorm = scale, fmt, terms, opnorm, rnorm
        self.n, self.kpad, self.count = n, kpad, hi.shape[1]
        self.dexp = dexp  # [count, 3] int32 row-digit exponents (uniform-weight K1s) or None


# uniform-weight one-term K1s (mc_center_split16_uniform); env MC_K1_UNIFORM=0 disables
K1_UNIFORM = __import__("os").environ.get("MC_K1_UNIFORM", "1") == "1"


def center_split(coords, w_align, w_disp, weighted, moments=False, fmt=None, terms=3, wuni=0.0):
    """K1s: centre, optionally fold w into the operand, split into hi/lo planes
    (fmt "f16": power-of-two scaled IEEE halves, "tf32": TF32 words; default
    env MC_OPERAND_FMT, f16).  terms=1 (f16 only): hi halves only, for the
    one-term screening estimate; the operand 2-norms are returned in .opnorm."""
    require_cuda(coords)
    fmt = fmt or OPERAND_FMT
    if fmt not in ("f16", "tf32"):
        raise ValueError(f"operand format {fmt!r}")
    if terms not in (1, 3) or (terms == 1 and fmt != "f16"):
        raise ValueError(f"terms={terms} with format {fmt!r}")
    coords = coords.contiguous()
    b, n, _ = coords.shape
    kpad = kpad_for(n, fmt, terms)
    dev = coords.device
    dt = _lib.MC_F64 if coords.dtype == torch.float64 else _lib.MC_F32
    opnorm = rnorm = None
    if fmt == "f16":  # interleaved [hi x32 | lo x32] rows (one-term: hi rows)
        hi = torch.empty((3, b, kpad if terms == 1 else 2 * kpad), dtype=torch.float16, device=dev)
        lo = None
        opnorm = torch.empty((b,), dtype=F64, device=dev)
        rnorm = torch.empty((b,), dtype=F64, device=dev) if terms == 1 else None
    else:
        hi = torch.empty((3, b, kpad), dtype=torch.float32, device=dev)
        lo = torch.empty((3, b, kpad), dtype=torch.float32, device=dev)
    scale = torch.empty((b,), dtype=F64, device=dev) if fmt == "f16" else None
    centroid = torch.empty((b, 3), dtype=F64, device=dev)
    g = torch.empty((b,), dtype=F64, device=dev)
    wbar = torch.empty((b, 3), dtype=F64, device=dev)
    mom = torch.empty((b, 6), dtype=F64, device=dev) if moments else None
    flags = torch.empty((b,), dtype=U8, device=dev)
    if (fmt == "f16" and terms == 1 and wuni > 0.0 and K1_UNIFORM and not weighted and not moments
            and dt == _lib.MC_F32 and n % 4 == 0 and coords.data_ptr() % 16 == 0):
        dexp = torch.empty((b, 3), dtype=I32, device=dev)
        call("mc_center_split16_uniform", ptr(coords), b, n, kpad, float(wuni), ptr(hi), ptr(scale), ptr(opnorm),
             ptr(rnorm), ptr(centroid), ptr(g), ptr(wbar), ptr(flags), ptr(dexp), stream_ptr())
        return Split(hi, lo, centroid, g, wbar, mom, flags, n, kpad, scale, fmt, terms, opnorm, rnorm, dexp)
    elif fmt == "f16":
        call("mc_center_split16", ptr(coords), dt, b, n, kpad, ptr(w_align), ptr(w_disp), 1 if weighted else 0,
             terms, ptr(hi), ptr(scale), ptr(opnorm), ptr(rnorm), ptr(centroid), ptr(g), ptr(wbar), ptr(mom),
             ptr(flags), stream_ptr())
    else:
        call("mc_center_split", ptr(coords), dt, b, n, kpad, ptr(w_align), ptr(w_disp), 1 if weighted else 0,
             ptr(hi), ptr(lo), ptr(centroid), ptr(g), ptr(wbar), ptr(mom), ptr(flags), stream_ptr())
    return Split(hi, lo, centroid, g, wbar, mom, flags, n, kpad, scale, fmt, terms, opnorm, rnorm)


TF32_2SM = __import__("os").environ.get("MC_TF32_2SM", "0") == "1"


def msd_estimate(fr: Split, lm: Split, D=None, grid=0, two_sm=None, tlist=None, nlist=None):
    """K2+K3: MSD estimate of every (frame, landmark) pair on tcgen05 (fp32 [T, L]),
    in the operand format of the splits.  two_sm (default: env MC_TF32_2SM, on)
    selects the CTA-pair kernel."""
    if fr.fmt != lm.fmt or fr.kpad != lm.kpad or fr.terms != lm.terms:
        raise ValueError("frame and landmark splits differ in format / terms / padding")
    T, L = fr.count, lm.count
    if D is None:
        D = torch.empty((T, L), dtype=torch.float32, device=fr.hi.device)
    pair = TF32_2SM if two_sm is None else two_sm
    if fr.fmt == "f16" and (fr.terms == 1 or not pair or tlist is not None):
        call("mc_msd_f16", ptr(fr.hi), ptr(lm.hi), ptr(fr.scale), ptr(lm.scale), ptr(fr.g), ptr(lm.g), T, L, fr.kpad,
             fr.terms, ptr(tlist), ptr(nlist), ptr(D), D.stride(0), grid, stream_ptr())
    elif fr.fmt == "f16":
        call("mc_msd_f16_2sm", ptr(fr.hi), ptr(lm.hi), ptr(fr.scale), ptr(lm.scale), ptr(fr.g), ptr(lm.g), T, L,
             fr.kpad, ptr(D), D.stride(0), grid, stream_ptr())
    else:
        call("mc_msd_tf32_2sm" if pair else "mc_msd_tf32", ptr(fr.hi), ptr(fr.lo), ptr(lm.hi), ptr(lm.lo),
             ptr(fr.g), ptr(lm.g), T, L, fr.kpad, ptr(D), D.stride(0), grid, stream_ptr())
    return D


msd_tf32 = msd_estimate

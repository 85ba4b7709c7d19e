"""Batched device entry points of the hot path.

* ``msd_matrix(frames, landmarks)``      all-pairs aligned MSD  [T, L]
* ``path_cv(frames, landmarks, lam)``    s, z, ds, dz (Alg. 1, exact MSD)
* ``close_structure_replay(...)``        Alg. 2 over a trajectory (or W walkers)

They are the batched counterparts of the reference's per-structure calls
(kearsley_fit, geometry.py:227; SPEC.md exact_distance / approx_distance /
step_close_structure / property_map) on torch CUDA tensors, all arithmetic in
libmcb200.so.  ``PathCV`` keeps the landmark set resident (centred planes,
norms, moments) across calls, the way a metadynamics run reuses it every step.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import kernels as K
from ._lib import FLAG_DEGENERATE, FLAG_NO_CONVERGE, FLAG_NON_FINITE, FLAG_SIG_OVERFLOW
from .errors import ConfigError, DegenerateFitError, EmptyActiveSetError, InvalidStructureError, MetadynError

# lam*(D_i - D_min) beyond which a landmark is dropped from s, z and the gradients:
# its weight is < e^-25 = 1.4e-11 of the leading term, so even L = 8192 dropped
# landmarks change Z by < 1.1e-7 relative.
DEFAULT_CUTOFF = 25.0
# window-selection estimate of PathCVTC.evaluate (env MC_SCREEN: "f16x1" | "split")
SCREEN = os.environ.get("MC_SCREEN", "f16x1")
# metric pruning of the one-term screen (env MC_PRUNE=0 disables)
PRUNE = os.environ.get("MC_PRUNE", "1") == "1"
# CTAs of the screening GEMM (0: one per SM).  Fewer CTAs draw less power: the
# tensor-core screen otherwise trips the board's power cap, and the clock
# recovery after it slows the fp64 kernels that follow.
K2_GRID = int(os.environ.get("MC_K2_GRID", "0"))
# fp32 inputs of the fp64 PathCV engine on the fp64 tensor cores (env MC_CLOSE_DMMA=0:
# the fp64-plane CUDA-core kernels)
CLOSE_DMMA = os.environ.get("MC_CLOSE_DMMA", "1") == "1"
# gradient contraction on the int8 tensor cores (exact int8 digits, csrc/grad_i8.cu);
# env MC_GRAD_I8=0 keeps the fp64 DMMA kernel for every group
GRAD_I8 = os.environ.get("MC_GRAD_I8", "1") == "1"
# exact window refits on the int8 tensor cores (exact int8 digits, csrc/refine_i8.cu);
# env MC_REFINE_I8=0 keeps the fp64 DMMA kernel
REFINE_I8 = os.environ.get("MC_REFINE_I8", "1") == "1"
# pruned close-structure replay (fp32 frames, w = w'): screened lifetime windows per
# refresh frame instead of the dense covariances; env
# MC_CLOSE_PRUNE=0 keeps the dense path
CLOSE_PRUNE = os.environ.get("MC_CLOSE_PRUNE", "1") == "1"
DEFAULT_WINDOW = 8      # speculative close-structure window (frames)
NB_MAX_L = 16384        # neighbour-list active-set bitmap capacity (csrc/pathcv.cu kNbMaxL)


def normalise_weights(w, n, kind, device):
    """geometry.py:49-61 on the host (argument validation), uploaded as fp64."""
    if w is None:
        arr = np.full(n, 1.0 / n)
    else:
        arr = np.array(w.detach().cpu().numpy() if torch.is_tensor(w) else w, dtype=float)
        if arr.shape != (n,):
            raise InvalidStructureError(f"{kind} weights must have length {n}")
        if not np.all(np.isfinite(arr)) or np.any(arr < 0.0):
            raise InvalidStructureError(f"{kind} weights must be finite and non-negative")
        total = arr.sum()
        if total <= 0.0:
            raise InvalidStructureError(f"{kind} weights sum to zero")
        arr = arr / total
    npad = K.npad_for(n)
    out = torch.zeros(npad, dtype=torch.float64, device=device)
    out[:n] = torch.from_numpy(arr).to(device)
    return out


def _as_cuda(x, device=None):
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x))
    if x.dtype not in (torch.float32, torch.float64):
        x = x.to(torch.float64)
    dev = device if device is not None else (x.device if x.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    return x.to(dev, non_blocking=True).contiguous()


def _check_shapes(frames, landmarks):
    if frames.ndim != 3 or frames.shape[-1] != 3:
        raise InvalidStructureError(f"frames must be [T, n, 3], got {tuple(frames.shape)}")
    if landmarks.ndim != 3 or landmarks.shape[-1] != 3:
        raise InvalidStructureError(f"landmarks must be [L, n, 3], got {tuple(landmarks.shape)}")
    if frames.shape[1] != landmarks.shape[1]:
        raise InvalidStructureError(f"atom count mismatch: {frames.shape[1]} vs {landmarks.shape[1]}")
    if frames.shape[1] < 2:
        raise InvalidStructureError("a structure needs at least 2 atoms")
    if landmarks.shape[0] < 1:
        raise EmptyActiveSetError("no landmarks")


def _raise_flags(flags, what):
    if flags is None or flags.numel() == 0:
        return
    f = int(torch.bitwise_or.reduce(flags.flatten()).item()) if hasattr(torch.bitwise_or, "reduce") else \
        int(np.bitwise_or.reduce(flags.flatten().cpu().numpy()))
    if f & FLAG_NON_FINITE:
        raise InvalidStructureError(f"{what}: non-finite coordinates or distances")
    if f & FLAG_NO_CONVERGE:
        raise MetadynError(f"{what}: Jacobi diagonalisation did not converge")


def _raise_bits(f, what):
    if f & FLAG_NON_FINITE:
        raise InvalidStructureError(f"{what}: non-finite coordinates or distances")
    if f & FLAG_NO_CONVERGE:
        raise MetadynError(f"{what}: Jacobi diagonalisation did not converge")


def _or_flags(flags):
    return int(np.bitwise_or.reduce(flags.flatten().cpu().numpy())) if flags.numel() else 0


_FLAG_BITS = (1, 2, 4, 8, 16)


_BITS = {}


def _flag_bits_dev(flags):
    """Bitwise OR of a uint8 flag array as a device bool[5] (no host sync; the bit
    table is cached per device, so the call is CUDA-graph capturable after one use)."""
    bits = _BITS.get(flags.device)
    if bits is None:
        bits = _BITS[flags.device] = torch.tensor(_FLAG_BITS, dtype=torch.int32, device=flags.device)
    if flags.numel() == 0:
        return torch.zeros(len(_FLAG_BITS), dtype=torch.bool, device=flags.device)
    return ((flags.flatten().to(torch.int32)[:, None] & bits) != 0).any(0)


# 128-frame bands of the pruned screen sorted by (hull start, hull width): frames that
# start on the same landmark tile are bucketed by how many tiles their hull spans, so a
# band's union is close to its frames' own hulls instead of the widest hull that happens
# to start there (env MC_BAND_WIDTH_SORT=0: by hull start only)
BAND_WIDTH_SORT = os.environ.get("MC_BAND_WIDTH_SORT", "1") == "1"
_WB = 16  # width buckets


def _band_key(key, hlo, hhi, ntl):
    """(sort key, bins) of the pruned screen's frame order: prune_plan's key (0 = wide
    hull, 1 + hull start, ntl + 1 = empty) refined by the hull width."""
    if not BAND_WIDTH_SORT:
        return key, ntl + 2
    width = (hhi - hlo).clamp(0, _WB - 1)
    return (key * _WB + width).to(torch.int32).contiguous(), (ntl + 2) * _WB


def _bits_value(row):
    return sum(b for b, on in zip(_FLAG_BITS, row) if on)


class _Cen:
    """Centroid view of a frame chunk (what the blocked gradient pass reads)."""

    __slots__ = ("centroid",)

    def __init__(self, centroid):
        self.centroid = centroid.contiguous()


class PathCV:
    """Resident landmark set + evaluator for s, z and their atom gradients.

    landmarks [L, n, 3] (fp32/fp64, any device); lam > 0; q [L] properties
    (default: landmark index); w / w_align the displacement and
    alignment weights shared by every structure.
    """

    def __init__(self, landmarks, lam, q=None, w=None, w_align=None, cutoff=DEFAULT_CUTOFF, device=None):
        K.require_cuda()
        lm = _as_cuda(landmarks, device)
        if lm.ndim != 3 or lm.shape[-1] != 3:
            raise InvalidStructureError("landmarks must be [L, n, 3]")
        if lm.shape[0] < 1:
            raise EmptyActiveSetError("no landmarks")
        if not (lam > 0):
            raise ConfigError("lambda must be positive")
        self.device = lm.device
        self.L, self.n = int(lm.shape[0]), int(lm.shape[1])
        if self.n < 2:
            raise InvalidStructureError("a structure needs at least 2 atoms")
        self.lam = float(lam)
        self.cutoff = float(cutoff)
        self.w = normalise_weights(w, self.n, "displacement", self.device)
        self.wa = normalise_weights(w_align, self.n, "alignment", self.device)
        qq = np.arange(self.L, dtype=float) if q is None else np.asarray(
            q.detach().cpu().numpy() if torch.is_tensor(q) else q, dtype=float)
        if qq.shape != (self.L,):
            raise ConfigError("q must have one value per landmark")
        self.q = torch.from_numpy(qq).to(self.device)
        self.lm = K.center(lm, self.wa, self.w, weighted=True, moments=True)
        if _or_flags(self.lm.flags) & FLAG_NON_FINITE:
            raise InvalidStructureError("landmark coordinates contain non-finite values")
        # fp32 coordinates with a uniform displacement weight: the covariances and the
        # gradient contraction run on the fp64 tensor cores from the raw fp32 rows
        # (DESIGN.md "Close structure on DMMA"); fp64 inputs keep the fp64 planes path
        self.wuni = float(self.w[0].item()) if bool((self.w[:self.n] == self.w[0]).all()) else 0.0
        self.lraw = lm.contiguous() if (lm.dtype == torch.float32 and CLOSE_DMMA and self.n % 4 == 0
                                        and self.wuni > 0.0) else None
        self.ldig = K.ldig_prep(self.lraw, self.lm.centroid) if (self.lraw is not None and GRAD_I8) else None
        self._tc = None  # one-term screen + int8 refit engine of the pruned close replay (lazy)

    # ------------------------------------------------------------------
    def _frames(self, frames):
        fr = _as_cuda(frames, self.device)
        _check_shapes(fr, torch.empty((self.L, self.n, 3)))
        c = K.center(fr, self.wa, self.w)
        if _or_flags(c.flags) & FLAG_NON_FINITE:
            raise InvalidStructureError("frame coordinates contain non-finite values")
        return fr, c

    def _dmma(self, raw):
        return self.lraw is not None and raw.dtype == torch.float32

    def _cov(self, raw, fr):
        if self._dmma(raw):
            return K.cov_dmma(raw.contiguous(), fr, self.lraw, self.lm, self.w, self.wuni)
        return K.cov_dense(fr, self.lm)

    def msd_matrix(self, frames, want_rot=False):
        """Exact aligned MSD of every (frame, landmark) pair: D [T, L] fp64."""
        raw, fr = self._frames(frames)
        S = self._cov(raw, fr)
        D, rot, _, flags = K.fit_dense(S, fr.g, self.lm.g, want_rot=want_rot)
        _raise_flags(flags, "msd_matrix")
        return (D, rot) if want_rot else D

    def _cap(self, cap):
        return int(min(self.L, 512) if cap is None else min(cap, self.L))

    def graph(self, T, grad=True, dtype=torch.float64, out_dtype=None):
        """A CUDA-graph replay of evaluate() for T frames of ``dtype`` (PathCVGraph)."""
        return PathCVGraph(self, T, grad=grad, dtype=dtype, out_dtype=out_dtype)

    def evaluate(self, frames, grad=True, cap=None, out_dtype=None):
        """Alg. 1 without neighbour list: exact D_i for every landmark."""
        raw, fr = self._frames(frames)
        S = self._cov(raw, fr)
        D, R, _, flags = K.fit_dense(S, fr.g, self.lm.g, want_rot=True)
        _raise_flags(flags, "path_cv")
        return self._finish(raw, fr, D, R, S, None, grad, cap, out_dtype)

    def close_replay(self, frames, eps, walkers=1, grad=True, window=DEFAULT_WINDOW, cap=None, out_dtype=None,
                     neighbours=None, nl_stride=1):
        """Alg. 2 replay: frames [T, n, 3] (walkers == 1) or [W, S, n, 3].

        neighbours = M: SPEC neighbourlist in close-structure mode -- each walker's
        list is updated at steps 0, nl_stride, 2 nl_stride, ... from that step's
        distances to all landmarks (approximated or exact, as the step has them;
        `mc_neighbour_topm`), and s, z and gradients sum over the active set only."""
        if eps is None or not (eps >= 0):
            raise ConfigError("eps must be >= 0")
        if neighbours is not None and not (1 <= int(neighbours) <= self.L):
            raise ConfigError("neighbour list size must satisfy 1 <= M <= L")
        if neighbours is not None and self.L > NB_MAX_L:
            raise ConfigError(f"neighbour lists support up to {NB_MAX_L} landmarks (the active set is a "
                              f"shared-memory bitmap in the K4 weights kernel); this set has {self.L}")
        if int(nl_stride) < 1:
            raise ConfigError("neighbour list stride must be >= 1")
        fr_in = _as_cuda(frames, self.device)
        if fr_in.ndim == 4:
            walkers, steps = int(fr_in.shape[0]), int(fr_in.shape[1])
            fr_in = fr_in.reshape(walkers * steps, self.n, 3)
        else:
            steps = int(fr_in.shape[0]) // walkers
        raw, fr = self._frames(fr_in)
        close = K.close_decisions(fr, self.w, eps, walkers, steps, window)
        if neighbours is None and self._close_prunable(raw):
            out = self._close_replay_pruned(raw, fr, close, grad, cap, out_dtype)
            if grad and _or_flags(close["xyflags"]) & FLAG_DEGENERATE:
                raise DegenerateFitError("close-structure fit x<->y has a degenerate spectrum")
            out.update(refresh=close["refresh"].bool(), dxy=close["dxy"], ridx=close["ridx"],
                       onthefly=close["onthefly"])
            return out
        S = self._cov(raw, fr)
        D, R, _, flags = K.fit_dense(S, fr.g, self.lm.g, rowmask=close["refresh"], want_rot=True)
        _raise_flags(flags, "close_structure_replay")
        nb = None
        if neighbours is not None:
            # distances of every step (Eq. 5 rows filled in), then the lists at the update steps
            K.pathcv_weights(D, self.q, self.lam, R, fr, self.lm, 1, self.cutoff, close=close, S=S, dmode=1)
            stride = int(nl_stride)
            nupd = (steps + stride - 1) // stride
            k = torch.arange(steps, device=self.device, dtype=torch.int32)
            w_ = torch.arange(walkers, device=self.device, dtype=torch.int32)
            upd_rows = (w_[:, None] * steps + torch.arange(0, steps, stride, device=self.device,
                                                           dtype=torch.int32)[None, :]).reshape(-1)
            nb = {"idx": K.neighbour_topm(D, int(neighbours), rows=upd_rows),
                  "row": (w_[:, None] * nupd + (k // stride)[None, :]).reshape(-1).contiguous()}
        out = self._finish(raw, fr, D, R, S, close, grad, cap, out_dtype, nb=nb)
        if nb is not None:
            out["active"] = nb["idx"][nb["row"].long()]
        if grad and _or_flags(close["xyflags"]) & FLAG_DEGENERATE:
            raise DegenerateFitError("close-structure fit x<->y has a degenerate spectrum")
        out.update(refresh=close["refresh"].bool(), dxy=close["dxy"], ridx=close["ridx"], onthefly=close["onthefly"])
        return out

    def _close_prunable(self, raw):
        return (CLOSE_PRUNE and REFINE_I8 and self._dmma(raw) and self.n < 32768
                and bool(torch.equal(self.w, self.wa)))

    def _close_replay_pruned(self, raw, fr, close, grad, cap, out_dtype):
        """Alg. 2 replay with screened windows instead of the dense [T, L] covariances.

        With one weight vector aligning and measuring, the optimally aligned RMSD d is a
        metric, and for a frame x that keeps the close structure y (D(x, y) <= delta):
        d~_l(x) >= d(x, a_l) >= d(y, a_l) - sqrt(delta) and min_l d~_l(x) <= sqrt(delta) +
        d_min(y) (Eq. 5 with R_xy, R_{a y} optimal).  So every landmark x can need has
        d(y, a_l) <= sqrt(delta) + sqrt((sqrt(delta) + d_min(y))^2 + thr / lam): a window
        of y fixed for y's whole lifetime (delta = the largest D(x, y) of its frames).  Only
        the refresh frames are screened (one-term FP16 tcgen05 estimate with its rigorous
        bound); every frame's covariances with its close structure's window, and the
        refresh frames' fits, come from one int8 tensor-core pass (mc_refine_i8_close);
        the K4 weights evaluate Eq. 5 on the window slots."""
        if self._tc is None:
            self._tc = PathCVTC(self.lraw, self.lam, self.q, self.w[:self.n], self.wa[:self.n], cutoff=self.cutoff,
                                prune=False, device=self.device)
        tc = self._tc
        T = raw.shape[0]
        refresh, ridx = close["refresh"], close["ridx"]
        rows = torch.nonzero(refresh).squeeze(1)
        keep = refresh == 0
        dlife = torch.zeros((T,), dtype=torch.float64, device=self.device)
        dlife.scatter_reduce_(0, ridx[keep].long(), close["dxy"][keep], reduce="amax")
        Dest, _, fsr = tc.estimate(raw[rows], terms=tc.screen_terms, check=False)
        one = tc.screen == "f16x1"
        lo_r, cnt_r, _, cflags = K.candidates_life(Dest, self.lam, tc.cutoff + tc.margin, self.L, dlife[rows],
                                                   fnorm=tc.frame_bound(fsr) if one else None,
                                                   fcoef=2.0 * self.lam if one else 0.0)
        del Dest
        src = (torch.cumsum(refresh.to(torch.int32), 0) - 1)[ridx.long()].long()
        lo, cnt = lo_r[src].contiguous(), cnt_r[src].contiguous()
        ld = max(1, int(cnt.max().item()))
        perm = K.sort_by_key((2 * lo + cnt).to(torch.int32), 2 * self.L + 1)
        fdig = K.row_digits(raw, fr.centroid, None, perm=perm, count=T, planes=True)
        S, D, R, rflags = K.refine_i8_close(tc.rdl, fdig, T, self.L, self.n, fr.g, self.lm.g, perm, lo, cnt, ld,
                                            refresh)
        del fdig
        f = _or_flags(cflags) | _or_flags(rflags)
        if f & FLAG_NON_FINITE:
            raise InvalidStructureError("close_structure_replay: non-finite coordinates or distances")
        if f & FLAG_NO_CONVERGE:
            raise MetadynError("close_structure_replay: Jacobi diagonalisation did not converge")
        out = self._finish(raw, fr, D, R, S, close, grad, cap, out_dtype, rowlo=lo, rowcnt=cnt)
        out["window_lo"], out["window_cnt"] = lo, cnt
        return out

    # significant-list buffers per chunk are bounded to ~this many bytes
    CHUNK_BYTES = 4 << 30

    def _finish(self, raw, fr, D, R, S, close, grad, cap, out_dtype, nb=None, rowlo=None, rowcnt=None):
        T = D.shape[0]
        raw = raw.contiguous()
        cap0 = self._cap(cap)
        dev = D.device
        s = torch.empty((T,), dtype=torch.float64, device=dev)
        z = torch.empty((T,), dtype=torch.float64, device=dev)
        nsig = torch.empty((T,), dtype=torch.int32, device=dev)
        ds = dz = None
        if grad:
            odt = out_dtype or (torch.float64 if raw.dtype == torch.float64 else torch.float32)
            ds = torch.empty((T, self.n, 3), dtype=odt, device=dev)
            dz = torch.empty((T, self.n, 3), dtype=odt, device=dev)
        t0 = 0
        while t0 < T:
            cap = cap0
            chunk = min(T - t0, max(8, self.CHUNK_BYTES // (cap * 160)))
            while True:
                wres = K.pathcv_weights(D, self.q, self.lam, R, fr, self.lm, cap, self.cutoff, close=close, S=S,
                                        t0=t0, count=chunk, s=s, z=z, nb=nb, dmode=2 if nb is not None else 0,
                                        L=self.L, rowlo=rowlo, rowcnt=rowcnt)
                f = _or_flags(wres["flags"])
                if f & FLAG_SIG_OVERFLOW and cap < self.L:
                    cap = self.L
                    chunk = min(chunk, max(8, self.CHUNK_BYTES // (cap * 160)))
                    continue
                break
            if f & FLAG_NON_FINITE:
                raise InvalidStructureError("non-finite distances in the path-CV reduction")
            nsig[t0:t0 + chunk] = wres["nsig"]
            if grad and self._dmma(raw):
                # contraction on DMMA (frame groups by significant span), then the
                # close-structure dR_xy term of the non-refresh rows
                sl = slice(t0, t0 + chunk)
                gperm = K.sort_by_key(K.sig_span_key(wres, self.L), 2 * self.L + 1)
                K.pathcv_grad_block(wres, _Cen(fr.centroid[sl]), self.lm, raw[sl], self.lraw, self.w, self.wa, cap,
                                    gperm, ds=ds[sl], dz=dz[sl], ldig=self.ldig)
                if close is not None:
                    K.close_grad_fix(wres, close, self.w, raw, fr.centroid, ds, dz)
            elif grad:
                K.pathcv_grad(wres, fr, self.lm, self.w, self.wa, cap, odt, close=close, ds=ds, dz=dz)
            t0 += chunk
        out = {"s": s, "z": z, "D": D, "nsig": nsig}
        if grad:
            out["ds"], out["dz"] = ds, dz
        return out


class PathCVGraph:
    """CUDA-graph replay of ``PathCV.evaluate`` for a fixed frame count (the small,
    launch-bound configurations: config 0 is ~0.12 ms of kernels behind ~0.23 ms of
    launches and host checks).  The whole pipeline -- centring, covariances, fits,
    K4 weights over every landmark (capacity L: no overflow retry), gradients -- is
    captured once on static buffers; ``evaluate(frames)`` copies the frames in,
    replays the graph and returns the static output tensors (overwritten by the next
    call).  No host synchronisation inside: the status bits of every stage are
    OR-ed on the device and raised by ``check()`` (call it whenever convenient)."""

    def __init__(self, pcv: "PathCV", T, grad=True, dtype=torch.float64, out_dtype=None):
        if int(T) < 1:
            raise ConfigError("graph frame count must be >= 1")
        if int(T) * pcv.L * 160 > 2 ** 31:
            raise ConfigError("graph mode keeps every landmark's coefficients: T * L too large")
        self.pcv, self.T, self.grad = pcv, int(T), bool(grad)
        self.x = torch.zeros((self.T, pcv.n, 3), dtype=dtype, device=pcv.device)
        self.out_dtype = out_dtype
        side = torch.cuda.Stream(device=pcv.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up: one-time attributes, allocator pools
            self._pipeline()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize(pcv.device)
        self.graph = torch.cuda.CUDAGraph()
        from . import _lib

        n0 = _lib.COUNTERS["launches"]
        with torch.cuda.graph(self.graph):
            self.out = self._pipeline()
        self.launches = _lib.COUNTERS["launches"] - n0  # library kernels per replay

    def _pipeline(self):
        p = self.pcv
        fr = K.center(self.x, p.wa, p.w)
        S = p._cov(self.x, fr)
        D, R, _, fflags = K.fit_dense(S, fr.g, p.lm.g, want_rot=True)
        T = self.T
        s = torch.empty((T,), dtype=torch.float64, device=p.device)
        z = torch.empty((T,), dtype=torch.float64, device=p.device)
        wres = K.pathcv_weights(D, p.q, p.lam, R, fr, p.lm, p.L, p.cutoff, s=s, z=z)
        out = {"s": s, "z": z, "D": D, "nsig": wres["nsig"]}
        if self.grad:
            raw = self.x
            odt = self.out_dtype or (torch.float64 if raw.dtype == torch.float64 else torch.float32)
            ds = torch.empty((T, p.n, 3), dtype=odt, device=p.device)
            dz = torch.empty((T, p.n, 3), dtype=odt, device=p.device)
            if p._dmma(raw):
                gperm = K.sort_by_key(K.sig_span_key(wres, p.L), 2 * p.L + 1)
                K.pathcv_grad_block(wres, fr, p.lm, raw, p.lraw, p.w, p.wa, p.L, gperm, ds=ds, dz=dz, ldig=p.ldig)
            else:
                K.pathcv_grad(wres, fr, p.lm, p.w, p.wa, p.L, odt, ds=ds, dz=dz)
            out["ds"], out["dz"] = ds, dz
        out["status"] = torch.stack([_flag_bits_dev(fr.flags), _flag_bits_dev(fflags), _flag_bits_dev(wres["flags"])])
        return out

    def evaluate(self, frames):
        """Copy ``frames`` [T, n, 3] (host or device) in, replay; returns the static outputs."""
        if tuple(frames.shape) != (self.T, self.pcv.n, 3):
            raise InvalidStructureError(f"graph captured for frames [{self.T}, {self.pcv.n}, 3]")
        from . import _lib

        self.x.copy_(frames, non_blocking=True)
        self.graph.replay()
        _lib.COUNTERS["launches"] += self.launches
        return self.out

    def check(self):
        """Raise the errors evaluate() would have raised for the last replay (one host read)."""
        ff, fit, wf = (_bits_value(r) for r in self.out["status"].cpu().tolist())
        if ff & FLAG_NON_FINITE:
            raise InvalidStructureError("frame coordinates contain non-finite values")
        _raise_bits(fit, "path_cv")
        if wf & FLAG_NON_FINITE:
            raise InvalidStructureError("non-finite distances in the path-CV reduction")


class PathCVTC:
    """fp32-coordinate path (configs 2-4): tcgen05 3xTF32 screening + exact refinement.

    evaluate():  K1s split -> K2/K3 tensor-core MSD estimate of every pair ->
    per-frame candidate window {lam (D_est - D_min) <= cutoff + margin} ->
    frames sorted by window -> exact fp64 refit of the candidates (CUDA
    cores) -> K4 weights on the exact windows -> gradient pass on the raw
    fp32 coordinates.  Landmarks outside a window carry weight < e^-cutoff
    relative to the leading term.

    msd_matrix(exact=True): the dense exact matrix (every pair refit in fp64;
    the 3xTF32 estimate error, ~1e-7..1e-5 absolute, cannot certify the
    1e-6 relative tolerance); exact=False returns the estimate.

    screen: the estimate evaluate() selects windows with.  "f16x1" (default
    with the f16 operand format): one-term FP16 (hi x hi) with the rigorous
    per-pair bound |D_est - D| <= c(n) ||x_t|| ||w a_l|| folded into each
    frame's window threshold; "split": the
    split-precision estimate (3 terms) with the measured margin.  Outputs are
    the exact refits either way.
    """

    def __init__(self, landmarks, lam, q=None, w=None, w_align=None, cutoff=25.0, window_cap=512, device=None,
                 operand_fmt=None, screen=None, prune=None, coarse_stride=None, knear=4, shard=None, route=False,
                 two_phase=False):
        """shard = (rank, world[, bounds]): landmark-sharded evaluation.
        ``landmarks`` (and q) are the FULL set; this engine keeps the contiguous landmarks
        [bounds[rank], bounds[rank + 1]) -- default shard_range(L, rank, world); work-
        balanced bounds from ``landmark_load`` + ``dist.balanced_bounds`` -- with their
        global q, and the landmark-norm maxima of the one-term error bound over the full
        set (identical windows on every shard count).  Evaluate with
        ``evaluate_sharded`` / ``sharded_steps``.  route=True (frame-routed variant,
        DESIGN.md section 7): bounds at multiples of the 48-landmark tile; the engine also
        keeps the GLOBAL coarse screen (coarse landmarks, tile tables) so each rank screens
        only its home frames and routes every frame to the shards its admissible tiles
        live on; evaluate with ``evaluate_routed`` / ``routed_steps``.  two_phase=True (the
        survey's two-phase plan): this engine screens its landmark shard
        for every frame (phase 1) and also keeps the FULL landmark set (``self._full``,
        unpruned) for the exact refits, weights and gradients of the rank's home frames
        (phase 2); evaluate with ``evaluate_two_phase`` / ``two_phase_steps``."""
        K.require_cuda()
        self.fmt = operand_fmt or K.OPERAND_FMT
        self.screen = screen or (SCREEN if self.fmt == "f16" else "split")
        if self.screen not in ("f16x1", "split") or (self.screen == "f16x1" and self.fmt != "f16"):
            raise ConfigError(f"screen {self.screen!r} with operand format {self.fmt!r}")
        lm = _as_cuda(landmarks, device).float().contiguous()
        if lm.ndim != 3 or lm.shape[-1] != 3:
            raise InvalidStructureError("landmarks must be [L, n, 3]")
        if lm.shape[0] < 1:
            raise EmptyActiveSetError("no landmarks")
        if not (lam > 0):
            raise ConfigError("lambda must be positive")
        self.device = lm.device
        self.L, self.n = int(lm.shape[0]), int(lm.shape[1])
        if self.n < 2:
            raise InvalidStructureError("a structure needs at least 2 atoms")
        self.lam, self.cutoff = float(lam), float(cutoff)
        self.window_cap = int(min(window_cap, self.L))
        self.w = normalise_weights(w, self.n, "displacement", self.device)
        self.wa = normalise_weights(w_align, self.n, "alignment", self.device)
        qq = np.arange(self.L, dtype=float) if q is None else np.asarray(
            q.detach().cpu().numpy() if torch.is_tensor(q) else q, dtype=float)
        if qq.shape != (self.L,):
            raise ConfigError("q must have one value per landmark")
        self.shard = None
        self._gprune = None
        self._full = None
        if shard is not None and two_phase and not route:
            self._full = PathCVTC(lm, lam, q, w, w_align, cutoff, window_cap, device, operand_fmt, screen, False,
                                  coarse_stride, knear)
        if shard is not None and route:
            g = PathCVTC(lm, lam, q, w, w_align, cutoff, window_cap, device, operand_fmt, screen, True,
                         coarse_stride, knear)
            if two_phase:  # routed two-phase: the full engine also serves the phase-2 refits
                self._full = g
            if not g.prune:
                raise ConfigError("frame routing needs the metric-pruned screen (>= 16 tiles, equal weights)")
            self._gprune = {"ls_coarse": g.ls_coarse, "mind": g.mind, "maxd": g.maxd, "cstride": g.cstride,
                            "knear": g.knear, "ntl": int(g.mind.shape[1])}
            del g
        if shard is not None:
            from .dist import shard_range
            rank, world = int(shard[0]), int(shard[1])
            if not (0 <= rank < world):
                raise ConfigError(f"shard {shard!r}")
            if len(shard) > 2 and shard[2] is not None:
                b = [int(v) for v in shard[2]]
                if len(b) != world + 1 or b[0] != 0 or b[-1] != self.L or any(x > y for x, y in zip(b, b[1:])):
                    raise ConfigError("shard bounds must be 0 = b_0 <= ... <= b_G = L")
                off, cnt = b[rank], b[rank + 1] - b[rank]
            else:
                b = None
                off, cnt = shard_range(self.L, rank, world)
            if route:
                if b is None or any(x % 48 for x in b[:-1]):
                    raise ConfigError("frame routing needs shard bounds at multiples of 48 (dist.tile_bounds)")
                self._tile_bounds = [x // 48 for x in b[:-1]] + [(self.L + 47) // 48]
            if cnt < 1:
                raise EmptyActiveSetError(f"landmark shard {rank} of {world} is empty (L = {self.L})")
            if self.screen == "f16x1":
                full = K.center_split(lm, self.wa, self.w, weighted=True, moments=False, fmt=self.fmt, terms=1)
                self._na_max_full = float(full.opnorm.max().item())
                self._nr_max_full = float(full.rnorm.max().item())
                del full
            lm = lm[off:off + cnt].contiguous()
            qq = qq[off:off + cnt]
            self.shard = (rank, world, off, cnt)
            self.L_total = self.L
            self.L = cnt
            self.window_cap = int(min(window_cap, self.L))
        self.q = torch.from_numpy(qq).to(self.device)
        self.lraw = lm
        # uniform displacement weights (the configs' default): the exact refits run on raw,
        # unweighted fp32 operands (refine_dmma RAW mode)
        self.wuni = float(self.w[0].item()) if bool((self.w[:self.n] == self.w[0]).all()) else 0.0
        # uniform w = w': the frame split takes the one-fp64-pass K1s (mc_center_split16_uniform)
        self._k1_wuni = self.wuni if bool(torch.equal(self.w, self.wa)) else 0.0
        self._ls = {}
        self.screen_terms = 1 if self.screen == "f16x1" else 3
        self.ls = self._lsplit(self.screen_terms)
        if _or_flags(self.ls.flags) & FLAG_NON_FINITE:
            raise InvalidStructureError("landmark coordinates contain non-finite values")
        # int8 digits of the centred landmarks for the tensor-core gradient contraction
        self.ldig = K.ldig_prep(self.lraw, self.ls.centroid) if (GRAD_I8 and self.n % 4 == 0) else None
        # ... and of the weighted centred landmark rows (over the atoms) for the exact refits
        self.rdl = K.row_digits(self.lraw, self.ls.centroid, w=self.w) if (REFINE_I8 and self.n < 32768) else None
        self._fdbuf = None
        # estimate error margin (in units of lam * D): the split (22 significant bits,
        # TF32 or scaled-F16 pair) + fp32-accumulation error grows ~ sqrt(n); measured
        # max 6.4e-6 (n=1000) and 6.4e-5 (n=10000)
        self.est_err = 2e-8 * self.n
        self.margin = 2.0 + self.lam * self.est_err
        if self.screen == "f16x1":
            # rigorous one-term bound per pair: |D_est - D| <= 4 ||dS||_F, ||dS||_F <=
            # (2u + u^2 + n 2^-27) ||x_t|| ||w a_l|| (u = 2^-11 rounding of both operands,
            # Cauchy-Schwarz per entry; n 2^-27: fp32 tensor-core accumulation), x1.25
            # safety, + fp32-eigenvector Rayleigh slack.  The window threshold of frame t
            # grows by 2 lam c ||x_t|| max_l ||w a_l|| (pair error + D_min error).
            # With the measured rounding residuals r = ||fl16(v) - v|| of both operands
            # (typically ~0.4 u ||v||) the same argument gives, per pair,
            #   ||dS||_F <= r_t o_l + o_t r_l + r_t r_l + n 2^-27 (o_t + r_t)(o_l + r_l)
            # (o = operand 2-norm), i.e. |D_est - D| <= e_tl = 5 (r_t o_l + o_t r_l + r_t r_l)
            # + kacc (o_t + r_t)(o_l + r_l) + 1e-6 o_t o_l with kacc = 5 n 2^-27 -- about
            # half the u-based bound; frame t's window allowance is 2 lam max_l e_tl.
            u = 2.0 ** -11
            c_unit = 4.0 * (2 * u + u * u + self.n * 2.0 ** -27) * 1.25 + 1e-6
            self.na_max = float(self.ls.opnorm.max().item())
            self.nr_max = float(self.ls.rnorm.max().item())
            if self.shard is not None:  # the D_min error term ranges over every shard's landmarks
                self.na_max, self.nr_max = self._na_max_full, self._nr_max_full
            self.kacc = 5.0 * self.n * 2.0 ** -27
            self.c_unit = c_unit  # the u-based bound (reported by the tests beside e_tl)
            self.margin = 2.0
        # metric pruning of the screen: one-term screen only,
        # worthwhile when there are many landmark tiles
        ntl = (self.L + 47) // 48
        # (RMSD is a pseudometric only when one weight vector both aligns and measures)
        self.prune = ((PRUNE if prune is None else bool(prune)) and self.screen == "f16x1" and ntl >= 16
                      and bool(torch.equal(self.w, self.wa)))
        if self.prune:
            cs = coarse_stride if coarse_stride is not None else int(os.environ.get("MC_COARSE_STRIDE", "32"))
            kn = int(os.environ.get("MC_KNEAR", knear))
            self._init_prune(int(cs), kn)

    def _exact_windows(self, Dest, fr, fs, cap, rlo=None, rhi=None, perm0=None, dref=None):
        """Screen estimate -> per-frame windows (mc_candidates, against dref when sharded)
        -> frames sorted by window centre (32-frame refit unions stay tight) -> exact fp64
        refits of the window pairs (DMMA) -> K4 weights.  Shared by evaluate() and the
        two landmark-sharded generators.  Returns (lo, cnt, wres, cflags, rflags)."""
        one = self.screen == "f16x1"
        lo, cnt, _, cflags = K.candidates(Dest, self.lam, self.cutoff + self.margin, cap,
                                          fnorm=self.frame_bound(fs) if one else None,
                                          fcoef=2.0 * self.lam if one else 0.0, rlo=rlo, rhi=rhi, dref=dref)
        perm = K.sort_by_key((2 * lo + cnt).to(torch.int32), 2 * self.L + 1)
        Dex, Rex, rflags = self._refine_windows(fr, fs, perm, lo, cnt, cap, perm0)
        wres = K.pathcv_weights(Dex, self.q, self.lam, Rex, fs, self.ls, cap, self.cutoff, L=self.L, rowlo=lo,
                                rowcnt=cnt)
        wres["D_window"] = Dex
        return lo, cnt, wres, cflags, rflags

    def _refine_windows(self, fr, fs, perm, lo, cnt, cap, fmap=None):
        """Exact fp64 refits of the window pairs: int8 tensor-core kernel (frame row digits in
        window-sorted order, then mc_refine_i8) or the fp64 DMMA kernel."""
        T = fs.count
        if self.rdl is not None:
            self._fdbuf = K.row_digits(fr, fs.centroid, None, perm=perm, fmap=fmap, count=T, out=self._fdbuf,
                                       ein=fs.dexp, planes=True)
            return K.refine_i8(self.rdl, self._fdbuf, T, self.L, self.n, fs.g, self.ls.g, perm=perm, lo=lo, cnt=cnt,
                               cap=cap)
        return K.refine(fr, fs, self.lraw, self.ls, self.w, perm=perm, lo=lo, cnt=cnt, cap=cap, fmap=fmap,
                        wuni=self.wuni)

    def frame_bound(self, fs):
        """max_l e_tl: the one-term estimate error bound of frame t against any landmark
        (the per-pair bound with the landmark norms at their maxima)."""
        o, r = fs.opnorm, fs.rnorm
        A, dA = self.na_max, self.nr_max
        return (5.0 * (r * (A + dA) + o * dA) + self.kacc * (o + r) * (A + dA) + 1e-6 * o * A).contiguous()

    def _init_prune(self, stride, knear):
        """Coarse landmark subset (every `stride`-th, <= 1024), its one-term split, and
        mind [C, ntl] = a lower bound of min over each 48-landmark tile of the exact
        RMSD coarse -> landmark (exact fp64 refits, stored fp32, shrunk by 1e-6)."""
        stride = max(stride, (self.L + 1023) // 1024)
        self.coarse = torch.arange(0, self.L, stride, device=self.device)
        lc = self.lraw[self.coarse].contiguous()
        self.ls_coarse = K.center_split(lc, self.wa, self.w, weighted=True, moments=False, fmt=self.fmt, terms=1)
        dcl = torch.empty((lc.shape[0], self.L), dtype=torch.float32, device=self.device)
        fsc = K.center_split(lc, self.wa, self.w, weighted=False, fmt=self.fmt)
        _, _, flags = K.refine(lc, fsc, self.lraw, self.ls, self.w, Dd=dcl)
        _raise_flags(flags, "metric pruning: landmark distances")
        ntl = (self.L + 47) // 48
        # exact RMSDs, widened for the fp32 storage of D and the fp64 cancellation near 0
        rm = dcl.double().clamp_min(0.0).sqrt_()
        lo_ = (rm * (1.0 - 1e-6) - 1e-6).clamp_min_(0.0)
        hi_ = rm * (1.0 + 1e-6) + 1e-6
        pad = ntl * 48 - self.L
        lo_ = torch.nn.functional.pad(lo_, (0, pad), value=float("inf"))
        hi_ = torch.nn.functional.pad(hi_, (0, pad), value=0.0)
        self.mind = lo_.view(lo_.shape[0], ntl, 48).amin(2).float().contiguous()
        self.maxd = hi_.view(hi_.shape[0], ntl, 48).amax(2).float().contiguous()
        self.cstride = stride
        self.knear = max(1, min(8, knear))

    def _lsplit(self, terms):
        """Landmark operand split for `terms` (cached; the scalar fields agree)."""
        if terms not in self._ls:
            self._ls[terms] = K.center_split(self.lraw, self.wa, self.w, weighted=True, moments=True, fmt=self.fmt,
                                             terms=terms if self.fmt == "f16" else 3)
        return self._ls[terms]

    def _frames(self, frames, terms=3, check=True):
        fr = _as_cuda(frames, self.device)
        if fr.dtype != torch.float32:
            fr = fr.float()
        _check_shapes(fr, self.lraw)
        fs = K.center_split(fr.contiguous(), self.wa, self.w, weighted=False, fmt=self.fmt,
                            terms=terms if self.fmt == "f16" else 3, wuni=self._k1_wuni)
        if check and _or_flags(fs.flags) & FLAG_NON_FINITE:
            raise InvalidStructureError("frame coordinates contain non-finite values")
        return fr.contiguous(), fs

    def estimate(self, frames, terms=3, check=True):
        """Split-precision (terms=3) or one-term (f16, terms=1) MSD estimate of every pair."""
        fr, fs = self._frames(frames, terms, check)
        return K.msd_estimate(fs, self._lsplit(terms if self.fmt == "f16" else 3)), fr, fs

    def msd_matrix(self, frames, exact=True, out=None):
        """[T, L] fp32 aligned MSDs: exact=True every pair refit exactly (int8 tensor cores,
        or DMMA), exact=False the split-precision estimate.  out: optional [T, L] buffer."""
        # exact refits need only the frames' centroids / G (one-term split: the uniform-weight
        # K1s also yields the row-digit exponents); the estimate needs the split operand
        fr, fs = self._frames(frames, 1 if (exact and self.fmt == "f16" and self.rdl is not None) else 3)
        D = torch.empty((fr.shape[0], self.L), dtype=torch.float32, device=self.device) if out is None else out
        if not exact:
            return K.msd_estimate(fs, self._lsplit(3), D)
        if self.rdl is not None:
            self._fdbuf = K.row_digits(fr, fs.centroid, None, count=fr.shape[0], out=self._fdbuf, ein=fs.dexp,
                                       planes=True)
            _, _, flags = K.refine_i8(self.rdl, self._fdbuf, fr.shape[0], self.L, self.n, fs.g, self.ls.g, Dd=D)
        else:
            _, _, flags = K.refine(fr, fs, self.lraw, self.ls, self.w, Dd=D, wuni=self.wuni)
        _raise_flags(flags, "msd_matrix")
        return D

    def _pruned_estimate(self, frames):
        """Metric-pruned one-term screen: coarse screen -> per-frame admissible tile hulls
        -> frames sorted by hull (perm0) -> banded tensor-core estimate of the sorted
        frames.  Returns the estimate (sorted rows), the caller's raw frames, the sorted
        split, the unsorted split, the row ranges and perm0 (sorted position -> frame)."""
        fr0, fs0 = self._frames(frames, 1, check=False)
        Dc = K.msd_estimate(fs0, self.ls_coarse, grid=K2_GRID)
        hlo, hhi, key = K.prune_plan(Dc, fs0.opnorm, self.ls_coarse.opnorm, self.kacc, self.mind,
                                     (self.cutoff + 2.0) / self.lam, self.knear, maxd=self.maxd, cstride=self.cstride,
                                     frnorm=fs0.rnorm, crnorm=self.ls_coarse.rnorm)
        ntl = self.mind.shape[1]
        perm0 = K.sort_by_key(*_band_key(key, hlo, hhi, ntl))
        # sorted view of the split (operand rows + scalars gathered, no second split); the
        # raw frames stay in place and are read through perm0 (refine fmap / grad out_map)
        fss = K.gather_split(fs0, perm0)
        tlist, nlist, rlo, rhi = K.band_tiles(perm0, hlo, hhi, 128, 48, self.L, ntl)
        Dest = torch.empty((fr0.shape[0], self.L), dtype=torch.float32, device=self.device)
        K.msd_estimate(fss, self.ls, Dest, grid=K2_GRID, tlist=tlist, nlist=nlist)
        self._last_tiles = nlist
        return Dest, fr0, fss, fs0, rlo, rhi, perm0

    def evaluate(self, frames, grad=True, out_dtype=torch.float32, return_estimate=False, bias=None, dV=None):
        """s, z (and with grad the atom gradients ds, dz) of every frame.

        bias (metadynamics.HillStore over (s, z)) or dV ([T, 2] dV/ds, dV/dz per frame, the
        caller's frame order): also the metadynamics bias force F = -(dV/ds ds + dV/dz dz)
        [T, n, 3] (SPEC bias_and_force, Eq. 1) as out["force"] -- computed by ONE fused
        tensor-core contraction over the K4 coefficients (csrc/grad_i8.cu, ncv = 1), so
        grad=False with a bias returns s, z, V and F without materialising ds, dz."""
        if bias is not None and dV is not None:
            raise ConfigError("pass either a HillStore (bias) or dV, not both")
        want_force = bias is not None or dV is not None
        if want_force and bias is not None and getattr(bias, "d", 2) != 2:
            raise ConfigError("the fused force needs a bias over the two path CVs (s, z)")
        rlo = rhi = perm0 = fs0 = None
        if self.prune:
            Dest, fr, fs, fs0, rlo, rhi, perm0 = self._pruned_estimate(frames)
        else:
            Dest, fr, fs = self.estimate(frames, self.screen_terms, check=False)
        cap = self.window_cap
        while True:
            # the whole pipeline is enqueued without host round trips; the status
            # flags of every stage are reduced on the device and read once at the end
            lo, cnt, wres, cflags, rflags = self._exact_windows(Dest, fr, fs, cap, rlo, rhi, perm0)
            Dex = wres["D_window"]
            out = {"s": wres["s"], "z": wres["z"], "window_lo": lo, "window_cnt": cnt, "D_window": Dex,
                   "nsig": wres["nsig"]}
            gperm = None
            if grad or want_force:
                # gradient groups by significant span (the refine groups are by window start)
                gperm = K.sort_by_key(K.sig_span_key(wres, self.L), 2 * self.L + 1)
            if grad:
                out["ds"], out["dz"] = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap,
                                                           gperm, out_dtype, out_map=perm0, ldig=self.ldig)
            wide = None
            if want_force:
                if bias is not None:
                    V, dVs = bias.bias(torch.stack([wres["s"], wres["z"]], 1))  # coefficient-row order
                    out["V"] = V
                else:
                    dVs = torch.as_tensor(dV, dtype=torch.float64).to(self.device).reshape(-1, 2)
                    if dVs.shape[0] != fr.shape[0]:
                        raise ConfigError("dV must be [T, 2]")
                    if perm0 is not None:
                        dVs = dVs[perm0.long()]
                dVs = dVs.contiguous()
                out["_dVs"] = dVs
                if self.ldig is not None:
                    wide = torch.zeros((1,), dtype=torch.int32, device=self.device)
                    out["force"] = K.pathcv_force_i8(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm,
                                                     self.ldig, dVs, out_dtype, out_map=perm0, wide=wide)
            fflags = fs.flags if fs0 is None else torch.cat([fs.flags, fs0.flags])
            status = torch.stack([_flag_bits_dev(fflags), _flag_bits_dev(cflags), _flag_bits_dev(rflags),
                                  _flag_bits_dev(wres["flags"]),
                                  (wide if wide is not None else torch.zeros(1, dtype=torch.int32, device=self.device)
                                   ).bool().expand(len(_FLAG_BITS))])
            ff, cf, rf, wf, wd = (_bits_value(r) for r in status.cpu().tolist())
            if ff & FLAG_NON_FINITE:
                raise InvalidStructureError("frame coordinates contain non-finite values")
            if (cf & FLAG_SIG_OVERFLOW) and cap < self.L:  # rare: a window wider than cap
                cap = min(self.L, 4 * cap)
                continue
            break
        if rf & FLAG_NON_FINITE:
            raise InvalidStructureError("path_cv refine: non-finite coordinates or distances")
        if rf & FLAG_NO_CONVERGE:
            raise MetadynError("path_cv refine: Jacobi diagonalisation did not converge")
        if wf & FLAG_NON_FINITE:
            raise InvalidStructureError("non-finite distances in the path-CV reduction")
        if want_force and (self.ldig is None or wd):
            # a 16-frame group wider than the tensor-core kernel's K extent (or no int8
            # operand): the force from the two gradients (mc_mtd_force, streaming)
            from . import _lib
            from ._lib import call, ptr, stream_ptr
            if "ds" in out:
                ds, dz = out["ds"], out["dz"]
            else:
                ds, dz = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm, out_dtype,
                                             out_map=perm0, ldig=self.ldig)
            # ds, dz rows are in the caller's order (out_map); dV is in coefficient-row order
            dVc = out["_dVs"]
            if perm0 is not None:
                back = torch.empty_like(dVc)
                back[perm0.long()] = dVc
                dVc = back
            F = torch.empty_like(ds)
            n = ds.shape[1]
            call("mc_mtd_force", ptr(dVc.contiguous()), ds.shape[0], 2, ptr(ds), ptr(dz), None,
                 _lib.MC_F64 if ds.dtype == torch.float64 else _lib.MC_F32, n, ptr(F), stream_ptr())
            out["force"] = F
        out.pop("_dVs", None)
        if perm0 is not None:
            out["screen_tiles"] = self._last_tiles  # (band, landmark tile) pairs the pruned screen computed
            # per-frame outputs back to the caller's frame order (the gradients were
            # written in place through out_map); the windows refer to the same rows
            p = perm0.long()
            for key_ in ("s", "z", "window_lo", "window_cnt", "D_window", "nsig", "V"):
                if key_ not in out:
                    continue
                v = out[key_]
                back = torch.empty_like(v)
                back[p] = v
                out[key_] = back
            if return_estimate:
                back = torch.empty_like(Dest)
                back[p] = Dest
                Dest = back
        if return_estimate:
            out["D_est"] = Dest  # pruned: entries outside each band are not computed
        return out


    def evaluate_nl(self, frames, neighbours, nl_stride=1, walkers=1, grad=True, out_dtype=torch.float32):
        """SPEC neighbourlist (``maybe_update``) on the tensor-core path with
        exact distances every frame (Alg. 1): frames [T, n, 3] (one trajectory, or
        ``walkers`` consecutive trajectories) or [W, S, n, 3].  Each walker's list is the M
        landmarks nearest (exact aligned MSD, ties by lower index) to its frames 0, nl_stride,
        2 nl_stride, ...; s, z and the gradients of every frame sum over the active set of
        its last update (SPEC colvar "active set"), like PathCV.close_replay(eps=0,
        neighbours=M) and the oracle.

        Certified top-M without a dense exact matrix: the one-term screen of the update
        frames bounds every pair (|D_est - D| <= e_t); with k_t the M-th smallest estimate,
        any landmark with D_est - e_t > k_t + e_t cannot be among the M nearest, so only the
        candidates' hull is refit exactly (int8 tensor cores) and the exact top-M taken
        among them (mc_neighbour_topm).  Every frame is then refit over the hull of its
        active set; window slots outside the set are masked (D = 1e300, weight 0)."""
        if self.shard is not None:
            raise ConfigError("evaluate_nl runs on an unsharded engine")
        M, stride = int(neighbours), int(nl_stride)
        if not (1 <= M <= self.L):
            raise ConfigError("neighbour list size must satisfy 1 <= M <= L")
        if stride < 1:
            raise ConfigError("neighbour list stride must be >= 1")
        fr_in = _as_cuda(frames, self.device)
        if fr_in.ndim == 4:
            walkers = int(fr_in.shape[0])
            fr_in = fr_in.reshape(-1, self.n, 3)
        T = int(fr_in.shape[0])
        if walkers < 1 or T % walkers:
            raise ConfigError("frames must split into equal walker trajectories")
        steps = T // walkers
        fr, fs = self._frames(fr_in, self.screen_terms)
        dev = self.device
        nupd = (steps + stride - 1) // stride
        w_ = torch.arange(walkers, device=dev, dtype=torch.int32)
        upd = (w_[:, None] * steps + torch.arange(0, steps, stride, device=dev, dtype=torch.int32)[None, :])
        upd = upd.reshape(-1).contiguous()
        k = torch.arange(steps, device=dev, dtype=torch.int32)
        row = (w_[:, None] * nupd + (k // stride)[None, :]).reshape(-1).contiguous()
        # 1. certified candidates of the update frames' top-M
        fsu = K.gather_split(fs, upd)
        Dest = K.msd_estimate(fsu, self._lsplit(self.screen_terms), grid=K2_GRID)
        one = self.screen == "f16x1"
        e = self.frame_bound(fsu) if one else torch.full((upd.numel(),), self.est_err, dtype=torch.float64, device=dev)
        kth = Dest.gather(1, K.neighbour_topm(Dest, M).long()).amax(1).double()
        m = Dest.amin(1).double()
        allow = self.lam * ((kth - m) * (1.0 + 1e-6) + 2.0 * e + 1e-6 * kth.abs() + 1e-12)
        lo_u, cnt_u, _, cflags = K.candidates(Dest, self.lam, 0.0, self.L, fnorm=allow.contiguous(), fcoef=1.0)
        del Dest
        cap_u = max(1, int(cnt_u.max().item()))
        perm_u = K.sort_by_key((2 * lo_u + cnt_u).to(torch.int32), 2 * self.L + 1)
        Dex_u, _, rflags_u = self._refine_windows(fr, fsu, perm_u, lo_u, cnt_u, cap_u, fmap=upd)
        # 2. exact top-M of every update frame among its candidates
        U = upd.numel()
        ri, si = torch.nonzero(torch.arange(cap_u, device=dev)[None, :] < cnt_u[:, None], as_tuple=True)
        Dfull = torch.full((U, self.L), float("inf"), dtype=torch.float64, device=dev)
        Dfull[ri, lo_u[ri].long() + si] = Dex_u[ri, si]
        idx = K.neighbour_topm(Dfull, M)
        del Dfull
        # 3. every frame over the hull of its active set, slots outside the set masked
        lst = idx[row.long()]
        lo = lst.amin(1).contiguous()
        cnt = (lst.amax(1) - lo + 1).contiguous()
        cap = max(1, int(cnt.max().item()))
        perm = K.sort_by_key((2 * lo + cnt).to(torch.int32), 2 * self.L + 1)
        Dex, Rex, rflags = self._refine_windows(fr, fs, perm, lo, cnt, cap)
        mem = torch.zeros((U, self.L), dtype=torch.bool, device=dev)
        mem.scatter_(1, idx.long(), True)
        slot = torch.arange(cap, device=dev)
        inw = slot[None, :] < cnt[:, None]
        cols = (lo[:, None].long() + slot[None, :]).clamp_(max=self.L - 1)
        member = mem[row.long()[:, None], cols] & inw
        Dex.masked_fill_(inw & ~member, 1e300)
        wres = K.pathcv_weights(Dex, self.q, self.lam, Rex, fs, self.ls, cap, self.cutoff, L=self.L, rowlo=lo,
                                rowcnt=cnt)
        out = {"s": wres["s"], "z": wres["z"], "nsig": wres["nsig"], "active": lst, "window_lo": lo,
               "window_cnt": cnt, "D_window": Dex}
        if grad:
            gperm = K.sort_by_key(K.sig_span_key(wres, self.L), 2 * self.L + 1)
            out["ds"], out["dz"] = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm,
                                                       out_dtype, ldig=self.ldig)
        f = (_or_flags(fs.flags) | _or_flags(cflags) | _or_flags(rflags_u) | _or_flags(rflags)
             | _or_flags(wres["flags"]))
        if f & FLAG_NON_FINITE:
            raise InvalidStructureError("evaluate_nl: non-finite coordinates or distances")
        if f & FLAG_NO_CONVERGE:
            raise MetadynError("evaluate_nl: Jacobi diagonalisation did not converge")
        if f & FLAG_SIG_OVERFLOW:
            raise ConfigError("evaluate_nl: more significant landmarks than the list capacity")
        return out

    # ------------------------------------------------------------ landmark sharding

    def landmark_load(self, frames):
        """Per-landmark work of an evaluation of ``frames`` (unsharded engine): how many
        frames' exact windows cover each landmark (refits and gradient rows scale with
        it).  Input to ``dist.balanced_bounds`` for work-balanced landmark shards."""
        out = self.evaluate(frames, grad=False)
        lo, cnt = out["window_lo"].long(), out["window_cnt"].long()
        diff = torch.zeros(self.L + 1, dtype=torch.int64, device=self.device)
        diff.index_add_(0, lo, torch.ones_like(lo))
        diff.index_add_(0, lo + cnt, -torch.ones_like(lo))
        return torch.cumsum(diff[:-1], 0)


    def evaluate_sharded(self, frames, grad=True, out_dtype=torch.float32, comm=None):
        """Landmark-sharded evaluate over a torch.distributed group (comm: dist.DistComm,
        default the world group).  Returns s, z [T] (global, every rank) and, with grad,
        ds, dz [T, n, 3] whose rows with owner == rank are complete (the others hold
        this shard's partial sums, or are left unwritten where this shard has no
        window), plus owner [T]."""
        from . import dist as Dd
        return Dd.drive(self.sharded_steps(frames, grad, out_dtype), comm or Dd.DistComm())

    def sharded_steps(self, frames, grad=True, out_dtype=torch.float32):
        """Generator of the landmark-sharded evaluation: yields ("min", t), ("gather", t)
        and ("exchange", ds, dz, z_parts) collectives (dist.drive / drive_lockstep run
        them) and returns the result dict.  Same windows, refits and truncation as
        evaluate() on the full landmark set."""
        from . import dist as Dd
        if self.shard is None:
            raise ConfigError("sharded_steps needs PathCVTC(..., shard=(rank, world))")
        rank, world = self.shard[0], self.shard[1]
        one = self.screen == "f16x1"
        rlo = rhi = perm0 = None
        if self.prune:
            fr, fs0 = self._frames(frames, 1, check=False)
            Dc = K.msd_estimate(fs0, self.ls_coarse, grid=K2_GRID)
            dub = K.screen_bound(Dc, fs0.opnorm, self.ls_coarse.opnorm, self.kacc, fs0.rnorm, self.ls_coarse.rnorm)
            dub = yield ("min", dub)
            hlo, hhi, key = K.prune_plan(Dc, fs0.opnorm, self.ls_coarse.opnorm, self.kacc, self.mind,
                                         (self.cutoff + 2.0) / self.lam, self.knear, maxd=self.maxd,
                                         cstride=self.cstride, frnorm=fs0.rnorm, crnorm=self.ls_coarse.rnorm,
                                         dub_in=dub)
            ntl = self.mind.shape[1]
            perm0 = K.sort_by_key(key, ntl + 1)
            fs = K.gather_split(fs0, perm0)
            tlist, nlist, rlo, rhi = K.band_tiles(perm0, hlo, hhi, 128, 48, self.L, ntl)
            Dest = torch.empty((fr.shape[0], self.L), dtype=torch.float32, device=self.device)
            K.msd_estimate(fs, self.ls, Dest, grid=K2_GRID, tlist=tlist, nlist=nlist)
        else:
            fs0 = None
            Dest, fr, fs = self.estimate(frames, self.screen_terms, check=False)
        T = fr.shape[0]
        p = perm0.long() if perm0 is not None else None
        fnorm = self.frame_bound(fs) if one else None
        fcoef = 2.0 * self.lam if one else 0.0
        # the estimate minimum over every shard (in the caller's frame order)
        _, _, dmin, _ = K.candidates(Dest, self.lam, self.cutoff + self.margin, 1, fnorm=fnorm, fcoef=fcoef,
                                     rlo=rlo, rhi=rhi)
        if p is not None:
            dm = torch.empty_like(dmin)
            dm[p] = dmin
            dmin = dm
        dref = yield ("min", dmin)
        if p is not None:
            dref = dref[p].contiguous()
        cap = self.window_cap
        while True:
            _, cnt, wres, cflags, rflags = self._exact_windows(Dest, fr, fs, cap, rlo, rhi, perm0, dref)
            sl, zl = wres["s"], wres["z"]
            if p is not None:
                sl, zl = torch.empty_like(sl), torch.empty_like(zl)
                sl[p], zl[p] = wres["s"], wres["z"]
            fflags = fs.flags if fs0 is None else torch.cat([fs.flags, fs0.flags])
            status = torch.stack([_flag_bits_dev(fflags), _flag_bits_dev(cflags), _flag_bits_dev(rflags),
                                  _flag_bits_dev(wres["flags"])]).to(torch.float64).flatten()
            # one gather: the partials and every shard's status bits (so all shards take
            # the same retry / error decision)
            parts = yield ("gather", torch.cat([sl, zl, status]))
            bits = parts[:, 2 * T:].reshape(world, 4, -1) > 0
            ff, cf, rf, wf = (_bits_value(b.tolist()) for b in bits.any(0).cpu())
            if ff & FLAG_NON_FINITE:
                raise InvalidStructureError("frame coordinates contain non-finite values")
            if (cf & FLAG_SIG_OVERFLOW) and cap < self.L:
                cap = min(self.L, 4 * cap)
                continue
            break
        if rf & FLAG_NON_FINITE:
            raise InvalidStructureError("path_cv refine: non-finite coordinates or distances")
        if rf & FLAG_NO_CONVERGE:
            raise MetadynError("path_cv refine: Jacobi diagonalisation did not converge")
        if wf & FLAG_NON_FINITE:
            raise InvalidStructureError("non-finite distances in the path-CV reduction")
        s_parts, z_parts = parts[:, :T], parts[:, T:2 * T]
        s, z, alpha, beta = Dd.shard_coefficients(s_parts, z_parts, self.lam, rank)
        out = {"s": s, "z": z, "z_parts": z_parts, "window_cnt": cnt if p is None else cnt[torch.argsort(p)],
               "nsig": wres["nsig"]}
        if grad:
            if p is not None:
                alpha, beta = alpha[p].contiguous(), beta[p].contiguous()
            K.shard_rescale(wres, alpha, beta, cap)
            gperm = K.sig_span_key(wres, self.L)
            gperm = K.sort_by_key(gperm, 2 * self.L + 1)
            ds, dz = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm, out_dtype,
                                         out_map=perm0, ldig=self.ldig)
            owner = yield ("exchange", ds, dz, z_parts)
            out.update(ds=ds, dz=dz, owner=owner)
        return out


    # ------------------------------------------------------------ frame-routed landmark sharding

    def evaluate_routed(self, frames, home_offset, t_total, grad=True, out_dtype=torch.float32, comm=None):
        """Frame-routed landmark-sharded evaluate over a torch.distributed group: this
        rank passes its HOME frames (global rows [home_offset, home_offset + len)) and
        gets back their s, z and complete ds, dz (frame-sharded outputs)."""
        from . import dist as Dd
        return Dd.drive(self.routed_steps(frames, home_offset, t_total, grad, out_dtype), comm or Dd.DistComm())

    def routed_steps(self, frames, home_offset, t_total, grad=True, out_dtype=torch.float32):
        """Generator ("frame routing"): home phase -- one-term split of
        the home frames and the coarse screen against the GLOBAL coarse landmarks, giving
        each frame's admissible tile hull; ("alltoallv") every frame goes to the shards
        whose tiles its hull meets; shard phase -- banded screen of the received frames
        against the local landmarks, ("min") the global estimate minimum of every frame,
        exact refits, K4 partials, ("gather") the per-frame partials of every shard, the
        coefficient rescale and the gradient pass; ("alltoallv") each shard's rows of the
        frames it holds a window of go back to their home rank, which sums them."""
        from . import dist as Dd
        if self._gprune is None:
            raise ConfigError("routed_steps needs PathCVTC(..., shard=(rank, world, bounds), route=True)")
        rank, world = self.shard[0], self.shard[1]
        gp, dev, n = self._gprune, self.device, self.n
        frh, fsh = self._frames(frames, 1, check=False)
        Th = frh.shape[0]
        # home phase: global coarse screen -> admissible global tile hulls
        Dc = K.msd_estimate(fsh, gp["ls_coarse"], grid=K2_GRID)
        hlo, hhi, _ = K.prune_plan(Dc, fsh.opnorm, gp["ls_coarse"].opnorm, self.kacc, gp["mind"],
                                   (self.cutoff + 2.0) / self.lam, gp["knear"], maxd=gp["maxd"],
                                   cstride=gp["cstride"], frnorm=fsh.rnorm, crnorm=gp["ls_coarse"].rnorm)
        del Dc
        tb = torch.tensor(self._tile_bounds, dtype=torch.int32, device=dev)
        dest = (hlo[:, None] < tb[None, 1:]) & (hhi[:, None] > tb[None, :-1])  # [Th, G]
        sends = [torch.nonzero(dest[:, r]).flatten() for r in range(world)]
        gids = torch.arange(home_offset, home_offset + Th, dtype=torch.int64, device=dev)
        if world == 1:  # nothing to route: the home frames are the received frames (no copies)
            src_counts, gid, fr, hull = [Th], gids, frh, torch.stack([hlo, hhi], 1)
        else:
            got = yield ("alltoallv", [[gids[i] for i in sends], [frh[i] for i in sends],
                                       [torch.stack([hlo[i], hhi[i]], 1) for i in sends]])
            src_counts = [int(x.shape[0]) for x in got[0]]
            gid = torch.cat(got[0])
            fr = torch.cat(got[1]).contiguous()
            hull = torch.cat(got[2])
            del got
        R = int(gid.numel())
        t0, t1 = self._tile_bounds[rank], self._tile_bounds[rank + 1]
        ntl = t1 - t0
        one = self.screen == "f16x1"
        big = torch.full((t_total,), float("inf"), dtype=torch.float32, device=dev)
        if R:
            if world == 1:
                fr, fs0 = frh, fsh  # the home split is the received split
            else:
                fr, fs0 = self._frames(fr, 1, check=False)
            lo = (hull[:, 0].clamp(min=t0) - t0).to(torch.int32)
            hi = (hull[:, 1].clamp(max=t1) - t0).to(torch.int32)
            wide = max(1, (3 * ntl) // 4)
            key = torch.where(hi - lo >= wide, torch.zeros_like(lo), 1 + lo).to(torch.int32).contiguous()
            perm0 = K.sort_by_key(key, ntl + 1)
            p = perm0.long()
            fs = K.gather_split(fs0, perm0)
            tlist, nlist, rlo, rhi = K.band_tiles(perm0, lo.contiguous(), hi.contiguous(), 128, 48, self.L, ntl)
            Dest = torch.empty((R, self.L), dtype=torch.float32, device=dev)
            K.msd_estimate(fs, self.ls, Dest, grid=K2_GRID, tlist=tlist, nlist=nlist)
            fnorm = self.frame_bound(fs) if one else None
            fcoef = 2.0 * self.lam if one else 0.0
            _, _, dmin, _ = K.candidates(Dest, self.lam, self.cutoff + self.margin, 1, fnorm=fnorm, fcoef=fcoef,
                                         rlo=rlo, rhi=rhi)
            big[gid[p]] = dmin
        dglob = yield ("min", big)
        s_loc = torch.zeros((t_total,), dtype=torch.float64, device=dev)
        z_loc = torch.full((t_total,), float("inf"), dtype=torch.float64, device=dev)
        cap = self.window_cap
        while True:
            status = torch.zeros(20, dtype=torch.float64, device=dev)
            if R:
                dref = dglob[gid[p]].contiguous()
                _, cnt, wres, cflags, rflags = self._exact_windows(Dest, fr, fs, cap, rlo, rhi, perm0, dref)
                s_loc[gid[p]] = wres["s"]
                z_loc[gid[p]] = wres["z"]
                fflags = torch.cat([fs.flags, fs0.flags])
                status = torch.stack([_flag_bits_dev(fflags), _flag_bits_dev(cflags), _flag_bits_dev(rflags),
                                      _flag_bits_dev(wres["flags"])]).to(torch.float64).flatten()
            parts = yield ("gather", torch.cat([s_loc, z_loc, status]))
            bits = parts[:, 2 * t_total:].reshape(world, 4, -1) > 0
            ff, cf, rf, wf = (_bits_value(b.tolist()) for b in bits.any(0).cpu())
            if ff & FLAG_NON_FINITE:
                raise InvalidStructureError("frame coordinates contain non-finite values")
            if (cf & FLAG_SIG_OVERFLOW) and cap < self.L:
                cap = min(self.L, 4 * cap)
                continue
            break
        if rf & FLAG_NON_FINITE:
            raise InvalidStructureError("path_cv refine: non-finite coordinates or distances")
        if rf & FLAG_NO_CONVERGE:
            raise MetadynError("path_cv refine: Jacobi diagonalisation did not converge")
        if wf & FLAG_NON_FINITE:
            raise InvalidStructureError("non-finite distances in the path-CV reduction")
        s_parts, z_parts = parts[:, :t_total], parts[:, t_total:2 * t_total]
        s, z, alpha, beta = Dd.shard_coefficients(s_parts, z_parts, self.lam, rank)
        sl = slice(home_offset, home_offset + Th)
        out = {"s": s[sl].contiguous(), "z": z[sl].contiguous(), "received": R,
               "window_cnt": cnt if R else torch.zeros(0, dtype=torch.int32, device=dev),
               "nsig": wres["nsig"] if R else torch.zeros(0, dtype=torch.int32, device=dev)}
        if not grad:
            return out
        odt = out_dtype
        i64 = torch.empty(0, dtype=torch.int64, device=dev)
        pos_back = [i64] * world  # per source rank: positions (in its list) of frames with a window here
        rows_back = [[torch.empty((0, n, 3), dtype=odt, device=dev)] * world for _ in range(2)]
        if R:
            K.shard_rescale(wres, alpha[gid[p]].contiguous(), beta[gid[p]].contiguous(), cap)
            gperm = K.sort_by_key(K.sig_span_key(wres, self.L), 2 * self.L + 1)
            if world == 1:  # every home frame's rows are complete here: write the outputs directly
                del Dest
                wres.pop("D_window", None)  # free the window refits before the gradient outputs
                ds, dz = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm, odt,
                                             out_map=perm0, ldig=self.ldig)
                out.update(ds=ds, dz=dz)
                return out
            rows_s, rows_z = K.pathcv_grad_block(wres, fs, self.ls, fr, self.lraw, self.w, self.wa, cap, gperm, odt,
                                                 out_map=perm0, ldig=self.ldig)
            cnt_recv = torch.empty_like(cnt)
            cnt_recv[p] = cnt  # window count of every received frame, in received order
            o = 0
            for r in range(world):
                c = src_counts[r]
                pos = torch.nonzero(cnt_recv[o:o + c] > 0).flatten()
                pos_back[r] = pos
                rows_back[0][r], rows_back[1][r] = rows_s[o + pos], rows_z[o + pos]
                o += c
        back = yield ("alltoallv", [pos_back, rows_back[0], rows_back[1]])
        ds = torch.zeros((Th, n, 3), dtype=odt, device=dev)
        dz = torch.zeros((Th, n, 3), dtype=odt, device=dev)
        for r in range(world):  # fixed source order: bitwise-reproducible sums
            pos = back[0][r]
            if pos.numel():
                home_rows = sends[r][pos]
                ds.index_add_(0, home_rows, back[1][r])
                dz.index_add_(0, home_rows, back[2][r])
        out.update(ds=ds, dz=dz)
        return out


    # ------------------------------------------------------------ two-phase landmark sharding

    def evaluate_two_phase(self, frames, home_offset, t_total, grad=True, out_dtype=torch.float32, comm=None):
        """Two-phase landmark-sharded evaluate over a torch.distributed group: this rank
        passes its HOME frames (global rows [home_offset, home_offset + len); None: the
        ranks' home frames concatenated in rank order) and gets back their s, z and complete
        ds, dz (frame-sharded outputs)."""
        from . import dist as Dd
        return Dd.drive(self.two_phase_steps(frames, home_offset, t_total, grad, out_dtype), comm or Dd.DistComm())

    def two_phase_steps(self, frames, home_offset, t_total, grad=True, out_dtype=torch.float32):
        """Generator of the survey's two-phase plan.
        With PathCVTC(..., shard=(rank, world, dist.tile_bounds(L, world)), route=True,
        two_phase=True) phase 1 is routed instead of all-gathered (_two_phase_routed_screen).

        Phase 1 -- landmark-sharded screen: ("allgather_split") the one-term split of every
        rank's home frames (one all-gather: each rank then holds the screening operand of
        all T frames); the metric-pruned one-term screen of all T frames against this
        rank's landmark shard, with ("min") the global D_min upper bound for the pruning and
        ("min") the global estimate minimum for the windows; each shard's window of every
        frame (global landmark indices) goes to every rank in one ("gather").  The window
        of a frame is the hull of its per-shard windows -- the unsharded window, since
        every shard selects against the same global threshold.
        Phase 2 -- frame-sharded exact work on the home frames against the replicated
        landmark set: fp64 refits of the windows, the K4 softmax (complete: the window
        holds every significant landmark), and the int8 tensor-core gradient contraction.
        No further collective; the collectives move O(T) scalars plus the frames' screening
        operand once."""
        if self._full is None or self.shard is None:
            raise ConfigError("two_phase_steps needs PathCVTC(..., shard=(rank, world[, bounds]), two_phase=True)")
        frh, fsh = self._frames(frames, 1, check=False)
        Th = frh.shape[0]
        if self._gprune is not None:
            # ---- phase 1, routed: every home frame's screening operand goes only to the shards
            # its admissible coarse hull meets (no all-gather of every frame's operand)
            lo_h, cnt_h, cflags = yield from self._two_phase_routed_screen(frh, fsh, home_offset, t_total)
        else:
            lo_h, cnt_h, cflags = yield from self._two_phase_allgather_screen(frh, fsh, home_offset, t_total)
        out = yield from self._two_phase_home(frh, fsh, lo_h, cnt_h, cflags, grad, out_dtype)
        return out

    def _two_phase_routed_screen(self, frh, fsh, home_offset, t_total):
        """Routed phase 1 of two_phase_steps: ("gather") the home frame counts; the coarse
        screen of the home frames against the GLOBAL coarse landmarks gives each frame's
        admissible tile hull; ("alltoallv") the one-term operand rows + 4 scalars of each
        frame to the shards its hull meets; each shard screens what it received (banded,
        metric-pruned), ("min") the global estimate minimum per frame, windows against it;
        ("alltoallv") each received frame's window (2 int32) back to its home rank, which
        takes the hull over the shards.  NCCL bytes per step: ~60 KB (halves) + 40 B per routed
        copy of a frame (a frame goes to the 1-2 shards its hull meets), 4 B per frame (min),
        8 B per copy (windows) -- instead of every frame's operand on every rank."""
        from .kernels import Split
        rank, world, off, cnt_l = self.shard
        gp, dev = self._gprune, self.device
        one = self.screen == "f16x1"
        Th = frh.shape[0]
        counts = yield ("gather", torch.tensor([Th], dtype=torch.int64, device=dev))
        counts = [int(c) for c in counts.flatten().cpu().tolist()]
        T = sum(counts)
        if t_total is not None and T != int(t_total):
            raise ConfigError(f"gathered {T} frames, expected {t_total}")
        if home_offset is None:
            home_offset = int(sum(counts[:rank]))
        Dc = K.msd_estimate(fsh, gp["ls_coarse"], grid=K2_GRID)
        hlo_g, hhi_g, _ = K.prune_plan(Dc, fsh.opnorm, gp["ls_coarse"].opnorm, self.kacc, gp["mind"],
                                       (self.cutoff + 2.0) / self.lam, gp["knear"], maxd=gp["maxd"],
                                       cstride=gp["cstride"], frnorm=fsh.rnorm, crnorm=gp["ls_coarse"].rnorm)
        del Dc
        tb = torch.tensor(self._tile_bounds, dtype=torch.int32, device=dev)
        dest = (hlo_g[:, None] < tb[None, 1:]) & (hhi_g[:, None] > tb[None, :-1])  # [Th, G]
        # every (destination, frame) pair in destination-major order with one host read of the
        # per-destination counts (instead of G nonzero round trips)
        pairs = torch.nonzero(dest.T)
        ncopy = dest.sum(0).cpu().tolist()
        sends = list(torch.split(pairs[:, 1], ncopy))
        gids = torch.arange(home_offset, home_offset + Th, dtype=torch.int64, device=dev)
        hull = torch.stack([hlo_g, hhi_g], 1)
        if world == 1:  # nothing to route: the home split is the received split (no copies)
            got = None
            sends = [torch.arange(Th, device=dev)]
            src_counts, gid, R = [Th], gids, Th
        else:
            # per destination: the 3 operand planes of its frames (library row gathers, contiguous
            # [k, kpad] blocks), 4 scalars and the global hull
            scal = torch.stack([fsh.scale, fsh.opnorm, fsh.rnorm, fsh.g], 1)
            planes = [[K.gather_rows(fsh.hi[pl].view(torch.int32), i.to(torch.int32)).view(fsh.hi.dtype)
                       for i in sends] for pl in range(3)]
            got = yield ("alltoallv", [[gids[i] for i in sends], *planes, [scal[i] for i in sends],
                                       [hull[i] for i in sends]])
            del planes
            src_counts = [int(x.shape[0]) for x in got[0]]
            gid = torch.cat(got[0])
            R = int(gid.numel())
        t0, t1 = self._tile_bounds[rank], self._tile_bounds[rank + 1]
        ntl = t1 - t0
        big = torch.full((T,), float("inf"), dtype=torch.float32, device=dev)
        lo_r = cnt_r = None
        cflags = torch.zeros((0,), dtype=torch.uint8, device=dev)
        if R:
            if got is None:
                fs0, hr = fsh, hull
            else:
                sc = torch.cat(got[4])
                hr = torch.cat(got[5])
                hi_r = torch.empty((3, R, fsh.kpad), dtype=fsh.hi.dtype, device=dev)
                for pl in range(3):  # one copy per plane into the received split
                    torch.cat(got[1 + pl], out=hi_r[pl])
                fs0 = Split(hi_r, None, None, sc[:, 3].contiguous(), None, None,
                            torch.zeros(R, dtype=torch.uint8, device=dev), fsh.n, fsh.kpad, sc[:, 0].contiguous(),
                            fsh.fmt, fsh.terms, sc[:, 1].contiguous(), sc[:, 2].contiguous())
            del got
            lo = (hr[:, 0].clamp(min=t0) - t0).to(torch.int32)
            hi = (hr[:, 1].clamp(max=t1) - t0).to(torch.int32)
            wide = max(1, (3 * ntl) // 4)
            key = torch.where(hi - lo >= wide, torch.zeros_like(lo), 1 + lo).to(torch.int32)
            perm0 = K.sort_by_key(*_band_key(key, lo, hi, ntl))
            p = perm0.long()
            fs = K.gather_split(fs0, perm0)
            tlist, nlist, rlo, rhi = K.band_tiles(perm0, lo.contiguous(), hi.contiguous(), 128, 48, self.L, ntl)
            Dest = torch.empty((R, self.L), dtype=torch.float32, device=dev)
            K.msd_estimate(fs, self.ls, Dest, grid=K2_GRID, tlist=tlist, nlist=nlist)
            fnorm = self.frame_bound(fs) if one else None
            fcoef = 2.0 * self.lam if one else 0.0
            _, _, dmin, _ = K.candidates(Dest, self.lam, self.cutoff + self.margin, 1, fnorm=fnorm, fcoef=fcoef,
                                         rlo=rlo, rhi=rhi)
            big[gid[p]] = dmin  # (a frame arrives at most once per shard)
        else:
            del got
        dglob = yield ("min", big)
        if R:
            dref = dglob[gid[p]].contiguous()
            lo_s, cnt_s, _, cflags = K.candidates(Dest, self.lam, self.cutoff + self.margin, self.L, fnorm=fnorm,
                                                  fcoef=fcoef, rlo=rlo, rhi=rhi, dref=dref)
            del Dest
            lo_r = torch.empty_like(lo_s)
            cnt_r = torch.empty_like(cnt_s)
            lo_r[p], cnt_r[p] = lo_s + off, cnt_s  # received order, global landmark index
            win = torch.stack([lo_r, cnt_r], 1)
        else:
            win = torch.zeros((0, 2), dtype=torch.int32, device=dev)
        blocks, o = [], 0
        for c in src_counts:  # each source rank's frames, in the order it sent them
            blocks.append(win[o:o + c])
            o += c
        if world == 1:
            back = [blocks]
        else:
            back = yield ("alltoallv", [blocks])
        big_i = torch.iinfo(torch.int64).max
        lo_t = torch.full((Th,), big_i, dtype=torch.int64, device=dev)
        hi_t = torch.full((Th,), -1, dtype=torch.int64, device=dev)
        for r in range(world):  # shard r's windows of the home frames sends[r]
            w_r = back[0][r].long()
            if w_r.numel() == 0:
                continue
            act = w_r[:, 1] > 0
            idx = sends[r][act]
            lo_t.scatter_reduce_(0, idx, w_r[act, 0], reduce="amin")
            hi_t.scatter_reduce_(0, idx, w_r[act, 0] + w_r[act, 1], reduce="amax")
        lo_h = lo_t.clamp(max=self._full.L).to(torch.int32).contiguous()
        cnt_h = (hi_t - lo_t).clamp(min=0).to(torch.int32).contiguous()
        return lo_h, cnt_h, cflags

    def _two_phase_allgather_screen(self, frh, fsh, home_offset, t_total):
        """Phase 1 of two_phase_steps with every frame's screening operand all-gathered."""
        rank, world, off, cnt_l = self.shard
        dev = self.device
        one = self.screen == "f16x1"
        Th = frh.shape[0]
        # ---- phase 1: screen all frames against this landmark shard
        fs_all, counts = yield ("allgather_split", fsh)
        T = fs_all.count
        if t_total is not None and T != int(t_total):
            raise ConfigError(f"gathered {T} frames, expected {t_total}")
        if home_offset is None:  # the ranks' home frames in rank order
            home_offset = int(sum(counts[:rank]))
        rlo = rhi = perm0 = None
        if self.prune:
            Dc = K.msd_estimate(fs_all, self.ls_coarse, grid=K2_GRID)
            dub = K.screen_bound(Dc, fs_all.opnorm, self.ls_coarse.opnorm, self.kacc, fs_all.rnorm,
                                 self.ls_coarse.rnorm)
            dub = yield ("min", dub)
            hlo, hhi, key = K.prune_plan(Dc, fs_all.opnorm, self.ls_coarse.opnorm, self.kacc, self.mind,
                                         (self.cutoff + 2.0) / self.lam, self.knear, maxd=self.maxd,
                                         cstride=self.cstride, frnorm=fs_all.rnorm, crnorm=self.ls_coarse.rnorm,
                                         dub_in=dub)
            del Dc
            ntl = self.mind.shape[1]
            # only the frames with an admissible tile in THIS shard are gathered and screened
            # (empty hulls [ntl, 0) get their own last bin): ~T/G x (shards per hull) rows
            # instead of all T
            act = hhi > 0
            perm0 = K.sort_by_key(*_band_key(torch.where(act, key, torch.full_like(key, ntl + 1)), hlo, hhi, ntl))
            nact = int(act.sum().item())
            perm0 = perm0[:nact].contiguous()
            fs = K.gather_split(fs_all, perm0)
            tlist, nlist, rlo, rhi = K.band_tiles(perm0, hlo, hhi, 128, 48, self.L, ntl)
            Dest = torch.empty((max(nact, 1), self.L), dtype=torch.float32, device=dev)
            if nact:
                K.msd_estimate(fs, self.ls, Dest[:nact], grid=K2_GRID, tlist=tlist, nlist=nlist)
            Dest = Dest[:nact]
        else:
            fs = fs_all
            Dest = K.msd_estimate(fs, self.ls)
        fnorm = self.frame_bound(fs) if one else None
        fcoef = 2.0 * self.lam if one else 0.0
        _, _, dmin, _ = K.candidates(Dest, self.lam, self.cutoff + self.margin, 1, fnorm=fnorm, fcoef=fcoef,
                                     rlo=rlo, rhi=rhi)
        p = perm0.long() if perm0 is not None else None
        if p is not None:  # frame order; frames screened on no tile of this shard: +inf
            dm = torch.full((T,), float("inf"), dtype=dmin.dtype, device=dev)
            dm[p] = dmin
            dmin = dm
        dref = yield ("min", dmin)
        if p is not None:
            dref = dref[p].contiguous()
        lo, cnt, _, cflags = K.candidates(Dest, self.lam, self.cutoff + self.margin, self.L, fnorm=fnorm,
                                          fcoef=fcoef, rlo=rlo, rhi=rhi, dref=dref)
        del Dest
        if p is not None:  # back to frame order (unscreened frames: empty window here)
            lo_f = torch.zeros((T,), dtype=lo.dtype, device=dev)
            cnt_f = torch.zeros((T,), dtype=cnt.dtype, device=dev)
            lo_f[p], cnt_f[p] = lo, cnt
            lo, cnt = lo_f, cnt_f
        win = torch.stack([lo + off, cnt]).to(torch.int32)
        parts = yield ("gather", win)  # [G, 2, T]: every shard's window of every frame
        glo, gcnt = parts[:, 0].long(), parts[:, 1].long()
        act = gcnt > 0
        big = torch.iinfo(torch.int64).max
        lo_t = torch.where(act, glo, torch.full_like(glo, big)).amin(0)
        hi_t = torch.where(act, glo + gcnt, torch.full_like(glo, -1)).amax(0)
        sl = slice(home_offset, home_offset + Th)
        lo_h = lo_t[sl].clamp(max=self._full.L).to(torch.int32).contiguous()
        cnt_h = (hi_t[sl] - lo_t[sl]).clamp(min=0).to(torch.int32).contiguous()
        return lo_h, cnt_h, cflags

    def _two_phase_home(self, frh, fsh, lo_h, cnt_h, cflags, grad, out_dtype):
        """Phase 2 of two_phase_steps: exact refits, weights and gradients of the home frames
        over their merged windows, against the replicated full landmark set (no collective)."""
        if False:
            yield None  # a generator like its callers (phase 2 issues no collective)
        full = self._full
        Th = frh.shape[0]
        cap = int(max(1, min(full.L, int(cnt_h.max().item()) if Th else 1)))
        perm = K.sort_by_key((2 * lo_h + cnt_h).to(torch.int32), 2 * full.L + 1)
        Dex, Rex, rflags = full._refine_windows(frh, fsh, perm, lo_h, cnt_h, cap)
        wres = K.pathcv_weights(Dex, full.q, full.lam, Rex, fsh, full.ls, cap, full.cutoff, L=full.L, rowlo=lo_h,
                                rowcnt=cnt_h)
        out = {"s": wres["s"], "z": wres["z"], "window_lo": lo_h, "window_cnt": cnt_h, "nsig": wres["nsig"],
               "D_window": Dex}
        if grad:
            gperm = K.sort_by_key(K.sig_span_key(wres, full.L), 2 * full.L + 1)
            out["ds"], out["dz"] = K.pathcv_grad_block(wres, fsh, full.ls, frh, full.lraw, full.w, full.wa, cap, gperm,
                                                       out_dtype, ldig=full.ldig)
        status = torch.stack([_flag_bits_dev(fsh.flags), _flag_bits_dev(cflags), _flag_bits_dev(rflags),
                              _flag_bits_dev(wres["flags"])])
        ff, cf, rf, wf = (_bits_value(r) for r in status.cpu().tolist())
        if ff & FLAG_NON_FINITE:
            raise InvalidStructureError("frame coordinates contain non-finite values")
        if rf & FLAG_NON_FINITE:
            raise InvalidStructureError("path_cv refine: non-finite coordinates or distances")
        if rf & FLAG_NO_CONVERGE:
            raise MetadynError("path_cv refine: Jacobi diagonalisation did not converge")
        if wf & FLAG_NON_FINITE:
            raise InvalidStructureError("non-finite distances in the path-CV reduction")
        if Th and bool((cnt_h == 0).any()):
            raise EmptyActiveSetError("a frame has no landmark in any shard's window")
        return out


# ---------------------------------------------------------------- functional API

def msd_matrix(frames, landmarks, w=None, w_align=None):
    """All-pairs aligned MSD (eigvals[0] of kearsley_fit for every pair)."""
    return PathCV(landmarks, 1.0, w=w, w_align=w_align).msd_matrix(frames)


def path_cv(frames, landmarks, lam, q=None, w=None, w_align=None, grad=True):
    return PathCV(landmarks, lam, q, w, w_align).evaluate(frames, grad=grad)


def close_structure_replay(frames, landmarks, lam, eps, q=None, w=None, w_align=None, grad=True, walkers=1,
                           neighbours=None, nl_stride=1):
    return PathCV(landmarks, lam, q, w, w_align).close_replay(frames, eps, walkers=walkers, grad=grad,
                                                              neighbours=neighbours, nl_stride=nl_stride)

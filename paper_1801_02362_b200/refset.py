"""Reference-set file format v1 (DESIGN DECISIONS of the reference's
cli module) -- reader and writer, plus loaders that feed the resident engines.

    # metadyn-close refset v1
    STRUCTURE <id> q=<real>
    x y z w wprime          (one line per atom: coordinates in nm, displacement
    ...                      weight w, alignment weight w')
    <blank line>
    STRUCTURE <id> q=<real>
    ...

Numbers are written with Python's shortest round-trip repr, so write(read(f))
reproduces every value bit for bit.  Malformed input raises RefsetParseError
with the 1-based line number (errors.py:28-35); a structure the reference's own
validation would reject (non-finite coordinates, negative or all-zero weights,
fewer than 2 atoms) raises it at the line of its STRUCTURE header.  Host-side
file I/O only: the engines built from a reference set compute on the device.
"""

from __future__ import annotations

import io
import math
import os
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, InvalidStructureError, RefsetParseError

HEADER = "# metadyn-close refset v1"


@dataclass(frozen=True)
class RefsetEntry:
    """One STRUCTURE block as read: id, property q, raw coords [n, 3], w [n], w' [n]."""

    id: str
    q: float
    coords: np.ndarray
    w: np.ndarray
    wprime: np.ndarray

    def structure(self):
        """The reference's Structure type (weights normalised on construction)."""
        from .geometry import Structure

        return Structure(self.coords, self.w, self.wprime)


def _num(tok, lineno, what):
    try:
        v = float(tok)
    except ValueError:
        raise RefsetParseError(f"{what}: {tok!r} is not a decimal number", line=lineno) from None
    return v


def read_refset(src):
    """Parse a refset v1 file (path, text, or file object) -> list[RefsetEntry]."""
    if hasattr(src, "read"):
        text = src.read()
    elif isinstance(src, (str, os.PathLike)) and "\n" not in str(src) and os.path.exists(src):
        with open(src) as f:
            text = f.read()
    else:
        text = str(src)
    lines = text.split("\n")
    if not lines or lines[0].rstrip("\r") != HEADER:
        raise RefsetParseError(f"missing header {HEADER!r}", line=1)
    entries = []
    cur = None  # [id, q, header line, atom rows]
    ids = set()

    def close(block):
        if block is None:
            return
        sid, q, hline, rows = block
        if not rows:
            raise RefsetParseError(f"structure {sid!r} has no atoms", line=hline)
        arr = np.array(rows, dtype=np.float64)
        coords, w, wp = arr[:, :3].copy(), arr[:, 3].copy(), arr[:, 4].copy()
        try:
            from .geometry import Structure

            Structure(coords, w, wp)  # the reference's validation (geometry.py:34-61)
        except InvalidStructureError as e:
            raise RefsetParseError(f"structure {sid!r}: {e}", line=hline) from None
        if entries and coords.shape[0] != entries[0].coords.shape[0]:
            raise RefsetParseError(f"structure {sid!r} has {coords.shape[0]} atoms, the first structure has "
                                   f"{entries[0].coords.shape[0]}", line=hline)
        entries.append(RefsetEntry(sid, q, coords, w, wp))

    for k, raw in enumerate(lines[1:], start=2):
        line = raw.rstrip("\r")
        if not line.strip():
            close(cur)
            cur = None
            continue
        toks = line.split()
        if toks[0] == "STRUCTURE":
            close(cur)
            if len(toks) != 3 or not toks[2].startswith("q="):
                raise RefsetParseError("expected 'STRUCTURE <id> q=<real>'", line=k)
            sid = toks[1]
            if sid in ids:
                raise RefsetParseError(f"duplicate structure id {sid!r}", line=k)
            ids.add(sid)
            q = _num(toks[2][2:], k, "property q")
            if not math.isfinite(q):
                raise RefsetParseError("property q must be finite", line=k)
            cur = [sid, q, k, []]
            continue
        if cur is None:
            raise RefsetParseError("atom line outside a STRUCTURE block", line=k)
        if len(toks) != 5:
            raise RefsetParseError(f"expected 5 columns 'x y z w wprime', got {len(toks)}", line=k)
        cur[3].append([_num(t, k, name) for t, name in zip(toks, ("x", "y", "z", "w", "wprime"))])
    close(cur)
    if not entries:
        raise RefsetParseError("no STRUCTURE blocks", line=len(lines))
    return entries


def _fmt(v):
    return repr(float(v))


def write_refset(dst, entries):
    """Write entries (RefsetEntry, or (id, q, coords, w, wprime) tuples) as refset v1 text
    to a path or file object; returns the text."""
    buf = io.StringIO()
    buf.write(HEADER + "\n")
    seen = set()
    for i, e in enumerate(entries):
        sid, q, coords, w, wp = (e.id, e.q, e.coords, e.w, e.wprime) if isinstance(e, RefsetEntry) else e
        sid = str(sid)
        if not sid or any(c.isspace() for c in sid) or sid in seen:
            raise ConfigError(f"structure id {sid!r} must be unique and contain no whitespace")
        seen.add(sid)
        coords = np.asarray(coords, dtype=np.float64)
        w = np.asarray(w, dtype=np.float64)
        wp = np.asarray(wp, dtype=np.float64)
        if coords.ndim != 2 or coords.shape[1] != 3 or w.shape != (coords.shape[0],) or wp.shape != w.shape:
            raise InvalidStructureError(f"structure {sid!r}: coords [n, 3] with weights [n] required")
        if i:
            buf.write("\n")
        buf.write(f"STRUCTURE {sid} q={_fmt(q)}\n")
        for (x, y, z), a, b in zip(coords, w, wp):
            buf.write(f"{_fmt(x)} {_fmt(y)} {_fmt(z)} {_fmt(a)} {_fmt(b)}\n")
    text = buf.getvalue()
    if dst is not None:
        if hasattr(dst, "write"):
            dst.write(text)
        else:
            with open(dst, "w") as f:
                f.write(text)
    return text


def entries_from_arrays(landmarks, q=None, w=None, wprime=None, ids=None):
    """RefsetEntry list from stacked arrays landmarks [L, n, 3] (weights shared, default 1)."""
    lm = np.asarray(landmarks, dtype=np.float64)
    L, n = lm.shape[0], lm.shape[1]
    qq = np.arange(L, dtype=np.float64) if q is None else np.asarray(q, dtype=np.float64)
    ww = np.ones(n) if w is None else np.asarray(w, dtype=np.float64)
    wp = np.ones(n) if wprime is None else np.asarray(wprime, dtype=np.float64)
    ids = [f"ref{i}" for i in range(L)] if ids is None else [str(i) for i in ids]
    return [RefsetEntry(ids[i], float(qq[i]), lm[i].copy(), ww.copy(), wp.copy()) for i in range(L)]


def _shared_weights(entries):
    w, wp = entries[0].w, entries[0].wprime
    for e in entries[1:]:
        if not (np.array_equal(e.w, w) and np.array_equal(e.wprime, wp)):
            raise ConfigError("the batched engines share one weight vector per kind across the reference set; "
                              f"structure {e.id!r} has different weights (use colvar.ReferenceSet per structure)")
    return w, wp


def reference_set(src, lam):
    """colvar.ReferenceSet (SPEC colvar module) from a refset file: per-structure weights kept."""
    from .colvar import ReferenceSet

    entries = read_refset(src)
    return ReferenceSet([e.structure() for e in entries], np.array([e.q for e in entries]), lam=lam)


def load_pathcv(src, lam, engine="tc", **kw):
    """A resident path-CV engine from a refset file: engine "tc" -> engine.PathCVTC (fp32
    coordinates, tensor-core path), "fp64" -> engine.PathCV; q, w and w' from the file."""
    from . import engine as E

    entries = read_refset(src)
    w, wp = _shared_weights(entries)
    lm = np.stack([e.coords for e in entries])
    q = np.array([e.q for e in entries])
    if engine == "tc":
        return E.PathCVTC(lm.astype(np.float32), lam, q=q, w=w, w_align=wp, **kw)
    if engine == "fp64":
        return E.PathCV(lm, lam, q=q, w=w, w_align=wp, **kw)
    raise ConfigError(f"engine must be 'tc' or 'fp64', got {engine!r}")

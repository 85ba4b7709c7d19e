"""Reference-set file format v1: bit-exact round trips, malformed input
-> RefsetParseError(line=) (errors.py:28-35), and the loaders that feed the engines."""

import numpy as np
import pytest
import torch

from paper_1801_02362_b200 import refset as RS
from paper_1801_02362_b200.errors import ConfigError, RefsetParseError


def _entries(seed=0, L=4, n=5, shared=True):
    rng = np.random.default_rng(seed)
    lm = rng.normal(0.0, 0.3, size=(L, n, 3))
    lm[0, 0, 0] = 1.0 / 3.0
    lm[0, 1, 1] = -1e-300
    lm[1, 2, 2] = 123456789.123456789
    w = rng.uniform(0.1, 2.0, n)
    wp = rng.uniform(0.1, 2.0, n)
    ents = RS.entries_from_arrays(lm, q=np.linspace(-1.5, 2.0 / 7.0, L), w=w, wprime=wp, ids=[f"s{i}" for i in range(L)])
    if not shared:
        ents[1] = RS.RefsetEntry("s1", ents[1].q, ents[1].coords, w * 2.0 + 0.1, wp)
    return ents


def test_round_trip_is_bit_exact(tmp_path):
    ents = _entries()
    p = tmp_path / "refs.txt"
    text = RS.write_refset(p, ents)
    assert text.splitlines()[0] == "# metadyn-close refset v1"
    assert text.splitlines()[1].startswith("STRUCTURE s0 q=")
    assert "\n\nSTRUCTURE s1 " in text  # blank-line separated blocks
    back = RS.read_refset(p)
    assert [e.id for e in back] == [e.id for e in ents]
    for a, b in zip(ents, back):
        assert a.q == b.q
        for x, y in ((a.coords, b.coords), (a.w, b.w), (a.wprime, b.wprime)):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))  # every bit
    assert RS.write_refset(None, back) == text
    # text and file-object sources parse the same
    assert [e.q for e in RS.read_refset(text)] == [e.q for e in back]
    with open(p) as f:
        assert len(RS.read_refset(f)) == 4


def test_structures_keep_the_reference_weight_semantics():
    e = _entries(L=2)[0]
    s = e.structure()
    np.testing.assert_allclose(s.disp_weights, e.w / e.w.sum())
    np.testing.assert_allclose(s.align_weights, e.wprime / e.wprime.sum())
    np.testing.assert_array_equal(s.coords, e.coords)


GOOD = RS.write_refset(None, _entries(L=2, n=3))


@pytest.mark.parametrize("text,line", [
    ("", 1),
    ("# metadyn-close refset v2\n", 1),
    (GOOD.replace("STRUCTURE s1 q=", "STRUCTURE s1 p="), 7),
    (GOOD.replace("STRUCTURE s1 q=", "STRUCTURE  q=", 1).replace("STRUCTURE  q=", "STRUCTURE q="), 7),
    (GOOD.replace("q=-1.5", "q=minus"), 2),
    (GOOD.replace("q=-1.5", "q=nan"), 2),
    ("# metadyn-close refset v1\n0 0 0 1 1\n", 2),
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 1\n1 1 1 1 1\n", 3),
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 zero 1 1\n1 1 1 1 1\n", 3),
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 1 1\n", 2),                       # one atom
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 -1 1\n1 1 1 1 1\n", 2),           # negative w
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 1 0\n1 1 1 1 0\n", 2),            # w' sums to 0
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\ninf 0 0 1 1\n1 1 1 1 1\n", 2),          # non-finite
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 1 1\n1 1 1 1 1\n\n"
     "STRUCTURE b q=1\n0 0 0 1 1\n1 1 1 1 1\n2 2 2 1 1\n", 6),                             # atom count
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n0 0 0 1 1\n1 1 1 1 1\n\n"
     "STRUCTURE a q=1\n0 0 0 1 1\n1 1 1 1 1\n", 6),                                        # duplicate id
    ("# metadyn-close refset v1\nSTRUCTURE a q=0\n\n", 2),                                 # empty block
    ("# metadyn-close refset v1\n\n\n", 4),                                                # no structures
])
def test_malformed_input_reports_the_line(text, line):
    with pytest.raises(RefsetParseError) as ei:
        RS.read_refset(text)
    assert ei.value.line == line, (str(ei.value), line)
    assert str(ei.value).startswith(f"line {line}:")


def test_reference_set_and_shared_weight_check():
    ents = _entries()
    text = RS.write_refset(None, ents)
    ref = RS.reference_set(text, lam=3.0)
    np.testing.assert_array_equal(ref.properties, [e.q for e in ents])
    assert ref.n == 4 and ref.lam == 3.0
    with pytest.raises(ConfigError):
        RS.load_pathcv(RS.write_refset(None, _entries(shared=False)), 3.0)
    with pytest.raises(ConfigError):
        RS.write_refset(None, [("a b", 0.0, np.zeros((2, 3)), np.ones(2), np.ones(2))])


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["tc", "fp64"])
def test_engine_from_refset_file_equals_engine_from_arrays(engine, tmp_path, cuda_device):
    """A path-CV engine built from a refset file (q, w, w' from the file) evaluates the same
    s, z and gradients as one built from the arrays."""
    from paper_1801_02362_b200 import engine as E, synth

    wl = synth.config4(seed=3, T=24, L=64, N=120) if engine == "tc" else synth.config0(seed=3, T=24)
    L, n = wl.landmarks.shape[0], wl.landmarks.shape[1]
    q = np.linspace(0.0, 1.0, L) ** 2
    lm = wl.landmarks.astype(np.float32) if engine == "tc" else wl.landmarks
    p = tmp_path / "refs.txt"
    RS.write_refset(p, RS.entries_from_arrays(lm, q=q))
    a = RS.load_pathcv(p, wl.lam, engine=engine)
    b = (E.PathCVTC(lm, wl.lam, q=q) if engine == "tc" else E.PathCV(lm, wl.lam, q=q))
    kw = {"out_dtype": torch.float64}
    oa, ob = a.evaluate(wl.frames, **kw), b.evaluate(wl.frames, **kw)
    for key in ("s", "z", "ds", "dz"):
        np.testing.assert_array_equal(oa[key].cpu().numpy(), ob[key].cpu().numpy())

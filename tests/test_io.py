"""Candidate / warm-start files (io.py:16-114): our loaders against the reference's on the
same files, the member-major fast path, and the SchemaError cases."""

import json
import os
import sys

import numpy as np
import pytest

from paper_2510_09204_b200 import io
from paper_2510_09204_b200.errors import SchemaError
from paper_2510_09204_b200.problem import (BasisConfig, ScenarioFamily, build_basis, generate,
                                           sample_naive_prior)

REF = "/root/reference/pkg/src"


@pytest.fixture
def scn_cands():
    hz = BasisConfig(11, 50, 5.0)
    scn = generate(ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=2), 5, 2, seed=9, horizon=hz)
    return scn, sample_naive_prior(scn, build_basis(hz), 3, seed=9)


def test_round_trip_and_member_major(tmp_path, scn_cands):
    scn, cands = scn_cands
    p = tmp_path / "c.json"
    io.save_candidates(p, cands, scn.n, scn.n_d, 11)
    back = io.load_candidates(p, scn)
    assert all(np.array_equal(a, b) for a, b in zip(back, cands))
    mm = io.load_candidates_mm(p, scn)
    assert mm.shape == (3, 2, 5, 11)
    assert np.array_equal(mm, np.stack([c.transpose(1, 0, 2) for c in cands]))
    w = tmp_path / "w.json"
    w.write_text(json.dumps({"version": 1, "entries": [
        {"xi0": c.transpose(1, 0, 2).ravel().tolist(), "lambda0": (0.5 * c).transpose(1, 0, 2).ravel().tolist()}
        for c in cands]}))
    ws = io.load_warmstarts(w, scn)
    assert np.array_equal(ws[1][0], cands[1]) and np.array_equal(ws[2][1], 0.5 * cands[2])


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_matches_reference_loaders(tmp_path, scn_cands):
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    try:
        from swarmplan import io as rio, scenario as rs, basis as rb
    finally:
        sys.path.remove(REF)
    scn, cands = scn_cands
    rscn = rs.generate(rs.ScenarioFamily("random_box", box=(-1.5, 1.5), n_obstacles=2), 5, 2, seed=9,
                       horizon=rb.BasisConfig(11, 50, 5.0))
    p = tmp_path / "c.json"
    rio.save_candidates(p, cands, 5, 2, 11)
    q = tmp_path / "d.json"
    io.save_candidates(q, cands, 5, 2, 11)
    assert p.read_text() == q.read_text()
    for a, b in zip(io.load_candidates(p, scn), rio.load_candidates(p, rscn)):
        assert np.array_equal(a, b)


def test_schema_errors(tmp_path, scn_cands):
    scn, cands = scn_cands
    good = {"version": 1, "n": 5, "n_d": 2, "n_xi": 11,
            "samples": [c.transpose(1, 0, 2).ravel().tolist() for c in cands]}
    cases = [
        ("{not json", "malformed JSON"),
        (json.dumps({k: v for k, v in good.items() if k != "samples"}), "missing field 'samples'"),
        (json.dumps({**good, "version": 2}), "unsupported candidate version"),
        (json.dumps({**good, "n": 4}), "candidate n mismatch"),
        (json.dumps({**good, "samples": [[0.0] * 7]}), "sample 0 has length 7"),
        (json.dumps({**good, "samples": [[float("nan")] * 110]}).replace("NaN", "NaN"), "non-finite"),
    ]
    for text, msg in cases:
        p = tmp_path / "bad.json"
        p.write_text(text)
        with pytest.raises(SchemaError, match=msg):
            io.load_candidates(p, scn)
    w = tmp_path / "w.json"
    w.write_text(json.dumps({"version": 1, "entries": [{"xi0": [0.0] * 110}]}))
    with pytest.raises(SchemaError, match="missing field 'lambda0'"):
        io.load_warmstarts(w, scn)

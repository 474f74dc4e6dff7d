"""Candidate and warm-start files of the reference (pkg/src/swarmplan/io.py:16-114) read
straight into the SF's member-major layout (file interop for the
sampler -> SF handoff).

The candidate file stores each sample flattened axis-major, then robot, then coefficient
(io.py:19-20) — byte-for-byte the member-major row [n_d][n][n_basis] the kernel reads —
so `load_candidates_mm` is a validated reshape with no transpose, and its result can be
handed to `DeviceBatch` / `pipeline.plan_many` (one H2D copy). `load_candidates`,
`save_candidates` and `load_warmstarts` keep the reference's signatures, per-sample
(n, n_d, n_basis) results and SchemaError messages.
"""

from __future__ import annotations

import json

import numpy as np

from .errors import SchemaError

CANDIDATE_VERSION = 1     # io.py:16
WARMSTART_VERSION = 1     # io.py:18


def save_candidates(path, coeff_list, n: int, n_d: int, n_basis: int) -> None:
    """io.py:19-30."""
    samples = [np.asarray(c).transpose(1, 0, 2).reshape(-1).tolist() for c in coeff_list]
    doc = {"version": CANDIDATE_VERSION, "n": n, "n_d": n_d, "n_xi": n_basis, "samples": samples}
    with open(path, "w") as fh:
        json.dump(doc, fh)
        fh.write("\n")


def _read_json(path):
    with open(path) as fh:
        try:
            return json.load(fh)
        except json.JSONDecodeError as exc:
            raise SchemaError(f"{path}: malformed JSON at line {exc.lineno}: {exc.msg}") from exc


def load_candidates_mm(path, scn) -> np.ndarray:
    """io.py:33-61 validation; returns (C, n_d, n, n_basis) member-major float64."""
    doc = _read_json(path)
    for key in ("version", "n", "n_d", "n_xi", "samples"):
        if key not in doc:
            raise SchemaError(f"candidate file missing field {key!r}")
    if doc["version"] != CANDIDATE_VERSION:
        raise SchemaError(f"unsupported candidate version {doc['version']!r}")
    n_xi = scn.horizon.n_basis
    for name, expect, actual in (("n", scn.n, doc["n"]), ("n_d", scn.n_d, doc["n_d"]),
                                 ("n_xi", n_xi, doc["n_xi"])):
        if actual != expect:
            raise SchemaError(f"candidate {name} mismatch: expected {expect}, got {actual}")
    size = scn.n * scn.n_d * n_xi
    out = np.empty((len(doc["samples"]), scn.n_d, scn.n, n_xi))
    for idx, flat in enumerate(doc["samples"]):
        arr = np.asarray(flat, dtype=float)
        if arr.size != size:
            raise SchemaError(f"sample {idx} has length {arr.size}")
        if not np.isfinite(arr).all():
            raise SchemaError(f"sample {idx} contains non-finite values")
        out[idx] = arr.reshape(scn.n_d, scn.n, n_xi)
    return out


def load_candidates(path, scn) -> list[np.ndarray]:
    """io.py:33-61: list of (n, n_d, n_basis) coefficient sets."""
    return [c.transpose(1, 0, 2) for c in load_candidates_mm(path, scn)]


def load_warmstarts_mm(path, scn) -> tuple[np.ndarray, np.ndarray]:
    """io.py:93-114 validation; returns member-major (xi0, lam0), each (E, n_d, n, n_basis)."""
    doc = _read_json(path)
    if doc.get("version") != WARMSTART_VERSION:
        raise SchemaError(f"unsupported warm-start version {doc.get('version')!r}")
    if "entries" not in doc:
        raise SchemaError("warm-start file missing field 'entries'")
    n, n_d, n_xi = scn.n, scn.n_d, scn.horizon.n_basis
    size = n * n_d * n_xi
    xi = np.empty((len(doc["entries"]), n_d, n, n_xi))
    lam = np.empty_like(xi)
    for idx, entry in enumerate(doc["entries"]):
        for key in ("xi0", "lambda0"):
            if key not in entry:
                raise SchemaError(f"warm-start entry {idx} missing field {key!r}")
            if len(entry[key]) != size:
                raise SchemaError(f"warm-start entry {idx} field {key!r} has wrong length")
        xi[idx] = np.asarray(entry["xi0"], float).reshape(n_d, n, n_xi)
        lam[idx] = np.asarray(entry["lambda0"], float).reshape(n_d, n, n_xi)
    return xi, lam


def load_warmstarts(path, scn) -> list[tuple[np.ndarray, np.ndarray]]:
    """io.py:93-114: (xi0 coeffs, lambda0 coeffs) per entry, aligned with a candidate file."""
    xi, lam = load_warmstarts_mm(path, scn)
    return [(x.transpose(1, 0, 2), l.transpose(1, 0, 2)) for x, l in zip(xi, lam)]

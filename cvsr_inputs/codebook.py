"""Code database ("we pre-built a database to store LDPC codes with their code rates
ranging from 0.01 to 0.8").

A code is stored as its RECIPE -- family, parameters, seed and block length -- together with
the SHA-256 digest of the parity-check matrix it builds and the frame-error test it passed or
failed in the rate back-off of PAPER.md:394 (`tools/backoff.py`, reading R-2' of DESIGN.md).
Constructions are deterministic, so the recipe reproduces the stored matrix bit for bit
(`verify_digest`); a 10^6-bit code would be ~14 MB of CSR per entry, the recipe is ~200 bytes.

This module holds no decoder arithmetic: it builds codes (cvsr_inputs.codes) and reads/writes
`codebook.json`.
"""
from __future__ import annotations

import json
import os
from typing import Dict, List, Optional

from . import codes as _codes

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "codebook.json")


def build(entry: Dict) -> _codes.Code:
    """The code of a database entry (family "irregular" | "met" | "met_irr")."""
    p = entry["params"]
    if entry["family"] == "irregular":
        kw = {}
        if p.get("lam"):
            kw["lam"] = {int(k): float(v) for k, v in p["lam"].items()}
        return _codes.irregular_rate(entry["n"], p["rate"], seed=entry["seed"], **kw)
    if entry["family"] == "met":
        return _codes.met_low_rate(entry["n"], p["alpha"], p["beta"], p.get("dv_core", 3), p.get("dc_core", 6),
                                   seed=entry["seed"])
    if entry["family"] == "met_irr":
        return _codes.met_irregular_core(entry["n"], p["alpha"], p["core_rate"], seed=entry["seed"])
    raise ValueError(f"unknown family {entry['family']!r}")


def load(path: str = PATH) -> List[Dict]:
    if not os.path.exists(path):
        return []
    with open(path) as f:
        return json.load(f)["codes"]


def save(entries: List[Dict], path: str = PATH, meta: Optional[Dict] = None) -> None:
    with open(path, "w") as f:
        json.dump({"meta": meta or {}, "codes": entries}, f, indent=1)
        f.write("\n")


def good(config: str, slice_j: int, n: int, path: str = PATH) -> Optional[Dict]:
    """The entry the back-off marked "good" for (config, slice, N_R), or None."""
    for e in load(path):
        if e["config"] == config and e["slice"] == slice_j and e["n"] == n and e["status"] == "good":
            return e
    return None


def verify_digest(entry: Dict) -> bool:
    return build(entry).digest() == entry["digest"]

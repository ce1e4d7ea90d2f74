"""Strategy names and the public fit entry points (reference: strategies.py).

``fast_stmf`` / ``fit`` keep the reference signatures.  Every method the reference
parses (FastSTMF, the other ByRow / ByElement / ByMatrix combinations and the STMF
baseline) runs on the device kernels; there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

from .engine import run_fit
from .fitrun import (UpdateCandidate, byelement_sweep, bymatrix_candidates, bymatrix_step, byrow_seq,  # noqa: F401
                     byrow_sweep, select_k_td, select_k_td_a, select_k_td_b)
from .types import MaskedMatrix, RunConfig

__all__ = ["StrategySpec", "BASELINE", "FASTSTMF", "parse_method", "fit", "fast_stmf", "UpdateCandidate",
           "select_k_td", "select_k_td_a", "select_k_td_b", "byrow_sweep", "byrow_seq", "byelement_sweep",
           "bymatrix_step", "bymatrix_candidates"]

FAMILIES = ("ByRow", "ByElement", "ByMatrix")
SELECTIONS = ("SEQ", "TD", "TD_A", "TD_B")
PERMUTATIONS = ("NoPerm", "PermR", "PermC", "RandPermR")

#: method name of the classic baseline (not a StrategySpec)
BASELINE = "STMF"


@dataclass(frozen=True)
class StrategySpec:
    """A valid (family, selection, permutation, shape) combination (strategies.py:77-105)."""

    family: str
    selection: str
    permutation: str
    prefer_wide: bool = True

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown family {self.family!r}")
        if self.selection not in SELECTIONS:
            raise ValueError(f"unknown selection {self.selection!r}")
        if self.permutation not in PERMUTATIONS:
            raise ValueError(f"unknown permutation {self.permutation!r}")
        if self.family == "ByElement" and (self.selection != "TD" or self.permutation != "PermC"):
            raise ValueError("ByElement pairs only with TD and PermC")
        if self.family == "ByMatrix" and (self.selection != "TD" or self.permutation != "NoPerm"):
            raise ValueError("ByMatrix pairs only with TD and NoPerm")
        if self.family == "ByRow" and self.permutation == "PermC":
            raise ValueError("ByRow does not use column permutation")

    @property
    def name(self) -> str:
        return f"STMF_{self.family}_{self.permutation}_{self.selection}{'_W' if self.prefer_wide else ''}"


FASTSTMF = StrategySpec("ByRow", "TD_A", "RandPermR", prefer_wide=True)

_CANON = {x.lower(): x for x in FAMILIES + SELECTIONS + PERMUTATIONS}
_CANON["randperm"] = "RandPermR"


def parse_method(name: str):
    """Method name -> StrategySpec (or BASELINE), case-insensitive (strategies.py:116-141)."""
    low = name.strip().lower()
    if low == "stmf":
        return BASELINE
    if low == "faststmf":
        return FASTSTMF
    parts = low.split("_")
    if parts and parts[0] == "stmf":
        parts = parts[1:]
    wide = bool(parts) and parts[-1] == "w"
    if wide:
        parts = parts[:-1]
    if len(parts) >= 3:
        family, perm, sel = _CANON.get(parts[0]), _CANON.get(parts[1]), _CANON.get("_".join(parts[2:]))
        if family in FAMILIES and perm in PERMUTATIONS and sel in SELECTIONS:
            return StrategySpec(family, sel, perm, prefer_wide=wide)
    raise ValueError(f"cannot parse method name {name!r}")


class _SpecStrategy:
    """The reference's strategy adapter (strategies.py:317-348) for the host part of the
    plugin protocol: ``orient`` (transpose / permutation with the fit's RNG).  The sweeps
    themselves run on the device (stmf_run), so there is no ``sweep`` here."""

    def __init__(self, spec: StrategySpec):
        self.spec = spec
        self.name = spec.name

    def orient(self, R: MaskedMatrix, rng):
        from .engine import _orient
        return _orient(self.spec, R, rng)


def fit(R: MaskedMatrix, rank: int, method, config: RunConfig, device: int | None = None, init=None):
    """Fit R with a method name or StrategySpec (strategies.py:351-357).  ``init``:
    optional warm-start factors (engine.run_fit)."""
    if isinstance(method, str):
        method = parse_method(method)
    return run_fit(R, rank, method, config, device=device, init=init)


def fast_stmf(R: MaskedMatrix, rank: int, config: RunConfig, device: int | None = None, init=None):
    """FastSTMF = ByRow, RandPermR, TD_A, wide (strategies.py:360-362), on the B200."""
    return fit(R, rank, FASTSTMF, config, device=device, init=init)

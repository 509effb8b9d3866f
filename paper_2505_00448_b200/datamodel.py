"""Host-side data model: matrices, requests and result sets.

This is the drop-in surface of the reference's ``pkg/src/pairstat/datamodel.py``:
the same vocabulary constants (``:40-78``), the same missingness rule
(``present_mask``, ``:86-104``), the same ``make_matrix`` validation
(``:144-196``, ``:199-235``), ``TestRequest`` validation (``:293-338``) and
``ResultSet`` (``:346-369``).  Validation stays on the host because it is part
of constructing the API types; all pairwise compute happens on the B200 behind
the C-ABI (see :mod:`paper_2505_00448_b200.engine`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import (
    EmptyMatrix,
    LabelOutOfRange,
    NegativeLabel,
    NonIntegerCategoryLabel,
    UnsupportedOutputForTest,
)

KINDS = ("continuous", "dichotomous", "categorical")
BASE_OUTPUTS = ("stat", "p", "p_bonferroni", "p_bh", "p_by")
EFFECTS_BY_TEST = {
    "pearson": ("r2",),
    "spearman": ("rho",),
    "chi2": ("phi", "cramers_v"),
    "ttest": ("cohens_d",),
    "mwu": ("r",),
    "anova": ("partial_eta2",),
    "kruskal": ("eta2",),
}
TESTS = tuple(EFFECTS_BY_TEST)
KINDS_BY_TEST = {
    "pearson": ("continuous", None),
    "spearman": ("continuous", None),
    "chi2": ("categorical", None),
    "ttest": ("dichotomous", "continuous"),
    "mwu": ("dichotomous", "continuous"),
    "anova": ("categorical", "continuous"),
    "kruskal": ("categorical", "continuous"),
}
T_VARIANTS = ("student", "welch")
U_MODES = ("exact", "asymptotic", "auto")


def outputs_for(test: str) -> tuple[str, ...]:
    """All output tokens of ``test``: the base five, then its effect sizes."""
    return BASE_OUTPUTS + EFFECTS_BY_TEST[test]


def present_mask(values: np.ndarray, na_sentinel: float) -> np.ndarray:
    """True where an entry is data (reference ``datamodel.py:86-104``).

    A NaN sentinel marks NaN entries missing; any other sentinel marks entries
    whose 64-bit pattern equals the sentinel's (so -0.0 and +0.0 differ).
    """
    if math.isnan(na_sentinel):
        return ~np.isnan(values)
    bits = np.ascontiguousarray(values, dtype=np.float64).view(np.uint64)
    return bits != np.array(na_sentinel, dtype=np.float64).view(np.uint64)


@dataclass(frozen=True)
class DataMatrix:
    """Features x samples fp64 matrix plus its missingness and label counts."""

    values: np.ndarray
    na_sentinel: float
    kind: str
    category_counts: np.ndarray | None = None
    present: np.ndarray = field(default=None, repr=False)  # type: ignore[assignment]

    @property
    def n_features(self) -> int:
        return int(self.values.shape[0])

    @property
    def n_samples(self) -> int:
        return int(self.values.shape[1])


def _label_counts(values: np.ndarray, present: np.ndarray, kind: str) -> np.ndarray:
    """c_f = 1 + largest present label; dichotomous is always 2.

    Follows reference ``datamodel.py:199-235`` including its error order:
    non-integer first, then negative, then (dichotomous) above one.
    """
    counts = np.empty(values.shape[0], dtype=np.int64)
    dichotomous = kind == "dichotomous"
    for f in range(values.shape[0]):
        row = values[f][present[f]]
        if row.size == 0:
            counts[f] = 2 if dichotomous else 0
            continue
        integral = np.isfinite(row) & (np.floor(row) == row)
        if not integral.all():
            bad = float(row[~integral][0])
            raise NonIntegerCategoryLabel(f"feature {f} has non-integer label {bad!r}")
        lo = float(row.min())
        if lo < 0:
            raise NegativeLabel(f"feature {f} has negative label {lo!r}")
        hi = float(row.max())
        if dichotomous:
            if hi > 1:
                raise LabelOutOfRange(
                    f"feature {f} has label {hi!r}; dichotomous labels must be 0 or 1"
                )
            counts[f] = 2
        else:
            counts[f] = int(hi) + 1
    return counts


def make_matrix(
    raw: np.ndarray,
    kind: str,
    na_sentinel: float = math.nan,
    features_on_rows: bool = True,
) -> DataMatrix:
    """Validate ``raw`` into a read-only features x samples ``DataMatrix``.

    ``features_on_rows=False`` means ``raw`` is samples x features (the
    reference's axis argument, ``datamodel.py:178-180``).
    """
    if kind not in KINDS:
        raise ValueError(f"unknown kind {kind!r}; expected one of {KINDS}")
    arr = np.asarray(raw, dtype=np.float64)
    if arr.ndim != 2 or arr.size == 0:
        raise EmptyMatrix(f"expected a non-empty 2-D matrix, got shape {arr.shape}")
    arr = np.ascontiguousarray(arr if features_on_rows else arr.T)
    arr.setflags(write=False)
    present = present_mask(arr, na_sentinel)
    present.setflags(write=False)
    counts = None
    if kind != "continuous":
        counts = _label_counts(arr, present, kind)
        counts.setflags(write=False)
    return DataMatrix(
        values=arr,
        na_sentinel=na_sentinel,
        kind=kind,
        category_counts=counts,
        present=present,
    )


@dataclass(frozen=True)
class TestRequest:
    """One run's configuration (reference ``datamodel.py:293-338``).

    ``threads`` is accepted for API compatibility; the device path ignores it.
    ``devices`` (an extension, SURVEY §8(b) "a device-count knob without
    changing signatures") shards one run over local GPUs from one process:
    an int N uses devices 0..N-1, a tuple names them (repeats allowed: logical
    shards on one GPU, for testing).  Results never depend on it.
    """

    __test__ = False  # not a pytest class

    test: str
    outputs: tuple[str, ...]
    t_variant: str = "student"
    u_mode: str = "auto"
    threads: int = 1
    features_on_rows: bool = True
    devices: int | tuple[int, ...] = 1

    def __post_init__(self) -> None:
        if isinstance(self.devices, int):
            if self.devices < 1:
                raise ValueError(f"devices must be >= 1, got {self.devices}")
        elif not self.devices or any((not isinstance(d, int)) or d < 0 for d in self.devices):
            raise ValueError(f"devices must be a count or a tuple of device ids, got {self.devices!r}")
        if self.test not in TESTS:
            raise ValueError(f"unknown test {self.test!r}; expected one of {TESTS}")
        if self.t_variant not in T_VARIANTS:
            raise ValueError(
                f"unknown t-test variant {self.t_variant!r}; expected one of {T_VARIANTS}"
            )
        if self.u_mode not in U_MODES:
            raise ValueError(
                f"unknown U-test mode {self.u_mode!r}; expected one of {U_MODES}"
            )
        if self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        allowed = outputs_for(self.test)
        for token in self.outputs:
            if token not in allowed:
                raise UnsupportedOutputForTest(
                    f"output {token!r} is not available for test {self.test!r};"
                    f" valid outputs: {', '.join(allowed)}"
                )
        if not self.outputs:
            raise ValueError("outputs must not be empty")


@dataclass(frozen=True)
class ResultSet:
    """Requested output matrices of one run, all of one shape."""

    matrices: dict[str, np.ndarray]
    shape: tuple[int, int]

    def __post_init__(self) -> None:
        for name, mat in self.matrices.items():
            if mat.shape != self.shape:
                raise ValueError(
                    f"matrix {name!r} has shape {mat.shape}, expected {self.shape}"
                )

    def __getitem__(self, name: str) -> np.ndarray:
        return self.matrices[name]

"""CSV tables for training and prediction: drop-in for ``binboost.dataset``
(/root/reference/pkg/src/binboost/dataset.py), with the per-cell Python
parsing replaced by the library's threaded native reader (bb_csv_*, csrc/
bb_csv.cpp).  Same layout rules, same values (cells follow Python float()),
same error messages with row/column coordinates.

Not covered by the native grammar: non-ASCII digits and whitespace, which
Python's float() also accepts; such cells are reported as not a number.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["DataError", "Dataset", "load_csv", "load_matrix", "make_synthetic"]


class DataError(ValueError):
    """Unusable input data (as opposed to a bad command line argument)."""


@dataclass
class Dataset:
    feature_names: list[str]
    X: np.ndarray        # (n, d) float64
    y: np.ndarray        # (n,) int, +1 signal / -1 background
    weights: np.ndarray  # (n,) float64


class _Table:
    """An opened CSV (records delimited natively) and its header."""

    def __init__(self, path: str):
        self.path = path
        h = C.c_void_p()
        rc = _lib.lib().bb_csv_open(path.encode(), C.byref(h))
        if rc != _lib.BB_OK:
            msg = _lib.lib().bb_last_error().decode("utf-8", "replace")
            # "cannot open <path>: <strerror>" as the reference words it
            raise DataError(msg)
        self.h = h
        nh = _lib.lib().bb_csv_n_header(h)
        if nh < 0:
            self.close()
            raise DataError(f"{path}: empty file")
        self.header = []
        for j in range(nh):
            ln = C.c_int64()
            p = _lib.lib().bb_csv_header(h, j, C.byref(ln))
            self.header.append(C.string_at(p, ln.value).decode("utf-8", "replace").strip())
        self.n = int(_lib.lib().bb_csv_n_records(h))

    def parse(self, cols, finite_col: int = -1) -> np.ndarray:
        cols = np.ascontiguousarray(cols, dtype=np.int32)
        out = np.empty((self.n, cols.size), dtype=np.float64)
        rc = _lib.lib().bb_csv_parse(self.h, _lib.ptr(cols), cols.size, finite_col, 0, _lib.ptr(out))
        if rc == _lib.BB_OK:
            return out
        if rc != _lib.BB_EINVAL:
            _lib.check(rc)
        row, kind, col, cells = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        cp, clen, val = C.c_void_p(), C.c_int64(), C.c_double()
        _lib.lib().bb_csv_error(self.h, C.byref(row), C.byref(kind), C.byref(col), C.byref(cells), C.byref(cp),
                                C.byref(clen), C.byref(val))
        if kind.value == 1:
            raise DataError(f"{self.path}: row {row.value} has {cells.value} cells, expected {len(self.header)}")
        if kind.value == 2:
            cell = C.string_at(cp, clen.value).decode("utf-8", "replace")
            raise DataError(f"{self.path}: row {row.value}, column '{self.header[col.value]}': not a number: {cell!r}")
        raise DataError(f"{self.path}: row {row.value}: non-finite weight {float(val.value)!r}")

    def close(self):
        if getattr(self, "h", None) is not None:
            _lib.lib().bb_csv_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def load_csv(path: str, label: str, weight: str | None = None) -> Dataset:
    """Training / prediction table (dataset.py:31-100): ``label`` names the
    class column ({0,1} or {-1,1}), ``weight`` optionally the weight column,
    every other column is a float feature."""
    with _Table(path) as t:
        header = t.header
        if label not in header:
            raise DataError(f"{path}: no column named '{label}'")
        if weight is not None and weight not in header:
            raise DataError(f"{path}: no column named '{weight}'")
        li = header.index(label)
        wi = header.index(weight) if weight is not None else None
        feat = [j for j in range(len(header)) if j != li and j != wi]
        if not feat:
            raise DataError(f"{path}: no feature columns besides label/weight")
        # every cell is parsed (the reference converts whole rows), the weight
        # column must be finite
        vals = t.parse(np.arange(len(header)), -1 if wi is None else wi)
    if vals.shape[0] == 0:
        raise DataError(f"{path}: no data rows")
    lab = vals[:, li]
    seen = set(np.unique(lab).tolist())
    if not (seen <= {0.0, 1.0} or seen <= {-1.0, 1.0}):
        raise DataError(f"{path}: label column '{label}' must use 0/1 or -1/1, got {sorted(seen)}")
    return Dataset(feature_names=[header[j] for j in feat], X=np.ascontiguousarray(vals[:, feat]),
                   y=np.where(lab > 0, 1, -1),
                   weights=np.ascontiguousarray(vals[:, wi]) if wi is not None else np.ones(vals.shape[0]))


def load_matrix(path: str, exclude: list[str] | None = None) -> tuple[list[str], np.ndarray]:
    """Every column as a float feature minus the ``exclude`` names
    (dataset.py:103-137); only the kept columns are parsed."""
    drop = set(exclude or ())
    with _Table(path) as t:
        keep = [j for j, name in enumerate(t.header) if name not in drop]
        if not keep:
            raise DataError(f"{path}: no feature columns left")
        X = t.parse(keep)
        names = [t.header[j] for j in keep]
    if X.shape[0] == 0:
        raise DataError(f"{path}: no data rows")
    return names, X


def make_synthetic(n_events: int, n_features: int, seed: int, shift: float = 0.5) -> Dataset:
    """Balanced two-class Gaussian toy data (dataset.py:140-155)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = np.where(rng.random(n_events) < 0.5, 1, -1)
    X = rng.standard_normal((n_events, n_features)) + shift * (y == 1)[:, None]
    return Dataset(feature_names=[f"f{j}" for j in range(n_features)], X=X, y=y, weights=np.ones(n_events))

"""Versioned JSON model document, format_version 1.

Interchangeable with the reference's model files
(``pkg/src/binboost/model_io.py:49-91`` writer, ``:111-237`` reader): a
forest fitted on the GPU loads in the reference CLI/binding and vice versa.
Document layout (key order fixed, shortest round-trip floats, no NaN/inf):

    {"format_version": 1,
     "config": {n_trees, depth, shrinkage, subsample, binning_levels, seed} | null,
     "f0": float,
     "binnings": [{"levels": int, "boundaries": [float, ...]}, ...],
     "trees": [{"depth": int,
                "nodes": [{"index", "valid", "featureIndex", "cutBin",
                           "threshold", "gain", "nodeBoostWeight",
                           "nodePurity"}, ...]}, ...]}

Cut fields are null on non-cut nodes.  Errors mirror the reference:
ModelParseError (bad JSON / shape), ModelVersionError, ModelValidationError
(an invariant broken, message names the field).
"""

from __future__ import annotations

import json
import math

import numpy as np

from .engine import FeatureBinning, FitConfig, Forest, Tree

__all__ = ["FORMAT_VERSION", "ModelParseError", "ModelVersionError", "ModelValidationError", "serialize_forest",
           "parse_forest", "save_forest", "load_forest"]

FORMAT_VERSION = 1
_KEYS = ("format_version", "config", "f0", "binnings", "trees")
_CONFIG_FIELDS = ("n_trees", "depth", "shrinkage", "subsample", "binning_levels", "seed")


class ModelParseError(ValueError):
    """Malformed document (bad JSON or wrong shape)."""


class ModelVersionError(ModelParseError):
    """Unknown format_version."""


class ModelValidationError(ModelParseError):
    """Well-formed JSON whose content breaks a model invariant."""


# ------------------------------------------------------------------ writer
def _node_record(tree: Tree, i: int) -> dict:
    cut = i < tree.n_internal and bool(tree.valid[i])
    return {
        "index": i,
        "valid": cut,
        "featureIndex": int(tree.feature[i]) if cut else None,
        "cutBin": int(tree.cut_bin[i]) if cut else None,
        "threshold": float(tree.threshold[i]) if cut else None,
        "gain": float(tree.gain[i]) if cut else None,
        "nodeBoostWeight": float(tree.node_weight[i]),
        "nodePurity": float(tree.node_purity[i]),
    }


def serialize_forest(forest: Forest) -> str:
    cfg = forest.config
    doc = {
        "format_version": FORMAT_VERSION,
        "config": None if cfg is None else {name: getattr(cfg, name) for name in _CONFIG_FIELDS},
        "f0": float(forest.f0),
        "binnings": [{"levels": int(b.levels), "boundaries": [float(x) for x in b.boundaries]}
                     for b in forest.binnings],
        "trees": [{"depth": int(t.depth), "nodes": [_node_record(t, i) for i in range(t.n_nodes)]}
                  for t in forest.trees],
    }
    return json.dumps(doc, indent=2, allow_nan=False) + "\n"


# ------------------------------------------------------------------ reader
class _Checker:
    """Field validators that raise ModelValidationError naming the field."""

    @staticmethod
    def require(ok: bool, field: str, why: str) -> None:
        if not ok:
            raise ModelValidationError(f"{field}: {why}")

    @classmethod
    def number(cls, value, field: str) -> float:
        cls.require(isinstance(value, (int, float)) and not isinstance(value, bool), field, "must be a number")
        x = float(value)
        cls.require(math.isfinite(x), field, "must be finite")
        return x

    @classmethod
    def integer(cls, value, field: str) -> int:
        cls.require(isinstance(value, int) and not isinstance(value, bool), field, "must be an integer")
        return int(value)


def _read_config(c) -> FitConfig | None:
    if c is None:
        return None
    _Checker.require(isinstance(c, dict), "config", "must be an object or null")
    kinds = {"shrinkage": _Checker.number, "subsample": _Checker.number}
    vals = {name: kinds.get(name, _Checker.integer)(c.get(name), f"config.{name}") for name in _CONFIG_FIELDS}
    try:
        return FitConfig(**vals)
    except ValueError as e:
        raise ModelValidationError(f"config: {e}") from e


def _read_binning(b, j: int) -> FeatureBinning:
    where = f"binnings[{j}]"
    _Checker.require(isinstance(b, dict), where, "must be an object")
    levels = _Checker.integer(b.get("levels"), f"{where}.levels")
    raw = b.get("boundaries")
    _Checker.require(isinstance(raw, list), f"{where}.boundaries", "must be a list")
    vals = np.array([_Checker.number(x, f"{where}.boundaries[{k}]") for k, x in enumerate(raw)], dtype=np.float64)
    try:
        return FeatureBinning(boundaries=vals, levels=levels)
    except ValueError as e:
        raise ModelValidationError(f"{where}: {e}") from e


def _read_tree(t, ti: int, binnings) -> Tree:
    where = f"trees[{ti}]"
    _Checker.require(isinstance(t, dict), where, "must be an object")
    depth = _Checker.integer(t.get("depth"), f"{where}.depth")
    _Checker.require(depth >= 1, f"{where}.depth", "must be >= 1")
    n_int, n_nodes = (1 << depth) - 1, (1 << (depth + 1)) - 1
    recs = t.get("nodes")
    _Checker.require(isinstance(recs, list), f"{where}.nodes", "must be a list")
    _Checker.require(len(recs) == n_nodes, f"{where}.nodes", f"must have {n_nodes} records for depth {depth}")
    tree = Tree(depth=depth, feature=np.full(n_int, -1, np.int32), cut_bin=np.zeros(n_int, np.int32),
                threshold=np.full(n_int, np.nan), gain=np.zeros(n_int), valid=np.zeros(n_int, bool),
                node_weight=np.zeros(n_nodes), node_purity=np.zeros(n_nodes))
    for i, r in enumerate(recs):
        w = f"{where}.nodes[{i}]"
        _Checker.require(isinstance(r, dict), w, "must be an object")
        _Checker.require(_Checker.integer(r.get("index"), f"{w}.index") == i, f"{w}.index", f"must equal {i}")
        cut = r.get("valid")
        _Checker.require(isinstance(cut, bool), f"{w}.valid", "must be a boolean")
        tree.node_weight[i] = _Checker.number(r.get("nodeBoostWeight"), f"{w}.nodeBoostWeight")
        tree.node_purity[i] = _Checker.number(r.get("nodePurity"), f"{w}.nodePurity")
        if not cut:
            continue
        _Checker.require(i < n_int, f"{w}.valid", "terminal nodes cannot carry cuts")
        f = _Checker.integer(r.get("featureIndex"), f"{w}.featureIndex")
        _Checker.require(0 <= f < len(binnings), f"{w}.featureIndex", f"must be in [0, {len(binnings) - 1}]")
        cb = _Checker.integer(r.get("cutBin"), f"{w}.cutBin")
        hi = binnings[f].n_bins - 1
        _Checker.require(1 <= cb <= hi, f"{w}.cutBin", f"must be in [1, {hi}]")
        g = _Checker.number(r.get("gain"), f"{w}.gain")
        _Checker.require(g >= 0.0, f"{w}.gain", "must be >= 0")
        tree.feature[i], tree.cut_bin[i], tree.gain[i], tree.valid[i] = f, cb, g, True
        tree.threshold[i] = _Checker.number(r.get("threshold"), f"{w}.threshold")
    return tree


def parse_forest(text: str) -> Forest:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ModelParseError(f"invalid JSON at line {e.lineno}, column {e.colno}: {e.msg}") from e
    _Checker.require(isinstance(doc, dict), "document", "must be a JSON object")
    extra = sorted(set(doc) - set(_KEYS))
    _Checker.require(not extra, "document", f"unknown keys {extra}")
    for key in _KEYS:
        _Checker.require(key in doc, "document", f"missing key '{key}'")
    v = doc["format_version"]
    if isinstance(v, bool) or not isinstance(v, int) or v != FORMAT_VERSION:
        raise ModelVersionError(f"format_version: expected {FORMAT_VERSION}, got {v!r}")
    config = _read_config(doc["config"])
    f0 = _Checker.number(doc["f0"], "f0")
    _Checker.require(isinstance(doc["binnings"], list), "binnings", "must be a list")
    binnings = [_read_binning(b, j) for j, b in enumerate(doc["binnings"])]
    _Checker.require(isinstance(doc["trees"], list), "trees", "must be a list")
    trees = [_read_tree(t, i, binnings) for i, t in enumerate(doc["trees"])]
    return Forest(f0=f0, trees=trees, binnings=binnings, shrinkage=config.shrinkage if config else 1.0,
                  config=config)


def save_forest(forest: Forest, path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(serialize_forest(forest))


def load_forest(path: str) -> Forest:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_forest(fh.read())

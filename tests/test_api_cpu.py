"""Host-side API behaviour that needs no GPU: validation messages mirror the
reference (boosting.py:47-57,138-144,205-213; bridge __init__.py:25-55),
model-file interop with the reference format, sharding arithmetic."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_1609_06119_b200 import FitConfig, bridge, fit_forest, predict_batch
from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree
from paper_1609_06119_b200.model_format import (ModelParseError, ModelValidationError, ModelVersionError,
                                                parse_forest, serialize_forest)
from paper_1609_06119_b200.sharding import class_block_shard, shard_rows, slice_mask


@pytest.mark.parametrize("kw,msg", [(dict(n_trees=0), "n_trees"), (dict(depth=0), "depth"),
                                    (dict(shrinkage=0.0), "shrinkage"), (dict(subsample=1.5), "subsample"),
                                    (dict(binning_levels=0), "binning_levels")])
def test_fitconfig_validation(kw, msg):
    with pytest.raises(ValueError, match=msg):
        FitConfig(**kw)


def test_engine_input_validation():
    with pytest.raises(ValueError, match="2-d"):
        fit_forest(np.zeros(5), np.ones(5))
    with pytest.raises(ValueError, match="both classes"):
        fit_forest(np.zeros((5, 2)), np.ones(5))
    with pytest.raises(ValueError, match="weights has shape"):
        fit_forest(np.zeros((4, 2)), np.array([0, 1, 0, 1]), np.ones(3))
    with pytest.raises(ValueError, match="finite"):
        fit_forest(np.zeros((4, 2)), np.array([0, 1, 0, 1]), np.array([1, np.inf, 1, 1]))


def test_predict_rejects_out_of_range_cut_feature():
    """bb_predict indexes the row by cut feature: a hand-built forest with a
    feature >= n_features is rejected before anything reaches the GPU."""
    from paper_1609_06119_b200.engine import FeatureBinning, Forest, Tree, predict_batch

    t = Tree(depth=1, feature=np.array([3]), cut_bin=np.array([1]), threshold=np.array([0.0]), gain=np.zeros(1),
             valid=np.array([True]), node_weight=np.zeros(3), node_purity=np.zeros(3))
    forest = Forest(f0=0.0, trees=[t], binnings=[FeatureBinning(np.array([0.0]), 1)] * 2)
    with pytest.raises(ValueError, match="out of range"):
        predict_batch(forest, np.zeros((4, 2)))


def test_bridge_validation_messages():
    with pytest.raises(ValueError, match="features must be a 2-d matrix"):
        bridge.fit(np.zeros(4), [0, 1, 0, 1])
    with pytest.raises(ValueError, match="labels length 3 does not match 4 feature rows"):
        bridge.fit(np.zeros((4, 2)), [0, 1, 0])
    with pytest.raises(ValueError, match=r"labels must be 0 or 1, found \[2.0\]"):
        bridge.fit(np.zeros((4, 2)), [0, 1, 2, 1])
    with pytest.raises(ValueError, match="weights shape"):
        bridge.fit(np.zeros((4, 2)), [0, 1, 0, 1], weights=[1, 2])


def _toy_forest():
    b = [FeatureBinning(np.array([0.0]), 1), FeatureBinning(np.array([1.0]), 1)]
    t = Tree(depth=1, feature=np.array([1], np.int32), cut_bin=np.array([1], np.int32), threshold=np.array([1.0]),
             gain=np.array([0.25]), valid=np.array([True]), node_weight=np.array([0.0, -0.1, 0.1]),
             node_purity=np.array([0.5, 0.2, 0.8]))
    return Forest(f0=0.0, trees=[t], binnings=b, shrinkage=0.1, config=FitConfig(n_trees=1, depth=1, binning_levels=1))


def test_model_roundtrip_is_byte_identical():
    text = serialize_forest(_toy_forest())
    assert serialize_forest(parse_forest(text)) == text


def test_reference_model_document_parses_and_reserialises(golden_dir):
    text = open(f"{golden_dir}/ref_model.json").read()
    f = parse_forest(text)
    assert serialize_forest(f) == text  # byte-identical with the reference writer
    assert f.config.n_trees == 5 and len(f.trees) == 5


def test_model_errors():
    with pytest.raises(ModelParseError, match="invalid JSON at line"):
        parse_forest("{")
    with pytest.raises(ModelVersionError):
        parse_forest(serialize_forest(_toy_forest()).replace('"format_version": 1', '"format_version": 2'))
    bad = serialize_forest(_toy_forest()).replace('"cutBin": 1', '"cutBin": 5')
    with pytest.raises(ModelValidationError, match=r"trees\[0\].nodes\[0\].cutBin"):
        parse_forest(bad)


def test_class_block_shard_partition():
    for n_sig, n_bkg, world in [(10, 7, 3), (1, 5, 2), (300_000, 700_000, 8), (0, 4, 2)]:
        covered_s, covered_b = [], []
        for r in range(world):
            (s0, s1), (b0, b1) = class_block_shard(n_sig, n_bkg, r, world)
            covered_s += list(range(s0, s1))
            covered_b += list(range(b0, b1))
        assert covered_s == list(range(n_sig)) and covered_b == list(range(n_bkg))
    y = np.array([1, 0, 0, 1, 1, 0, 1])
    parts = [shard_rows(y, r, 2) for r in range(2)]
    assert sorted(np.concatenate(parts).tolist()) == list(range(7))
    ms, mb = np.array([1, 0, 1, 1], bool), np.array([0, 1, 1], bool)
    assert np.concatenate([slice_mask(ms, mb, r, 2) for r in range(2)]).sum() == ms.sum() + mb.sum()


def test_gpu_written_model_loads_in_reference(golden_dir):
    """A model file written by the GPU binding on a B200
    (tests/golden/gpu_model.json, tools/gen_gpu_model.py) loads through the
    reference's own model_io.load_forest (model_io.py:111-237) and the
    reference's predict_batch reproduces the GPU predictions.  Needs the
    reference tree (build container only)."""
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    sys.path.insert(0, ref)
    try:
        from binboost.boosting import predict_batch as ref_predict
        from binboost.model_io import load_forest as ref_load
    finally:
        sys.path.remove(ref)
    f = ref_load(os.path.join(golden_dir, "gpu_model.json"))
    z = np.load(os.path.join(golden_dir, "gpu_model_inputs.npz"))
    assert len(f.trees) == int(z["trees"])
    np.testing.assert_allclose(ref_predict(f, z["X"]), z["pred"], rtol=0, atol=1e-15)

"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the FastBDT hot path.

This package restates, in numpy, the reference implementation's fit/apply
algorithm (``/root/reference/pkg/src/binboost``: binning.py, sample.py,
trees.py, boosting.py) so parity tests can check the CUDA path against it.

Rules:
- only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import this package;
- it is the checker, never the thing measured or shipped: the product
  package ``paper_1609_06119_b200`` never imports it and fails loudly when
  its CUDA library is missing.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by running the unmodified reference in the build
container (``tests/golden/gen_golden.py``) plus the reference tests'
known-answer vectors.
"""

from .binboost_np import (  # noqa: F401
    OracleForest,
    bin_codes,
    fit_boundaries,
    fit_forest,
    predict,
    predict_scores,
    subsample_masks,
)

"""B200-native FastBDT hot path (arXiv 1609.06119) behind the reference
``binboost`` / ``binboost_bridge`` API.

Engine names mirror ``binboost`` (fit_forest, predict_batch, FitConfig,
Forest, Tree, FeatureBinning); ``bridge`` mirrors ``binboost_bridge``
(fit, load, BoundModel).  All arithmetic of fit and apply runs in the
hand-written sm_100a CUDA library behind include/fastbdt_b200.h.
"""

from .engine import Cut, FeatureBinning, FitConfig, Forest, Tree, fit_forest, predict, predict_batch  # noqa: F401

__version__ = "0.1.0"
__all__ = ["Cut", "FeatureBinning", "FitConfig", "Forest", "Tree", "fit_forest", "predict", "predict_batch"]

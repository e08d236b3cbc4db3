"""paper_1606_05732_b200 -- B200-native CountGauss (T.X = G.(S.X), arXiv 1606.05732).

The hot path (seeded CountSketch construction, the S.X sketch over dense or CSR X, the
Gaussian-fused G.(S.X) contraction, anchor selection) is hand-written sm_100a CUDA in
``csrc/`` behind the C-ABI of ``include/cgx.h`` (``libcgx.so``).  This package is the
host-side mirror of the reference library's API (see :mod:`.api`).
"""
from .api import (AnchorSet, Context, CountGaussTransform, CountSketchMap, SeededRng, SparseMatrix, cg_nmf,
                  context, countgauss_apply, countgauss_new, countsketch_apply, countsketch_batch_gram,
                  countsketch_injective,
                  countsketch_new, gaussian_project, gp_nmf, inverse_normal_cdf, inverse_normal_cdf_array, mix64,
                  select_extremes)

__all__ = [
    "AnchorSet", "Context", "CountGaussTransform", "CountSketchMap", "SeededRng", "SparseMatrix", "cg_nmf",
    "context", "countgauss_apply", "countgauss_new", "countsketch_apply", "countsketch_batch_gram", "countsketch_injective",
    "countsketch_new", "gaussian_project", "gp_nmf", "inverse_normal_cdf", "inverse_normal_cdf_array", "mix64",
    "select_extremes",
]

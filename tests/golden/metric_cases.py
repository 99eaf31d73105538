"""Metric golden cases shared by make_golden.py (values from the reference)
and tests/test_gpu_metrics.py (the device metrics on the same inputs)."""

import numpy as np

METRIC_CASES = [
    # name, data seed, (n_a, n_b, dim), b = a + shift (else a fresh draw), projections, w2 seed, bandwidth
    ("eq", 11, (300, 300, 3), None, 32, 5, 1.0),
    ("uneq", 12, (257, 100, 2), None, 16, 9, 0.7),
    ("shift1d", 13, (200, 200, 1), 1.5, 8, 0, 1.0),
    ("latent", 14, (96, 80, 4096), None, 64, 3, 64.0),
]


def metric_inputs(seed, n_a, n_b, dim, shift):
    """Sample sets of a metrics case: a ~ N(0, 1), b = a + shift or N(0.3, 1.2)."""
    rng = np.random.default_rng(seed)
    a = rng.normal(size=(n_a, dim))
    b = a + shift if shift is not None else rng.normal(0.3, 1.2, size=(n_b, dim))
    return a, b

"""Seeded random vectors for operator parity tests (inputs only)."""
from __future__ import annotations

import numpy as np


def complex_normal(shape, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2.0)

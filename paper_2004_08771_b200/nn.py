"""Model layout of the drop-in surface (mirror of hogtrain.nn's types).

`Architecture` / `Model` / `init_model` follow pkg/src/hogtrain/nn.py:29-105
exactly (same validation, same RNG draws), so a model built here and one
built by the reference are interchangeable: every GPU entry point also
accepts the reference's own `Model` objects (duck-typed on `.arch.layer_sizes`
and `.weights`).  There is no forward/backward here -- that math runs only in
the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np


class InitScheme(Enum):  # nn.py:29-35
    FAN_IN_STD = "fan_in_std"
    SCALED_GAUSSIAN = "scaled_gaussian"


@dataclass(frozen=True)
class Architecture:  # nn.py:37-60
    layer_sizes: tuple

    def __post_init__(self):
        if len(self.layer_sizes) < 2:
            raise ValueError("architecture needs at least input and output layers")
        if any(s < 1 for s in self.layer_sizes):
            raise ValueError(f"layer sizes must be >= 1, got {self.layer_sizes}")

    @property
    def input_dim(self) -> int:
        return self.layer_sizes[0]

    @property
    def class_count(self) -> int:
        return self.layer_sizes[-1]

    @property
    def depth(self) -> int:
        return len(self.layer_sizes) - 1


@dataclass
class Model:  # nn.py:63-78: weights[l] is (d_{l+1}, d_l) float64
    arch: Architecture
    weights: list

    def __post_init__(self):
        sizes = self.arch.layer_sizes
        if len(self.weights) != self.arch.depth:
            raise ValueError("weight count does not match architecture")
        for l, w in enumerate(self.weights):
            if w.shape != (sizes[l + 1], sizes[l]):
                raise ValueError(f"weights[{l}] has shape {w.shape}, expected {(sizes[l + 1], sizes[l])}")


def init_model(arch: Architecture, seed, scheme: InitScheme = InitScheme.SCALED_GAUSSIAN) -> Model:
    """Gaussian weights, std 1/sqrt(fan_in) by default (nn.py:96-105)."""
    rng = np.random.default_rng(seed)
    weights = []
    for l in range(arch.depth):
        fan_in, fan_out = arch.layer_sizes[l], arch.layer_sizes[l + 1]
        std = float(fan_in) if scheme is InitScheme.FAN_IN_STD else 1.0 / np.sqrt(fan_in)
        weights.append(rng.normal(0.0, std, size=(fan_out, fan_in)))
    return Model(arch=arch, weights=weights)


def deep_copy(model) -> Model:
    """Independent snapshot (nn.py:182-184)."""
    return Model(arch=Architecture(tuple(model.arch.layer_sizes)), weights=[np.array(w, copy=True) for w in model.weights])


def layer_sizes_of(model) -> tuple:
    return tuple(int(s) for s in model.arch.layer_sizes)

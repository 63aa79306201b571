"""MLP topology and seeded initialisation (mirror of nystromngd/model.py).

Host-side bookkeeping only: the flat parameter layout (model.py:41-51) is the
layout every device kernel uses, and ``init`` reproduces the reference's
seeded draw bit for bit (model.py:94-100) so theta0 is a shared, seeded input.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class MlpTopology:
    """Layer widths (n0, ..., n_{L+1}); tanh on hidden layers (model.py:12-67)."""

    widths: tuple
    activation: str = "tanh"

    def __post_init__(self):
        if len(self.widths) < 2:
            raise ValueError("topology needs at least input and output widths")
        if any(w < 1 for w in self.widths):
            raise ValueError("layer widths must be >= 1")
        object.__setattr__(self, "widths", tuple(int(w) for w in self.widths))
        if self.activation != "tanh":
            raise ValueError(f"second derivatives unsupported for activation {self.activation!r}")

    @property
    def input_dim(self):
        return self.widths[0]

    @property
    def output_dim(self):
        return self.widths[-1]

    @property
    def param_count(self):
        return sum(o * i + o for i, o in zip(self.widths[:-1], self.widths[1:]))

    @property
    def weight_count(self):
        """P_w = sum n_l n_{l-1} (SURVEY 8 notation)."""
        return sum(o * i for i, o in zip(self.widths[:-1], self.widths[1:]))

    def layer_slices(self):
        out, off = [], 0
        for n_in, n_out in zip(self.widths[:-1], self.widths[1:]):
            ws = slice(off, off + n_out * n_in)
            off += n_out * n_in
            bs = slice(off, off + n_out)
            off += n_out
            out.append((ws, bs, n_out, n_in))
        return out

    def unflatten(self, theta):
        return [(theta[ws].reshape((n_out, n_in)), theta[bs]) for ws, bs, n_out, n_in in self.layer_slices()]

    def flatten(self, layers):
        return np.concatenate([np.concatenate([np.asarray(w).reshape(-1), np.asarray(b).reshape(-1)]) for w, b in layers])


@dataclass(frozen=True)
class ParamVector:
    values: np.ndarray
    topology: MlpTopology

    def __post_init__(self):
        values = np.asarray(self.values, dtype=float)
        if values.shape != (self.topology.param_count,):
            raise ValueError(f"expected {self.topology.param_count} parameters, got {values.shape}")
        object.__setattr__(self, "values", values)

    def __len__(self):
        return self.values.shape[0]


def init(topology, seed):
    """Weights ~ N(0, 1/fan_in), biases zero, drawn layer by layer (model.py:94-100)."""
    rng = np.random.default_rng(seed)
    theta = np.zeros(topology.param_count)
    for ws, _, n_out, n_in in topology.layer_slices():
        theta[ws] = rng.standard_normal(n_out * n_in) / np.sqrt(n_in)
    return ParamVector(theta, topology)


def init_xavier_normal(topology, seed):
    """Xavier-normal weights N(0, 2/(fan_in+fan_out)), zero biases (BASELINE.json's wording)."""
    rng = np.random.default_rng(seed)
    theta = np.zeros(topology.param_count)
    for ws, _, n_out, n_in in topology.layer_slices():
        theta[ws] = rng.standard_normal(n_out * n_in) * np.sqrt(2.0 / (n_in + n_out))
    return ParamVector(theta, topology)

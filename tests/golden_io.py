"""Readers for the committed golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


class Grid(SimpleNamespace):
    """Duck-typed QuantParams (alpha_min, alpha_max, bits, scale)."""

    def __init__(self, arr):
        lo, hi, bits = float(arr[0]), float(arr[1]), int(arr[2])
        super().__init__(alpha_min=lo, alpha_max=hi, bits=bits, scale=(hi - lo) / (1 << bits))


def model_case(d, i: int):
    """Rebuild one golden model case as plain namespaces (oracle-friendly)."""
    p = f"m{i}_"
    layers = []
    for li in range(int(d[p + "n_layers"])):
        q = f"{p}L{li}_"
        in_dim, out_dim, order, act, mode = (int(v) for v in d[q + "meta"])
        bn = None
        if q + "bn" in d:
            mean, var, gamma, beta = d[q + "bn"]
            bn = SimpleNamespace(mean=mean, var=var, gamma=gamma, beta=beta,
                                 eps=float(d[q + "bn_eps"]))
        layers.append(SimpleNamespace(
            in_dim=in_dim, out_dim=out_dim, weight=d[q + "w"],
            weight_params=Grid(d[q + "wgrid"]),
            bias=d[q + "b"] if q + "b" in d else None,
            activation=["none", "relu", "tanh"][act], bn=bn,
            order="aggregate-then-update" if order == 0 else "update-then-aggregate",
            output_mode="bitplanes" if mode == 0 else "full-precision",
            mid_params=Grid(d[q + "mid"]),
            out_params=Grid(d[q + "out"]) if q + "out" in d else None))
    return SimpleNamespace(
        kind=str(d[p + "kind"]), adj_words=d[p + "adj_words"],
        adj_dims=tuple(int(v) for v in d[p + "adj_dims"]), feats=d[p + "feats"],
        feat_words=d[p + "feat_words"], x_params=Grid(d[p + "x_grid"]), layers=layers,
        logits=d[p + "logits"], tally=d[p + "tally"], compound=d[p + "compound"].tobytes(),
        node_ids=d[p + "node_ids"], boundaries=d[p + "boundaries"], degrees=d[p + "degrees"])

"""Shared test helpers: golden-cell decoding and spec/config builders."""

from __future__ import annotations

from paper_2406_18820_b200 import parse_config_string, spec_from_dict
from paper_2406_18820_b200.zoo import make_model

SCALES = {
    "DenseGPT": {"n_layers": 4, "hidden": 64},
    "MoE": {"n_layers": 4, "hidden": 64, "n_experts": 4},
    "GQA": {"n_layers": 4, "hidden": 64, "q_heads": 8, "kv_heads": 2},
}
PIPE_SPECS = {
    "cfg1": ("DenseGPT", {"n_layers": 12, "hidden": 768}),
    "pad": ("DenseGPT", {"n_layers": 2, "hidden": 32}),
    "gqa": ("GQA", SCALES["GQA"]),
    "moe": ("MoE", SCALES["MoE"]),
}


def cell_spec(golden, row):
    """ModelSpec of a golden pipeline cell, via the product's make_model."""
    name = row["name"]
    if name in PIPE_SPECS:
        fam, sc = PIPE_SPECS[name]
    else:
        fam = name.split(".")[0]
        sc = SCALES[fam]
    return make_model(fam, sc)


def cell_cfgs(row):
    return parse_config_string(row["src"]), parse_config_string(row["tgt"])


def golden_spec(golden, key):
    return spec_from_dict(golden["models"][key])

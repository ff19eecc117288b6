"""Model presets (tensor registration sizes) are bit-exact with the reference's
preset_model (golden fixtures from oracle/_ref)."""
import json
import os

import pytest

from paper_2302_12445_b200.presets import PRESETS, preset_param_counts

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_presets_match_reference():
    g = json.load(open(os.path.join(GOLD, "plans.json")))["models"]
    for name in PRESETS:
        for prof in ("uniform", "imbalanced"):
            assert preset_param_counts(name, prof) == g[f"{name}/{prof}"]["param_counts"]
    assert preset_param_counts("mlp4x1024") == g["mlp4x1024"]["param_counts"]


def test_unknown_preset_names_alternatives():
    with pytest.raises(ValueError, match="resnet50"):
        preset_param_counts("alexnet")

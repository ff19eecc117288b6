"""The product's host partitioner and shard layout (libdear.so, C ABI) are
bit-exact with the reference (golden fixtures from oracle/_ref) — no GPU."""
import json
import os

import numpy as np
import pytest

import paper_2302_12445_b200 as dear

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_plans_bit_exact_with_reference():
    g = _load("plans.json")
    n = 0
    for name, m in g["models"].items():
        bytes_ = [4 * c for c in m["param_counts"]]
        for buf, groups in m["plans"].items():
            assert dear.build_fusion_plan(bytes_, int(buf)) == [tuple(x) for x in groups], \
                (name, buf)
            n += 1
    assert n > 100


def test_survey_goldens():
    """SURVEY §8(a) golden partitions (reference output)."""
    mlp = [4 * 1_049_600] * 4
    assert dear.build_fusion_plan(mlp, 4_000_000) == [(4, 4), (3, 3), (2, 2), (1, 1)]
    assert dear.build_fusion_plan(mlp, 8_396_800) == [(3, 4), (1, 2)]
    assert dear.build_fusion_plan(mlp, 16_000_000) == [(2, 4), (1, 1)]
    assert dear.build_fusion_plan(mlp, 25_000_000) == [(1, 4)]
    g = _load("plans.json")["models"]
    rn = [4 * c for c in g["resnet50/uniform"]["param_counts"]]
    assert dear.build_fusion_plan(rn, 25_000_000) == [(123, 161), (84, 122), (45, 83), (6, 44),
                                                     (1, 5)]
    bl = [4 * c for c in g["bert_large/uniform"]["param_counts"]]
    p = dear.build_fusion_plan(bl, 25_000_000)
    assert len(p) == 57 and p[0] == (392, 398) and p[-2] == (7, 13) and p[-1] == (1, 6)
    counts = {"resnet50/uniform": (161, 27, 5, 2, 2), "bert_base/uniform": (206, 206, 19, 8, 5),
              "bert_large/uniform": (398, 398, 57, 23, 14)}
    for k, want in counts.items():
        b = [4 * c for c in g[k]["param_counts"]]
        got = tuple(len(dear.build_fusion_plan(b, x)) for x in
                    (1_000_000, 4_000_000, 25_000_000, 64_000_000, 100_000_000))
        assert got == want, k


def test_chunk_layout_bit_exact():
    for c in _load("chunks.json")["cases"]:
        r = dear.chunk_ranges(c["d"], c["P"])
        assert [a for a, _ in r] == c["begin"] and [b for _, b in r] == c["end"]


def test_owner_and_slot_maps():
    for P in (1, 2, 3, 4, 8):
        for c in range(P):
            r = dear.chunk_owner(c, P)
            assert dear.slot_chunk(r, P) == c  # slot r carries chunk (r+1) mod P
        assert sorted(dear.chunk_owner(c, P) for c in range(P)) == list(range(P))


def test_slot_stride():
    for d, P in ((0, 1), (1, 1), (4198400, 2), (5913061, 8), (7, 3)):
        s = dear.slot_stride(d, P)
        assert s % 64 == 0 and s >= -(-d // P) and s - (-(-d // P)) < 64


def test_errors_mirror_reference():
    with pytest.raises(ValueError, match="empty model"):
        dear.build_fusion_plan([], 1_000_000)
    with pytest.raises(ValueError, match="param_count must be >= 0"):
        dear.build_fusion_plan([4, -4], 1_000_000)
    with pytest.raises(ValueError, match="buffer_bytes must be > 0"):
        dear.build_fusion_plan([4], -1)
    with pytest.raises(ValueError, match="workers must be >= 1"):
        dear.chunk_ranges(10, 0)
    with pytest.raises(ValueError, match="d_elems must be >= 0"):
        dear.chunk_ranges(-1, 2)


def test_random_against_restatement(restated):
    rng = np.random.default_rng(99)
    for _ in range(300):
        L = int(rng.integers(1, 120))
        b = (rng.integers(0, 3_000_000, L) * 4).tolist()
        buf = int(rng.choice([0, 1, 1_000_000, 4_000_000, 25_000_000, 10**12]))
        assert dear.build_fusion_plan(b, buf) == restated.build_fusion_plan(b, buf)

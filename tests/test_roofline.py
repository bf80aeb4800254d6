"""Pins for the byte/flop accounting used by bench.py's roofline (host logic)."""
import json
import os

import pytest

from paper_2512_00722_b200 import roofline

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


@pytest.mark.parametrize("case", GOLD["kv_bytes"])
def test_kv_bytes_paper_anchor(case):
    assert roofline.kv_bytes(case["L"], case["H"], case["D"], case["S"],
                             case["bytes_per_elem"]) == case["expect"]


@pytest.mark.parametrize("case", GOLD["retrieval_overhead_eq3"])
def test_eq3(case):
    assert roofline.retrieval_overhead(*case["args"]) == case["expect"]


def test_step_bytes_config_b():
    # 67,108,864 + 268,435,456 = 335,544,320 bytes for config B
    assert roofline.score_bytes([32768], 8, 128) == 67108864
    assert roofline.attn_bytes([32768], 32, 8, 128, 2048) == 268435456
    assert roofline.step_bytes([32768], 32, 8, 128, 2048) == 335544320
    # the selected-KV term is the dense KV formula at S = k (P:225 scaling)
    assert roofline.attn_bytes([32768], 32, 8, 128, 2048) == roofline.kv_bytes(32, 8, 128, 2048)
    # config A: 524,288 + 65,536
    assert roofline.step_bytes([4096], 1, 1, 64, 256) == 589824
    # Eq.3 with layers = 1 is the scoring FMA count
    assert roofline.step_flops([1024], 0, 32, 128, 0) == 2 * roofline.retrieval_overhead(
        1, 1, 32, 128, 1024)

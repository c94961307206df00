"""Loads tests/golden/oracle_golden.json (written by tests/golden/make_golden.py)."""

import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_golden.json")


def load_golden():
    with open(GOLDEN) as f:
        return json.load(f)


def f32hex(x: float) -> str:
    return np.float32(x).tobytes().hex()


def check_golden():
    import oracle_lib as o
    for case in load_golden():
        m = o.OracleModel.create(case["cfg"], seed=case["seed"])
        for key, int8 in (("int8", True), ("f32", False)):
            want = case["results"][key]
            hyps = m.translate_batch(case["sources"], case["beam"], 0, 1.0, int8=int8)
            assert [h["tokens"] for h in hyps] == want["tokens"], (case["name"], key)
            assert [f32hex(h["logprob"]) for h in hyps] == want["logprob_hex"], (case["name"], key)
            forced = m.forced_logits(case["sources"][0], [4, 5, 6], int8=int8)
            assert hashlib.sha256(forced.tobytes()).hexdigest() == want["forced_logits_sha"], (
                case["name"], key)

"""Regenerates tests/golden/oracle_golden.json from the CPU oracle.

The reference (minimt) cannot be built or imported in this image (Eigen3 and
vendor/ are absent), so these vectors come from the oracle restatement, which
tests/test_oracle_kats.py pins to the reference's own KATs. They freeze the
oracle's outputs (int8 bit patterns included) so both the oracle build on
another host and the GPU path are checked against the same committed numbers.

    python tests/golden/make_golden.py
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as o  # noqa: E402

CASES = [
    dict(name="micro_1_1", seed=51, beam=3, n=4, slen=4,
         cfg=dict(num_encoder_layers=1, num_decoder_layers=1, d_model=8, d_ff=16, num_heads=2,
                  src_vocab_size=12, tgt_vocab_size=12, dropout=0.0, max_seq_len=32)),
    dict(name="tiny_2_2", seed=11, beam=4, n=5, slen=6,
         cfg=dict(num_encoder_layers=2, num_decoder_layers=2, d_model=16, d_ff=32, num_heads=2,
                  src_vocab_size=11, tgt_vocab_size=13, dropout=0.0, max_seq_len=32)),
    dict(name="small_3_2", seed=5, beam=5, n=6, slen=9,
         cfg=dict(num_encoder_layers=3, num_decoder_layers=2, d_model=64, d_ff=256, num_heads=4,
                  src_vocab_size=700, tgt_vocab_size=900, dropout=0.1, max_seq_len=64)),
]


def f32hex(x: float) -> str:
    return np.float32(x).tobytes().hex()


def build():
    out = []
    for c in CASES:
        m = o.OracleModel.create(c["cfg"], seed=c["seed"])
        srcs = o.synthetic_sources(c["n"], c["slen"], c["cfg"]["src_vocab_size"], seed=c["seed"])
        entry = dict(name=c["name"], seed=c["seed"], beam=c["beam"], cfg=c["cfg"], sources=srcs,
                     results={})
        for int8 in (True, False):
            hyps = m.translate_batch(srcs, c["beam"], 0, 1.0, int8=int8)
            forced = m.forced_logits(srcs[0], [4, 5, 6], int8=int8)
            entry["results"]["int8" if int8 else "f32"] = dict(
                tokens=[h["tokens"] for h in hyps],
                logprob_hex=[f32hex(h["logprob"]) for h in hyps],
                norm_hex=[f32hex(h["norm"]) for h in hyps],
                finished=[h["finished"] for h in hyps],
                forced_logits_sha=__import__("hashlib").sha256(forced.tobytes()).hexdigest(),
                forced_logits_head=[float(v) for v in forced[:, :4].ravel()],
            )
        out.append(entry)
    return out


if __name__ == "__main__":
    data = build()
    with open(os.path.join(HERE, "oracle_golden.json"), "w") as f:
        json.dump(data, f, indent=1)
    print("wrote", len(data), "cases")

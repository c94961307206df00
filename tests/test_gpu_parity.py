"""End-to-end parity of the B200 translation path (C ABI) with the CPU oracle.

Bars (BASELINE.json north_star):
  int8  -- bit-exact: encoder rows, per-step logits, tokens, logprob and
           normalised-score bits.
  fp32  -- identical hypotheses (>= 99% of sentences; all in practice) and
           logits / scores within 1e-3 relative.
  bf16  -- logits within 5e-2 relative to the fp32 oracle (stated tolerance).
"""

import os

import numpy as np
import pytest

import oracle_lib as o
import paper_2008_04885_b200 as mt
from golden_util import f32hex, load_golden

pytestmark = pytest.mark.gpu


def cfg(enc=2, dec=2, d=16, ff=32, heads=2, vs=11, vt=13, msl=32, dropout=0.0):
    return dict(num_encoder_layers=enc, num_decoder_layers=dec, d_model=d, d_ff=ff,
                num_heads=heads, src_vocab_size=vs, tgt_vocab_size=vt, dropout=dropout,
                max_seq_len=msl)


MID = cfg(3, 2, 64, 256, 4, 700, 900, 64)
BIG = cfg(20, 2, 512, 2048, 8, 32000, 32000, 128, 0.1)


def derive(src, msl):
    return min(msl, 2 * len(src) + 5)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


# ---- golden fixtures ------------------------------------------------------------

@pytest.mark.parametrize("case", load_golden(), ids=lambda c: c["name"])
def test_golden_int8_bit_exact(case):
    m = mt.Model.create(case["cfg"], seed=case["seed"], precision=mt.INT8)
    hyps = m.translate(case["sources"], mt.BeamConfig(case["beam"], 0, 1.0))
    want = case["results"]["int8"]
    assert [h.tokens for h in hyps] == want["tokens"]
    assert [f32hex(h.logprob) for h in hyps] == want["logprob_hex"]
    assert [f32hex(h.normalized) for h in hyps] == want["norm_hex"]
    assert [h.finished for h in hyps] == want["finished"]


@pytest.mark.parametrize("case", load_golden(), ids=lambda c: c["name"])
def test_golden_f32_within_tolerance(case):
    m = mt.Model.create(case["cfg"], seed=case["seed"], precision=mt.F32)
    hyps = m.translate(case["sources"], mt.BeamConfig(case["beam"], 0, 1.0))
    want = case["results"]["f32"]
    assert [h.tokens for h in hyps] == want["tokens"]
    for h, hx in zip(hyps, want["logprob_hex"]):
        ref = float(np.frombuffer(bytes.fromhex(hx), np.float32)[0])
        assert abs(h.logprob - ref) <= 1e-3 * abs(ref) + 1e-6


# ---- layer-level parity -------------------------------------------------------------

@pytest.mark.parametrize("config", [cfg(), cfg(1, 1, 8, 16, 2, 12, 12), MID, cfg(0, 1, 16, 32, 4)],
                         ids=["tiny", "micro", "mid", "enc0"])
def test_encode_and_step_logits(config):
    om = o.OracleModel.create(config, seed=3)
    srcs = o.synthetic_sources(3, 5, config["src_vocab_size"], seed=9)
    forced = [4, 5, 6, 7, 8]
    for prec in (mt.INT8, mt.F32):
        gm = mt.Model.create(config, seed=3, precision=prec)
        int8 = prec == mt.INT8
        enc = gm.encode(srcs)
        ref_enc = np.concatenate([om.encode(s, int8) for s in srcs])
        lg = gm.forced_logits(srcs, forced)
        ref_lg = np.stack([om.forced_logits(s, forced, int8) for s in srcs])
        if int8:
            assert np.array_equal(enc, ref_enc)
            assert np.array_equal(lg, ref_lg)
        else:
            assert rel(enc, ref_enc) < 1e-4
            assert rel(lg, ref_lg) < 1e-4


@pytest.mark.parametrize("batch", [1, 6], ids=["b1", "b6"])
def test_encoder_long_and_short_sentences_bit_exact(batch):
    """Encoder attention paths: sentences up to 32 tokens (a warp's queries
    attended together; split over several CTAs at small batches) and longer
    ones (query per warp), mixed in one batch; int8 encoder states and
    forced logits bit-exact against the oracle, fp32 within 1e-4."""
    c = cfg(2, 1, 64, 128, 1, 500, 300, 128)  # one head of 64
    om = o.OracleModel.create(c, seed=11)
    lens = [5, 31, 33, 60, 17, 45][:batch] if batch > 1 else [47]
    srcs = [o.synthetic_sources(1, n, c["src_vocab_size"], seed=40 + n)[0] for n in lens]
    forced = [4, 5, 6]
    for prec in (mt.INT8, mt.F32):
        gm = mt.Model.create(c, seed=11, precision=prec)
        int8 = prec == mt.INT8
        enc = gm.encode(srcs)
        ref_enc = np.concatenate([om.encode(s, int8) for s in srcs])
        lg = gm.forced_logits(srcs, forced)
        ref_lg = np.stack([om.forced_logits(s, forced, int8) for s in srcs])
        if int8:
            assert np.array_equal(enc, ref_enc)
            assert np.array_equal(lg, ref_lg)
        else:
            assert rel(enc, ref_enc) < 1e-4
            assert rel(lg, ref_lg) < 1e-4


def test_encoder_192_column_tiles_fp32():
    """64 sentences x 25 tokens at d = 512 give the fp32 encoder QKV / FFN-up
    GEMMs 156 / 208 128-column tiles (just over one wave), which the planner
    runs as 104 / 143 192-column tiles; encoder states within the fp32 bar
    (bf16 QKV takes the same tiles)."""
    c = cfg(2, 1, 512, 2048, 8, 3000, 300, 64)
    om = o.OracleModel.create(c, seed=13)
    srcs = o.synthetic_sources(64, 25, c["src_vocab_size"], seed=77)
    ref = np.concatenate([om.encode(s, False) for s in srcs])
    gm = mt.Model.create(c, seed=13, precision=mt.F32)
    assert rel(gm.encode(srcs), ref) < 1e-4
    gb = mt.Model.create(c, seed=13, precision=mt.BF16)
    assert rel(gb.encode(srcs), ref) < 5e-2


def test_incremental_matches_teacher_forced_on_gpu():  # test_model.cpp:211-228, C2
    worst = 0.0
    for trial in range(12):
        rng = np.random.default_rng(1000 + trial)
        d = 8 << int(rng.integers(0, 3))
        heads = 2 if rng.integers(0, 2) else 4
        c = cfg(int(1 + rng.integers(0, 2)), int(1 + rng.integers(0, 2)), d, 2 * d, heads,
                int(8 + rng.integers(0, 13)), int(8 + rng.integers(0, 13)), 64)
        om = o.OracleModel.create(c, seed=900 + trial)
        gm = mt.Model.create(c, seed=900 + trial, precision=mt.F32)
        src = [int(4 + rng.integers(0, c["src_vocab_size"] - 4)) for _ in range(1 + rng.integers(0, 6))] + [3]
        tgt = [int(4 + rng.integers(0, c["tgt_vocab_size"] - 4)) for _ in range(1 + rng.integers(0, 6))] + [3]
        worst = max(worst, float(np.abs(gm.forced_logits([src], tgt)[0] - om.teacher_forced(src, tgt)).max()))
    assert worst <= 1e-4


def test_bf16_logits_within_stated_tolerance():
    om = o.OracleModel.create(MID, seed=3)
    gm = mt.Model.create(MID, seed=3, precision=mt.BF16)
    srcs = o.synthetic_sources(2, 7, MID["src_vocab_size"], seed=4)
    lg = gm.forced_logits(srcs, [4, 5, 6])
    ref = np.stack([om.forced_logits(s, [4, 5, 6]) for s in srcs])
    assert rel(lg, ref) < 5e-2


# ---- search semantics -------------------------------------------------------------------

@pytest.mark.parametrize("beam", [1, 2, 5, 10, 16])
def test_beam_sizes_bit_exact_int8(beam):
    om = o.OracleModel.create(MID, seed=21)
    gm = mt.Model.create(MID, seed=21, precision=mt.INT8)
    srcs = o.synthetic_sources(5, 6, MID["src_vocab_size"], seed=beam)
    hyps = gm.translate(srcs, mt.BeamConfig(beam, 0, 1.0))
    for s, h in zip(srcs, hyps):
        r = om.beam_search(s, beam, derive(s, 64), 1.0, True)
        assert (h.tokens, f32hex(h.logprob), h.finished, h.truncated) == (
            r["tokens"], f32hex(r["logprob"]), r["finished"], r["truncated"])


def test_beam_larger_than_vocab_and_alpha():
    c = cfg(1, 1, 8, 16, 2, 6, 6, 16)
    om = o.OracleModel.create(c, seed=2)
    gm = mt.Model.create(c, seed=2, precision=mt.INT8)
    srcs = [[4, 5, 3], [5, 3], [4, 4, 4, 5, 3]]
    for beam, alpha in ((8, 1.0), (3, 0.0), (4, 0.6), (2, 2.0)):
        hyps = gm.translate(srcs, mt.BeamConfig(beam, 7, alpha))
        for s, h in zip(srcs, hyps):
            r = om.beam_search(s, beam, 7, alpha, True)
            assert h.tokens == r["tokens"]
            assert f32hex(h.logprob) == f32hex(r["logprob"])
            assert f32hex(h.normalized) == f32hex(r["norm"])


def test_beam1_equals_greedy_on_gpu():  # test_decode.cpp:52-76
    c = cfg(1, 1, 8, 16, 2, 12, 12, 32)
    gm = mt.Model.create(c, seed=51, precision=mt.F32)
    src = [4, 7, 5, 3]
    h = gm.translate([src], mt.BeamConfig(1, 10, 0.0))[0]
    greedy = []
    for t in range(10):
        lg = gm.forced_logits([src], greedy + [0])[0][t]
        best = int(np.argmax(lg))
        if best == mt.EOS_ID:
            break
        greedy.append(best)
    assert h.tokens == greedy


def test_finished_hypotheses_gnmt_selection():
    """A model biased towards EOS exercises the finished list + GNMT pick."""
    c = cfg(1, 1, 16, 32, 2, 20, 20, 32)
    om = o.OracleModel.create(c, seed=5)
    te = om.get("tgt_embed", (20, 16))
    te[3] *= 4.0  # make EOS logits large
    om.set("tgt_embed", te)
    path = "/tmp/eos_biased.bin"
    om.save(path)
    gm8 = mt.Model.load(path, precision=mt.INT8)
    srcs = o.synthetic_sources(8, 5, 20, seed=1)
    n_fin = 0
    for s, h in zip(srcs, gm8.translate(srcs, mt.BeamConfig(4, 0, 1.0))):
        r = om.beam_search(s, 4, derive(s, 32), 1.0, True)
        assert h.tokens == r["tokens"] and h.finished == r["finished"]
        assert f32hex(h.normalized) == f32hex(r["norm"])
        n_fin += h.finished
    assert n_fin > 0


def test_uniform_zero_model_latency_fixture(tmp_path):  # test_decode.cpp:171-206
    om = o.OracleModel.create(cfg(1, 1, 8, 16, 2, 8, 8, 32), seed=1, init=False)
    p = str(tmp_path / "zero.bin")
    om.save(p)
    for prec in (mt.F32, mt.INT8):
        gm = mt.Model.load(p, precision=prec)
        hyps = gm.translate([mt.prepare_source([4, 5], 32)] * 10, mt.BeamConfig(1, 3, 1.0))
        assert all(h.tokens == [0, 0, 0] and h.truncated for h in hyps)
        assert sum(len(h.tokens) for h in hyps) == 30


def test_batch_composition_invariance():
    """Per-sentence results do not depend on what else is in the batch
    (per-sentence int8 scales)."""
    gm = mt.Model.create(MID, seed=8, precision=mt.INT8)
    srcs = o.synthetic_sources(9, 7, MID["src_vocab_size"], seed=8)
    srcs[2] = srcs[2][:3] + [3]
    srcs[5] = srcs[5] * 3
    batch = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))
    split = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0), max_batch=2)
    for i, s in enumerate(srcs):
        alone = gm.translate([s], mt.BeamConfig(5, 0, 1.0))[0]
        for other in (batch[i], split[i]):
            assert (other.tokens, f32hex(other.logprob)) == (alone.tokens, f32hex(alone.logprob))


def test_per_sentence_errors_and_call_errors():  # decode.cpp:38-39, model.cpp:548, tensor.cpp:456
    c = cfg(1, 1, 8, 16, 2, 12, 12, 8)
    gm = mt.Model.create(c, seed=1, precision=mt.INT8)
    srcs = [[4, 3], [], [4] * 9 + [3], [4, 99, 3], [5, 3]]
    hyps = gm.translate(srcs, mt.BeamConfig(2, 0, 1.0))
    assert [h.status for h in hyps] == [0, 6, 2, 3, 0]
    om = o.OracleModel.create(c, seed=1)
    assert hyps[4].tokens == om.beam_search([5, 3], 2, derive([5, 3], 8), 1.0, True)["tokens"]
    with pytest.raises(mt.UsageError):
        gm.translate(srcs, mt.BeamConfig(0, 0, 1.0))
    # explicit max_len beyond max_seq_len: decode_step throws past the cap
    hyp = gm.translate([[4, 3]], mt.BeamConfig(2, 20, 1.0))[0]
    assert hyp.status == 2


# ---- persistence interop (io.cpp / model.cpp:699-807) --------------------------------------

def test_sqnt_interop_with_oracle(tmp_path):
    om = o.OracleModel.create(MID, seed=12)
    f32p, q8p = str(tmp_path / "f.bin"), str(tmp_path / "q.bin")
    om.save(f32p)
    om.save(q8p, quantized=True)
    srcs = o.synthetic_sources(4, 6, MID["src_vocab_size"], seed=12)
    ref = [om.beam_search(s, 5, derive(s, 64), 1.0, True) for s in srcs]
    for path, prec in ((f32p, mt.INT8), (q8p, mt.F32), (q8p, mt.INT8)):
        gm = mt.Model.load(path, precision=prec)
        assert gm.precision == mt.INT8  # quantized files always decode int8
        hyps = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))
        assert [h.tokens for h in hyps] == [r["tokens"] for r in ref]
        assert [f32hex(h.logprob) for h in hyps] == [f32hex(r["logprob"]) for r in ref]
    # the GPU side writes byte-identical SQNT files
    gm = mt.Model.create(MID, seed=12, precision=mt.F32)
    gpath = str(tmp_path / "g.bin")
    gm.save(gpath)
    assert open(gpath, "rb").read() == open(f32p, "rb").read()
    gq = mt.Model.create(MID, seed=12, precision=mt.INT8)
    gqpath = str(tmp_path / "gq.bin")
    gq.save(gqpath)
    assert open(gqpath, "rb").read() == open(q8p, "rb").read()
    with open(f32p, "r+b") as f:
        f.truncate(os.path.getsize(f32p) - 3)
    with pytest.raises(mt.FormatError):
        mt.Model.load(f32p)


# ---- full-size configs (BASELINE.json configs[1], [3]) ------------------------------------

@pytest.fixture(scope="module")
def big_oracle():
    return o.OracleModel.create(BIG, seed=1)


def test_20_2_int8_bit_exact(big_oracle):
    gm = mt.Model.create(BIG, seed=1, precision=mt.INT8)
    srcs = o.synthetic_sources(3, 25, 32000, seed=7)
    srcs[1] = srcs[1][:11] + [3]
    hyps = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))
    for s, h in zip(srcs, hyps):
        r = big_oracle.beam_search(s, 5, derive(s, 128), 1.0, True)
        assert (h.tokens, f32hex(h.logprob), f32hex(h.normalized)) == (
            r["tokens"], f32hex(r["logprob"]), f32hex(r["norm"]))
    lg = gm.forced_logits(srcs[:1], [5, 6, 7])
    assert np.array_equal(lg[0], big_oracle.forced_logits(srcs[0], [5, 6, 7], True))


def test_20_2_f32_within_tolerance(big_oracle):
    gm = mt.Model.create(BIG, seed=1, precision=mt.F32)
    srcs = o.synthetic_sources(2, 25, 32000, seed=7)
    hyps = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))
    for s, h in zip(srcs, hyps):
        r = big_oracle.beam_search(s, 5, derive(s, 128), 1.0, False)
        assert h.tokens == r["tokens"]
        assert abs(h.logprob - r["logprob"]) <= 1e-3 * abs(r["logprob"])
    lg = gm.forced_logits(srcs[:1], [5, 6, 7])[0]
    assert rel(lg, big_oracle.forced_logits(srcs[0], [5, 6, 7], False)) < 1e-3


def test_ragged_lengths_batch_bit_exact():
    """configs[4]-style ragged lengths (5..60 tokens) in one length-bucketed call."""
    c = cfg(4, 2, 128, 512, 8, 2000, 2500, 128)
    om = o.OracleModel.create(c, seed=4)
    gm = mt.Model.create(c, seed=4, precision=mt.INT8)
    rng = np.random.default_rng(4)
    srcs = [list(map(int, rng.integers(4, 2000, int(n)))) + [3] for n in rng.integers(5, 61, 10)]
    hyps = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0), max_batch=4)
    for s, h in zip(srcs, hyps):
        r = om.beam_search(s, 5, derive(s, 128), 1.0, True)
        assert (h.tokens, f32hex(h.logprob)) == (r["tokens"], f32hex(r["logprob"]))


def test_topk_ties_across_slices_bit_exact(tmp_path):
    """Duplicated output-embedding rows make many logits tie across the
    32-column slices: the softmax/top-k merge must rescan every tied slice
    (long-list path) and still rank by (score desc, token asc)."""
    c = cfg(1, 1, 16, 32, 2, 20, 2000, 32)
    om = o.OracleModel.create(c, seed=11)
    te = om.get("tgt_embed", (2000, 16))
    om.set("tgt_embed", np.ascontiguousarray(te[np.arange(2000) % 7]))
    p = str(tmp_path / "ties.bin")
    om.save(p)
    srcs = o.synthetic_sources(6, 6, 20, seed=4)
    gm8 = mt.Model.load(p, precision=mt.INT8)
    for s, h in zip(srcs, gm8.translate(srcs, mt.BeamConfig(5, 0, 1.0))):
        r = om.beam_search(s, 5, derive(s, 32), 1.0, True)
        assert h.tokens == r["tokens"]
        assert f32hex(h.logprob) == f32hex(r["logprob"])
    gm32 = mt.Model.load(p, precision=mt.F32)
    for s, h in zip(srcs, gm32.translate(srcs, mt.BeamConfig(5, 0, 1.0))):
        assert h.tokens == om.beam_search(s, 5, derive(s, 32), 1.0, False)["tokens"]


def test_step_fusion_modes_agree():
    """The decode-step start can run as three kernels (default) or fused
    (MTG_STEP_FUSION=1/2); every mode gives the same bits."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2008_04885_b200 as mt, oracle_lib as o\n"
        "from golden_util import f32hex\n"
        "c = dict(num_encoder_layers=2, num_decoder_layers=2, d_model=64, d_ff=256, num_heads=4,"
        " src_vocab_size=700, tgt_vocab_size=900, dropout=0.0, max_seq_len=64)\n"
        "gm = mt.Model.create(c, seed=3, precision=mt.INT8)\n"
        "srcs = o.synthetic_sources(12, 9, 700, seed=2)\n"
        "print([(h.tokens, f32hex(h.logprob)) for h in gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))])\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))
    outs = []
    variants = [dict(MTG_STEP_FUSION="0"), dict(MTG_STEP_FUSION="1"), dict(MTG_STEP_FUSION="2"),
                dict(MTG_FUSED_TAIL="0"), dict(MTG_LOGITS_PERSISTENT="1"),
                dict(MTG_NO_SPLIT_K="1"), dict(MTG_ENC_GRAPH="0"), dict(MTG_NO_ENC_FUSION="1"),
                dict(MTG_STEPS_PER_GRAPH="1"), dict(MTG_DEVICE_LOOP="0"),
                dict(MTG_SPLIT_CTAS="148"), dict(MTG_MIN_BN="64"), dict(MTG_NO_PDL="1"),
                dict(MTG_FOLD_REORDER="0"), dict(MTG_SPLITK_DIST="0"), dict(MTG_CLUSTER_CAP="0"),
                dict(MTG_SMALL_BATCH="0")]
    for v in variants:  # every A/B switch must leave the bits unchanged
        env = dict(os.environ, **v)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, check=True,
                                   capture_output=True, text=True).stdout)
    assert outs[0].strip() and all(o == outs[0] for o in outs)


@pytest.mark.gpu
def test_bf16_direct_operands_agree():
    """bf16 encoder: the attention and the FFN-up GEMM write the bf16
    operands themselves (default) or through cast kernels
    (MTG_BF16_DIRECT=0): both round the same fp32 values, so the results are
    identical."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2008_04885_b200 as mt, oracle_lib as o\n"
        "from golden_util import f32hex\n"
        "c = dict(num_encoder_layers=2, num_decoder_layers=2, d_model=128, d_ff=512, num_heads=2,"
        " src_vocab_size=700, tgt_vocab_size=900, dropout=0.0, max_seq_len=64)\n"
        "gm = mt.Model.create(c, seed=3, precision=mt.BF16)\n"
        "srcs = o.synthetic_sources(12, 9, 700, seed=2) + o.synthetic_sources(3, 40, 700, seed=5)\n"
        "print([(h.tokens, f32hex(h.logprob)) for h in gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))])\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("1", "0"):
        env = dict(os.environ, MTG_BF16_DIRECT=v)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, check=True,
                                   capture_output=True, text=True).stdout)
    assert outs[0].strip() and outs[0] == outs[1]


@pytest.mark.gpu
def test_f32_projection_kernels_agree():
    """The fp32 output projection runs on CTA pairs (cta_group::2, default),
    one persistent CTA per tile (MTG_LOGITS_PAIR=0) or one tile per CTA
    (MTG_LOGITS_PERSISTENT=0): same hypotheses and score bits. 60 sentences x
    beam 5 = 300 rows covers a second, partly live pair tile; 30 sentences
    (150 rows) one pair tile whose second CTA is partly live; 1 sentence the
    single-CTA kernel."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_2008_04885_b200 as mt, oracle_lib as o\n"
        "from golden_util import f32hex\n"
        "c = dict(num_encoder_layers=2, num_decoder_layers=2, d_model=64, d_ff=256, num_heads=4,"
        " src_vocab_size=700, tgt_vocab_size=900, dropout=0.0, max_seq_len=64)\n"
        "gm = mt.Model.create(c, seed=3, precision=mt.F32)\n"
        "srcs = o.synthetic_sources(60, 9, 700, seed=2)\n"
        "print([(h.tokens, f32hex(h.logprob)) for h in gm.translate(srcs, mt.BeamConfig(5, 0, 1.0))])\n"
        "print([(h.tokens, f32hex(h.logprob)) for h in gm.translate(srcs[:1], mt.BeamConfig(5, 0, 1.0))])\n"
        "print([(h.tokens, f32hex(h.logprob)) for h in gm.translate(srcs[:30], mt.BeamConfig(5, 0, 1.0))])\n"
    ) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in (dict(), dict(MTG_LOGITS_PAIR="0"), dict(MTG_LOGITS_PERSISTENT="0")):
        env = dict(os.environ, **v)
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, check=True,
                                   capture_output=True, text=True, timeout=300).stdout)
    assert outs[0].strip() and all(o == outs[0] for o in outs)


@pytest.mark.parametrize("combine,shared", [("concat", False), ("sum", False), ("average", True),
                                            ("sum", True)])
def test_source_factors_bit_exact(combine, shared):
    """Source-factor embedding (model.cpp:539-581): concat / sum / average,
    own or shared tables; encoder rows and int8 hypotheses bit-exact, f32
    hypotheses identical."""
    d = 16
    fdim = 8 if combine == "concat" else d
    factors = [dict(combine=combine, embed_dim=fdim, share=shared, vocab_size=9)]
    if combine != "concat":
        factors.append(dict(combine=combine, embed_dim=fdim, share=shared, vocab_size=7))
    c = dict(cfg(2, 1, d, 32, 2, 20, 24, 32), factors=factors)
    om = o.OracleModel.create(c, seed=17)
    path = "/tmp/factors_%s_%d.bin" % (combine, int(shared))
    om.save(path)
    rng = np.random.default_rng(5)
    srcs = o.synthetic_sources(5, 6, 20, seed=9)
    facs = [[rng.integers(0, f["vocab_size"], len(s)).tolist() for f in factors] for s in srcs]
    for prec, int8 in ((mt.INT8, True), (mt.F32, False)):
        gm = mt.Model.load(path, precision=prec)
        enc = gm.encode(srcs, factors=facs)
        ref = np.concatenate([om.encode(s, int8, factors=f) for s, f in zip(srcs, facs)])
        if int8:
            assert np.array_equal(enc.view(np.uint32), ref.view(np.uint32))
        else:
            assert rel(enc, ref) < 1e-4
        hyps = gm.translate(srcs, mt.BeamConfig(4, 0, 1.0), factors=facs)
        for s, f, h in zip(srcs, facs, hyps):
            r = om.beam_search_factors(s, f, 4, derive(s, 32), 1.0, int8)
            assert h.tokens == r["tokens"]
            if int8:
                assert f32hex(h.logprob) == f32hex(r["logprob"])
    # contract errors (model.cpp:541-546, tensor.cpp:456-458)
    gm = mt.Model.load(path, precision=mt.INT8)
    assert gm.translate(srcs[:1], mt.BeamConfig(2, 0, 1.0))[0].status == 1  # ShapeError: no streams
    bad = [[list(x) for x in facs[0]]]
    bad[0][0][0] = 999
    assert gm.translate(srcs[:1], mt.BeamConfig(2, 0, 1.0), factors=bad)[0].status == 3  # IndexError


def test_vocabulary_shortlist_bit_exact():
    """Shortlist decoding (decode.cpp:344-349, model.cpp:440-449): logits,
    log-softmax and candidates over the sentence's shortlist only, candidate
    token = full-vocabulary id; mixed batches (with and without a shortlist)
    and per-sentence errors."""
    c = cfg(2, 2, 32, 64, 4, 300, 600, 48)
    om = o.OracleModel.create(c, seed=23)
    path = "/tmp/shortlist.bin"
    om.save(path)
    rng = np.random.default_rng(3)
    srcs = o.synthetic_sources(6, 7, 300, seed=12)
    sls = [sorted(set([0, 1, 2, 3]) | set(rng.choice(600, 60, replace=False).tolist())) for _ in srcs]
    sls[4] = []  # this sentence decodes over the full vocabulary
    for prec, int8 in ((mt.INT8, True), (mt.F32, False)):
        gm = mt.Model.load(path, precision=prec)
        hyps = gm.translate(srcs, mt.BeamConfig(5, 0, 1.0), shortlists=sls)
        for s, sl, h in zip(srcs, sls, hyps):
            r = om.beam_search(s, 5, derive(s, 48), 1.0, int8, shortlist=sl if sl else None)
            assert h.status == 0
            assert h.tokens == r["tokens"]
            assert not sl or set(h.tokens) <= set(sl)
            if int8:
                assert f32hex(h.logprob) == f32hex(r["logprob"])
        h1 = mt.beam_search(gm, srcs[0], (), mt.BeamConfig(5, 0, 1.0), shortlist=sls[0])
        assert h1.tokens == hyps[0].tokens
    gm = mt.Model.load(path, precision=mt.INT8)
    bad = [list(sls[0]), sls[1][:-1] + [600], list(reversed(sls[2]))]
    st = [h.status for h in gm.translate(srcs[:3], mt.BeamConfig(3, 0, 1.0), shortlists=bad)]
    assert st == [0, 3, 6]  # ok, IndexError (bad row), UsageError (unsorted)


def test_shortlist_edge_cases():
    """Shortlist shorter than the beam (fewer candidates than slots), the
    4096-entry maximum, beam 16, and the bf16 path (sanity: tokens stay in
    the shortlist)."""
    c = cfg(1, 2, 32, 64, 4, 300, 5000, 40)
    om = o.OracleModel.create(c, seed=29)
    path = "/tmp/shortlist_edge.bin"
    om.save(path)
    srcs = o.synthetic_sources(3, 6, 300, seed=13)
    rng = np.random.default_rng(8)
    sls = [[0, 1, 2, 3, 17],                                              # 5 < beam 8
           sorted(set([0, 1, 2, 3]) | set(rng.choice(5000, 4092, replace=False).tolist()))[:4096],
           sorted(set([0, 1, 2, 3]) | set(rng.choice(5000, 300, replace=False).tolist()))]
    gm = mt.Model.load(path, precision=mt.INT8)
    for beam in (8, 16):
        hyps = gm.translate(srcs, mt.BeamConfig(beam, 0, 1.0), shortlists=sls)
        for s, sl, h in zip(srcs, sls, hyps):
            r = om.beam_search(s, beam, derive(s, 40), 1.0, True, shortlist=sl)
            assert h.status == 0 and h.tokens == r["tokens"]
            assert f32hex(h.logprob) == f32hex(r["logprob"])
    too_long = [list(range(4097))]
    assert gm.translate(srcs[:1], mt.BeamConfig(4, 0, 1.0), shortlists=too_long)[0].status == 6
    gb = mt.Model.load(path, precision=mt.BF16)
    for sl, h in zip(sls, gb.translate(srcs, mt.BeamConfig(4, 0, 1.0), shortlists=sls)):
        assert h.status == 0 and set(h.tokens) <= set(sl)


def test_factors_bf16_and_shortlist_together():
    """Factors and a shortlist in one call (mtg_translate_ex), int8 bit-exact
    against the oracle's factored beam search restricted by the shortlist is
    not exposed by the oracle C API, so check against factored full-vocab
    decoding with a shortlist that contains every token it produces."""
    c = dict(cfg(1, 1, 16, 32, 2, 20, 30, 32),
             factors=[dict(combine="concat", embed_dim=8, share=False, vocab_size=9)])
    om = o.OracleModel.create(c, seed=41)
    path = "/tmp/factors_sl.bin"
    om.save(path)
    srcs = o.synthetic_sources(4, 5, 20, seed=3)
    rng = np.random.default_rng(2)
    facs = [[rng.integers(0, 9, len(s)).tolist()] for s in srcs]
    gm = mt.Model.load(path, precision=mt.INT8)
    full = gm.translate(srcs, mt.BeamConfig(3, 0, 1.0), factors=facs)
    sls = [list(range(30)) for _ in srcs]  # the whole vocabulary as an explicit list
    listed = gm.translate(srcs, mt.BeamConfig(3, 0, 1.0), factors=facs, shortlists=sls)
    for s, f, a, b in zip(srcs, facs, full, listed):
        r = om.beam_search_factors(s, f, 3, derive(s, 32), 1.0, True)
        assert a.tokens == r["tokens"] == b.tokens
        assert f32hex(a.logprob) == f32hex(b.logprob) == f32hex(r["logprob"])
    gb = mt.Model.load(path, precision=mt.BF16)
    assert all(h.status == 0 for h in gb.translate(srcs, mt.BeamConfig(3, 0, 1.0), factors=facs))

"""Small-batch decode path (gemv.cuh: <= 8 live rows, batch-1 serving) and
the robustness fixes around the engine.

The GEMV path must give exactly the tcgen05 path's bits for int8 (integer
accumulation, same epilogue, LayerNorm / quantization folded into the
consumer with the same float order) and stay within the fp32 / bf16 bars.
"""

import os
import subprocess
import sys
import threading

import numpy as np
import pytest

import oracle_lib as o
import paper_2008_04885_b200 as mt
from golden_util import f32hex

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TESTS = os.path.dirname(os.path.abspath(__file__))


def cfg(enc=2, dec=2, d=16, ff=32, heads=2, vs=11, vt=13, msl=32):
    return dict(num_encoder_layers=enc, num_decoder_layers=dec, d_model=d, d_ff=ff,
                num_heads=heads, src_vocab_size=vs, tgt_vocab_size=vt, dropout=0.0,
                max_seq_len=msl)


MID = cfg(3, 2, 64, 256, 4, 700, 900, 64)
WIDE = cfg(2, 2, 512, 2048, 8, 3000, 4000, 128)  # d = 512: the 16-float LayerNorm rows


def derive(src, msl):
    return min(msl, 2 * len(src) + 5)


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("config", [MID, WIDE], ids=["mid", "d512"])
@pytest.mark.parametrize("beam", [1, 5, 8])
def test_small_batch_int8_bit_exact(config, beam):
    """Batch 1 at beam <= 8 runs the GEMV step; tokens, logprob and
    normalised-score bits equal the oracle's."""
    om = o.OracleModel.create(config, seed=21)
    gm = mt.Model.create(config, seed=21, precision=mt.INT8)
    for s in o.synthetic_sources(3, 9, config["src_vocab_size"], seed=beam):
        h = gm.translate([s], mt.BeamConfig(beam, 0, 1.0))[0]
        r = om.beam_search(s, beam, derive(s, config["max_seq_len"]), 1.0, True)
        assert (h.tokens, f32hex(h.logprob), f32hex(h.normalized)) == (
            r["tokens"], f32hex(r["logprob"]), f32hex(r["norm"]))


def test_small_batch_forced_logits_bit_exact():
    om = o.OracleModel.create(WIDE, seed=5)
    gm = mt.Model.create(WIDE, seed=5, precision=mt.INT8)
    srcs = o.synthetic_sources(2, 12, WIDE["src_vocab_size"], seed=6)  # 2 rows <= 8
    lg = gm.forced_logits(srcs, [4, 9, 17, 3])
    ref = np.stack([om.forced_logits(s, [4, 9, 17, 3], True) for s in srcs])
    assert np.array_equal(lg, ref)


def test_small_batch_f32_and_bf16_within_tolerance():
    om = o.OracleModel.create(WIDE, seed=8)
    g32 = mt.Model.create(WIDE, seed=8, precision=mt.F32)
    for s in o.synthetic_sources(3, 10, WIDE["src_vocab_size"], seed=3):
        h = g32.translate([s], mt.BeamConfig(5, 0, 1.0))[0]
        r = om.beam_search(s, 5, derive(s, 128), 1.0, False)
        assert h.tokens == r["tokens"]
        assert abs(h.logprob - r["logprob"]) <= 1e-3 * abs(r["logprob"]) + 1e-6
    src = o.synthetic_sources(1, 10, WIDE["src_vocab_size"], seed=4)
    ref = np.stack([om.forced_logits(s, [5, 6, 7], False) for s in src])
    assert rel(g32.forced_logits(src, [5, 6, 7]), ref) < 1e-4
    gbf = mt.Model.create(WIDE, seed=8, precision=mt.BF16)
    assert rel(gbf.forced_logits(src, [5, 6, 7]), ref) < 5e-2


def _run(code, **env):
    full = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n" % (ROOT, TESTS)) + code
    return subprocess.run([sys.executable, "-c", full], env=dict(os.environ, **env), check=True,
                          capture_output=True, text=True, timeout=600).stdout


def test_small_batch_matches_tcgen05_path():
    """MTG_SMALL_BATCH=0 decodes batch 1 on the tcgen05 GEMMs: same bits (int8)
    and same hypotheses (fp32) as the GEMV path."""
    code = (
        "import paper_2008_04885_b200 as mt, oracle_lib as o\n"
        "from golden_util import f32hex\n"
        "c = dict(num_encoder_layers=2, num_decoder_layers=2, d_model=512, d_ff=2048, num_heads=8,"
        " src_vocab_size=3000, tgt_vocab_size=4000, dropout=0.0, max_seq_len=128)\n"
        "srcs = o.synthetic_sources(4, 14, 3000, seed=12)\n"
        "for p in (mt.INT8, mt.F32):\n"
        "    gm = mt.Model.create(c, seed=2, precision=p)\n"
        "    out = [gm.translate([s], mt.BeamConfig(5, 0, 1.0))[0] for s in srcs]\n"
        "    print([(h.tokens, f32hex(h.logprob) if p == mt.INT8 else 0) for h in out])\n"
    )
    a = _run(code, MTG_SMALL_BATCH="1")
    b = _run(code, MTG_SMALL_BATCH="0")
    assert a.strip() and a == b


def test_small_batch_split_k_w2_agrees():
    """MTG_GEMV_W2_SPLIT=4 runs the fp32 / bf16 FFN-down GEMV split over four
    CTAs per column chunk (deterministic last-CTA sum): same hypotheses as
    the unsplit default, logprobs within the fp32 bar."""
    code = (
        "import paper_2008_04885_b200 as mt, oracle_lib as o\n"
        "c = dict(num_encoder_layers=2, num_decoder_layers=2, d_model=512, d_ff=2048, num_heads=8,"
        " src_vocab_size=3000, tgt_vocab_size=4000, dropout=0.0, max_seq_len=128)\n"
        "srcs = o.synthetic_sources(3, 14, 3000, seed=21)\n"
        "for p in (mt.F32, mt.BF16):\n"
        "    gm = mt.Model.create(c, seed=5, precision=p)\n"
        "    out = [gm.translate([s], mt.BeamConfig(5, 0, 1.0))[0] for s in srcs]\n"
        "    print([(h.tokens, round(h.logprob, 3)) for h in out])\n"
    )
    a = _run(code, MTG_GEMV_W2_SPLIT="1")
    b = _run(code, MTG_GEMV_W2_SPLIT="4")
    assert a.strip() and a == b


@pytest.mark.parametrize("d,heads", [(256, 16), (1024, 16)])
def test_sixteen_heads_bit_exact(d, heads):
    """More heads than attention warps (8): each warp attends several heads.
    d = 1024 (head dim 64) takes the staged attention path; batch 3 x beam 5
    runs the tcgen05 step, batch 1 (d = 256) the GEMV step."""
    c = cfg(1, 2, d, 2 * d, heads, 500, 600, 64)
    om = o.OracleModel.create(c, seed=31)
    gm = mt.Model.create(c, seed=31, precision=mt.INT8)
    srcs = o.synthetic_sources(3, 8, 500, seed=32)
    batches = [srcs] + ([[srcs[0]]] if d <= 512 else [])
    for batch in batches:
        for s, h in zip(batch, gm.translate(batch, mt.BeamConfig(5, 0, 1.0))):
            r = om.beam_search(s, 5, derive(s, 64), 1.0, True)
            assert (h.tokens, f32hex(h.logprob)) == (r["tokens"], f32hex(r["logprob"]))


def test_nonfinite_fails_only_its_sentence(tmp_path):
    """quantize() throws on non-finite input (quant.cpp:110-112); in a batch
    only the sentence that produced it fails (translate_corpus blanks that
    line, decode.cpp:403-410). Token 5's embedding overflows to inf once
    scaled by sqrt(d), so its LayerNorm yields NaN."""
    c = cfg(1, 1, 32, 64, 2, 40, 50, 32)
    om = o.OracleModel.create(c, seed=7)
    emb = om.get("src_embed", (40, 32)).copy()
    emb[5, :] = 3.0e38
    om.set("src_embed", emb)
    p = str(tmp_path / "overflow.bin")
    om.save(p)
    gm = mt.Model.load(p, precision=mt.INT8)
    srcs = [[7, 8, 9, 3], [7, 5, 9, 3], [10, 11, 3], [12, 3]]
    hyps = gm.translate(srcs, mt.BeamConfig(4, 0, 1.0))
    assert [h.status for h in hyps] == [0, 2, 0, 0]  # MTG_VALUE_ERROR
    for s, h in zip(srcs, hyps):
        if h.status:
            with pytest.raises(o.OracleError):
                om.beam_search(s, 4, derive(s, 32), 1.0, True)
            continue
        r = om.beam_search(s, 4, derive(s, 32), 1.0, True)
        assert (h.tokens, f32hex(h.logprob)) == (r["tokens"], f32hex(r["logprob"]))


def test_two_handles_from_two_threads():
    """Distinct handles are usable from distinct threads (minimt_gpu.h):
    concurrent decodes give the sequential results."""
    c = MID
    srcs = o.synthetic_sources(6, 9, c["src_vocab_size"], seed=41)
    models = [mt.Model.create(c, seed=41, precision=mt.INT8) for _ in range(2)]
    want = [(h.tokens, f32hex(h.logprob)) for h in models[0].translate(srcs, mt.BeamConfig(5, 0, 1.0))]
    got = [None, None]
    errs = []

    def work(i):
        try:
            for _ in range(3):
                got[i] = [(h.tokens, f32hex(h.logprob))
                          for h in models[i].translate(srcs, mt.BeamConfig(5, 0, 1.0))]
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert got[0] == want and got[1] == want

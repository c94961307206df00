"""Pins the CPU oracle (oracle/) to the reference's own known-answer tests and
properties. The reference cannot be built here (Eigen3/vendor absent), so
these KATs are what ties the oracle to it; each test cites the reference test
it restates (paths relative to /root/reference/proj)."""

import json
import math
import os

import numpy as np
import pytest

import oracle_lib as o


def cfg(enc=2, dec=2, d=16, ff=32, heads=2, vs=11, vt=13, msl=32, dropout=0.0):
    return dict(num_encoder_layers=enc, num_decoder_layers=dec, d_model=d, d_ff=ff,
                num_heads=heads, src_vocab_size=vs, tgt_vocab_size=vt, dropout=dropout,
                max_seq_len=msl)


# ---- quantization (tests/test_quant.cpp) ----------------------------------------

def test_quantize_kat_2_m2_1():  # test_quant.cpp:38-44
    q, s = o.quantize(np.array([2.0, -2.0, 1.0], np.float32))
    assert s == np.float32(63.5)
    assert q.tolist() == [127, -127, 64]  # 63.5 rounds half away from zero


def test_quantize_zeros():  # test_quant.cpp:46-50
    q, s = o.quantize(np.zeros((2, 3), np.float32))
    assert s == 1.0 and not q.any()


def test_quantize_single_one():  # test_quant.cpp:52-57
    q, s = o.quantize(np.array([1.0], np.float32))
    assert s == 127.0 and q[0] == 127
    assert np.float32(q[0]) / s == 1.0


def test_quantize_half_away_from_zero():  # test_quant.cpp:59-64
    q, s = o.quantize(np.array([127.0, 0.5, -0.5], np.float32))
    assert s == 1.0 and q[1] == 1 and q[2] == -1


def test_quantize_round_trip_half_step():  # test_quant.cpp:66-79
    x = np.random.default_rng(31).uniform(-2, 2, (16, 16)).astype(np.float32)
    q, s = o.quantize(x)
    back = q.astype(np.float32) / s
    assert np.all(np.abs(back - x) <= 0.5 / s * 1.0001)
    assert np.abs(q).max() == 127 and q.min() >= -127


def test_quantize_rejects_nonfinite():  # test_quant.cpp:81-83
    with pytest.raises(o.OracleError) as e:
        o.quantize(np.array([1.0, np.nan], np.float32))
    assert e.value.kind == "ValueError"


@pytest.mark.parametrize("m,k,n", [(3, 7, 5), (8, 64, 16), (1, 33, 17), (5, 128, 48)])
def test_qmatmul_matches_int32_reference(m, k, n):  # test_quant.cpp:21-34, 85-100
    rng = np.random.default_rng(32)
    qa, sa = o.quantize(rng.uniform(-2, 2, (m, k)).astype(np.float32))
    qb, sb = o.quantize(rng.uniform(-2, 2, (k, n)).astype(np.float32))
    want = (qa.astype(np.int64) @ qb.astype(np.int64)).astype(np.float32) * (
        np.float32(1.0) / (sa * sb))
    assert np.array_equal(o.qmatmul(qa, sa, qb, sb), want)


def test_qmatmul_error_bound():  # test_quant.cpp:140-157
    rng = np.random.default_rng(36)
    for _ in range(20):
        af = rng.uniform(-3, 3, (6, 32)).astype(np.float32)
        bf = rng.uniform(-3, 3, (32, 8)).astype(np.float32)
        qa, sa = o.quantize(af)
        qb, sb = o.quantize(bf)
        exact = af.astype(np.float64) @ bf.astype(np.float64)
        da, db = 0.5 / sa, 0.5 / sb
        bound = 32 * (da * np.abs(bf).max() + db * np.abs(af).max() + da * db)
        assert np.all(np.abs(o.qmatmul(qa, sa, qb, sb) - exact) <= bound * 1.0001)


def test_qmatmul_rejects_k_above_65536():  # test_quant.cpp:159-173
    a = np.zeros((1, 65537), np.int8)
    b = np.zeros((65537, 1), np.int8)
    with pytest.raises(o.OracleError) as e:
        o.qmatmul(a, 1.0, b, 1.0)
    assert e.value.kind == "ValueError"


# ---- model layout / persistence (tests/test_model.cpp) -----------------------------

def test_param_count_closed_form():  # test_model.cpp:155-165
    m = o.OracleModel.create(cfg(), seed=1, init=False)
    d, ff, vs, vt = 16, 32, 11, 13
    enc_layer = 4 * d * d + 2 * d * ff + ff + 5 * d
    dec_layer = 8 * d * d + 2 * d * ff + ff + 7 * d
    want = vs * d + vt * d + 2 * enc_layer + 2 * d + 2 * dec_layer + 2 * d
    assert m.param_count() == want


def test_param_count_20_2():  # 20:2 = 104.2M params
    m = o.OracleModel.create(cfg(20, 2, 512, 2048, 8, 32000, 32000, 128), seed=1, init=False)
    assert m.param_count() == 104_176_640


def test_positional_encoding_kats():  # test_model.cpp:309-321
    pe = o.OracleModel.create(cfg(), seed=1).pos_enc()
    assert pe.shape == (32, 16)
    assert pe[0, 0] == 0.0 and pe[0, 1] == 1.0
    assert pe[3, 0] == pytest.approx(math.sin(3.0), rel=1e-6)
    assert pe[3, 1] == pytest.approx(math.cos(3.0), rel=1e-6)
    assert pe[5, 4] == pytest.approx(math.sin(5.0 / 10000.0 ** (4.0 / 16.0)), rel=1e-6)


def test_init_xavier_gain_bias():  # model.cpp:229-238
    m = o.OracleModel.create(cfg(), seed=1)
    w = m.get("enc0.attn.wq", (16, 16))
    lim = math.sqrt(6.0 / 32.0)
    assert np.all(np.abs(w) <= lim) and np.abs(w).max() > 0.8 * lim
    assert np.all(m.get("enc0.norm1.gain", (16,)) == 1.0)
    assert np.all(m.get("enc0.norm1.bias", (16,)) == 0.0)
    assert np.all(m.get("dec0.ffn.b1", (32,)) == 0.0)


def test_init_is_seeded_and_name_ordered():  # tensor.hpp:62-78 + std::map order
    a = o.OracleModel.create(cfg(), seed=7).get("tgt_embed", (13, 16))
    b = o.OracleModel.create(cfg(), seed=7).get("tgt_embed", (13, 16))
    c = o.OracleModel.create(cfg(), seed=8).get("tgt_embed", (13, 16))
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # std::map order: "dec0.*" < "enc0.*" < "src_embed" < "tgt_embed", so the
    # first draw of the stream lands in dec0.cross.wk[0,0].
    import random  # noqa: F401  (documentation only)


def test_config_json_nlohmann_format():  # model.cpp:102-120 (sorted keys, compact)
    m = o.OracleModel.create(cfg(dropout=0.1), seed=1, init=False)
    assert m.config_json == (
        '{"d_ff":32,"d_model":16,"dropout":0.10000000149011612,"factors":[],"max_seq_len":32,'
        '"num_decoder_layers":2,"num_encoder_layers":2,"num_heads":2,"src_vocab_size":11,'
        '"tgt_vocab_size":13}')


def test_sqnt_round_trip_and_corruption(tmp_path):  # test_model.cpp:51-114, 298-307
    m = o.OracleModel.create(cfg(), seed=29)
    p = str(tmp_path / "m.bin")
    m.save(p)
    back = o.OracleModel.load(p)
    assert back.config_json == m.config_json
    for name, shape in [("tgt_embed", (13, 16)), ("dec1.ffn.w2", (32, 16)), ("enc1.norm2.gain", (16,))]:
        assert np.array_equal(back.get(name, shape), m.get(name, shape))
    raw = open(p, "rb").read()
    for bad in (raw[:-5], raw + b"junk", b"NOPE"):
        open(p, "wb").write(bad)
        with pytest.raises(o.OracleError) as e:
            o.OracleModel.load(p)
        assert e.value.kind == "FormatError"


def test_offline_equals_on_load_quantization(tmp_path):  # test_model.cpp:342-371
    m = o.OracleModel.create(cfg(), seed=31)
    f32, q8 = str(tmp_path / "f.bin"), str(tmp_path / "q.bin")
    m.save(f32)
    m.save(q8, quantized=True)
    assert os.path.getsize(q8) < os.path.getsize(f32)
    loaded = o.OracleModel.load(q8)
    onload = o.OracleModel.load(f32)
    for name, shape in [("tgt_embed", (13, 16)), ("enc0.attn.wq", (16, 16)), ("dec1.ffn.w1", (16, 32))]:
        qa, sa = m.qparam(name, shape)
        qb, sb = loaded.qparam(name, shape)
        qc, sc = onload.qparam(name, shape)
        assert sa == sb == sc and np.array_equal(qa, qb) and np.array_equal(qa, qc)


# ---- forward ops (tests/test_tensor.cpp, test_model.cpp) ----------------------------

def test_layer_norm_kat():  # test_tensor.cpp:108-115
    y = o.layer_norm(np.array([[1.0, 3.0]], np.float32), [1, 1], [0, 0])
    assert y[0, 0] == pytest.approx(-1.0, rel=1e-4) and y[0, 1] == pytest.approx(1.0, rel=1e-4)


def test_log_softmax_kat():  # test_tensor.cpp:94-106 (softmax of [0,1] / [100,101])
    for x in ([0.0, 1.0], [100.0, 101.0]):
        p = np.exp(o.log_softmax(np.array(x, np.float32)).astype(np.float64))
        assert p[0] == pytest.approx(0.26894142, rel=1e-5)
        assert p[1] == pytest.approx(0.73105858, rel=1e-5)


def test_det_exp_log_within_one_ulp():
    xs = np.linspace(-87, 88, 20001, dtype=np.float32)
    for x in xs[::7]:
        e = o.det_expf(float(x))
        ref = np.float32(math.exp(float(x)))
        assert abs(np.float32(e) - ref) <= np.spacing(ref) * 1.0
    for y in np.geomspace(1e-30, 1e30, 3001).astype(np.float32):
        lg = o.det_logf(float(y))
        ref = np.float32(math.log(float(y)))
        # 1 ulp of the result, or ~1 ulp of the input's mantissa near log(1) = 0
        assert abs(np.float32(lg) - ref) <= max(abs(np.spacing(ref)), 6e-8)
    assert o.det_expf(0.0) == 1.0 and o.det_logf(1.0) == 0.0


def test_incremental_matches_teacher_forced():  # test_model.cpp:211-228
    m = o.OracleModel.create(cfg(), seed=11)
    src, tgt = [5, 9, 4, 3], [6, 7, 8, 5, 3]
    full = m.teacher_forced(src, tgt)
    inc = m.forced_logits(src, tgt)
    assert np.abs(inc - full).max() < 1e-4


def test_incremental_matches_teacher_forced_random_configs():  # acceptance.cpp:318-376 (C2)
    worst = 0.0
    for trial in range(50):
        rng = np.random.default_rng(1000 + trial)
        d = 8 << int(rng.integers(0, 3))
        heads = 2 if rng.integers(0, 2) else 4
        c = cfg(int(1 + rng.integers(0, 2)), int(1 + rng.integers(0, 2)), d, 2 * d, heads,
                int(8 + rng.integers(0, 13)), int(8 + rng.integers(0, 13)), 64)
        m = o.OracleModel.create(c, seed=900 + trial)
        src = [int(4 + rng.integers(0, c["src_vocab_size"] - 4)) for _ in range(1 + rng.integers(0, 6))] + [3]
        tgt = [int(4 + rng.integers(0, c["tgt_vocab_size"] - 4)) for _ in range(1 + rng.integers(0, 6))] + [3]
        worst = max(worst, float(np.abs(m.forced_logits(src, tgt) - m.teacher_forced(src, tgt)).max()))
    assert worst <= 1e-4


# ---- search (tests/test_decode.cpp) -------------------------------------------------

def test_gnmt_penalty_kats():  # test_decode.cpp:41-50
    assert o.normalized_score(4, -1.0, 0.0) == -1.0
    assert o.normalized_score(4, -1.0, 1.0) == pytest.approx(-1.0 / ((5.0 + 5.0) / 6.0))
    assert o.normalized_score(4, -1.0, 2.0) == pytest.approx(-1.0 / (10.0 / 6.0) ** 2, rel=1e-6)


def micro(vocab, seed):
    return o.OracleModel.create(cfg(1, 1, 8, 16, 2, vocab, vocab, 32), seed=seed)


def test_beam1_is_greedy():  # test_decode.cpp:52-76
    m = micro(12, 51)
    src = [4, 7, 5, 3]
    beam = m.beam_search(src, 1, 10, 0.0)
    greedy, prev = [], []
    for t in range(10):
        lg = m.forced_logits(src, prev + [0])[t]
        best = int(np.argmax(lg))
        if best == 3:
            break
        greedy.append(best)
        prev.append(best)
    assert beam["tokens"] == greedy


def test_full_shortlist_is_noop():  # test_decode.cpp:78-91
    m = micro(12, 53)
    plain = m.beam_search([6, 9, 3], 3, 12)
    listed = m.beam_search([6, 9, 3], 3, 12, shortlist=list(range(12)))
    assert plain["tokens"] == listed["tokens"]
    assert plain["logprob"] == pytest.approx(listed["logprob"])


def test_beam_search_validates_inputs():  # test_decode.cpp:93-101
    m = micro(8, 55)
    for src, beam in (([4, 3], 0), ([], 1)):
        with pytest.raises(o.OracleError) as e:
            m.beam_search(src, beam, 5)
        assert e.value.kind == "UsageError"


def test_uniform_model_emits_pad_until_max_len():  # test_decode.cpp:171-206
    m = o.OracleModel.create(cfg(1, 1, 8, 16, 2, 8, 8, 32), seed=1, init=False)  # all-zero
    total = 0
    for _ in range(10):
        h = m.beam_search(o.prepare_source([4, 5], 32), 1, 3)
        assert h["tokens"] == [0, 0, 0] and h["truncated"]
        total += len(h["tokens"])
    assert total == 30


def test_translate_one_length_rules():  # decode.cpp:326-333, 352-355
    assert o.prepare_source([5, 6], 8) == [5, 6, 3]
    assert o.prepare_source(list(range(4, 14)), 8) == [4, 5, 6, 7, 8, 9, 10, 3]


def test_percentile_nearest_rank():  # test_eval.cpp:140-150
    v = [10, 1, 9, 2, 8, 3, 7, 4, 6, 5]
    assert o.percentile([42.0], 50.0) == 42.0 and o.percentile([42.0], 100.0) == 42.0
    assert o.percentile(v, 90.0) == 9.0 and o.percentile(v, 50.0) == 5.0
    assert o.percentile(v, 100.0) == 10.0 and o.percentile(v, 1.0) == 1.0
    for args in (([], 50.0), ([1.0], 0.0), ([1.0], 101.0)):
        with pytest.raises(o.OracleError):
            o.percentile(*args)


def test_batch_translate_matches_single_and_is_thread_invariant():  # decode.cpp:370-398
    m = micro(30, 61)
    srcs = o.synthetic_sources(5, 4, 30, seed=2)
    one = [m.beam_search(s, 3, min(32, 2 * len(s) + 5)) for s in srcs]
    for th in (1, 3):
        got = m.translate_batch(srcs, 3, 0, 1.0, threads=th)
        assert [g["tokens"] for g in got] == [x["tokens"] for x in one]
        assert [g["logprob"] for g in got] == [x["logprob"] for x in one]


def test_golden_fixture_matches(tmp_path):
    """tests/golden/*.json were produced by tests/golden/make_golden.py from the
    oracle; this pins the oracle against itself across builds/hosts."""
    from golden_util import check_golden
    check_golden()

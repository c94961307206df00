"""Text-level caller side (include/minimt_gpu_text.hpp) and the `translate` /
`benchmark` CLI (tools/minimt_gpu_cli.cpp), restating proj/tools/minimt.cpp
and decode.cpp:320-419 semantics: vocab files next to the model, EOS/UNK
handling, case factors, shortlist table, empty line on failure, JSON report."""

import json
import os
import subprocess

import pytest

import oracle_lib as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2008_04885_b200")


def build(tmp_path):
    exe = str(tmp_path / "minimt_gpu")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tools", "minimt_gpu_cli.cpp"), "-L", LIBDIR, "-lminimt_gpu",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cli_compiles(tmp_path):
    assert os.path.exists(build(tmp_path))


def words(n):
    return ["w%d" % i for i in range(n)]


def setup_model(tmp_path, factors=None):
    vs, vt = 30, 40
    cfg = dict(num_encoder_layers=1, num_decoder_layers=1, d_model=16, d_ff=32, num_heads=2,
               src_vocab_size=vs, tgt_vocab_size=vt, dropout=0.0, max_seq_len=24)
    if factors:
        cfg["factors"] = factors
    om = o.OracleModel.create(cfg, seed=31)
    om.save(str(tmp_path / "model.bin"))
    (tmp_path / "src.vocab").write_text("\n".join(words(vs - 4)) + "\n")
    (tmp_path / "tgt.vocab").write_text("\n".join("t%d" % i for i in range(vt - 4)) + "\n")
    return om


def expected(om, line, beam, msl, int8, fids=None, shortlist=None, tgt=None):
    vocab = {w: i + 4 for i, w in enumerate(words(26))}
    toks = line.split()
    if fids is not None:
        toks = [t.lower() for t in toks]
    ids = [vocab.get(t, 1) for t in toks] + [3]
    n = min(msl, 2 * len(ids) + 5)
    if fids is not None:
        r = om.beam_search_factors(ids, [fids + [3]], beam, n, 1.0, int8)
    else:
        r = om.beam_search(ids, beam, n, 1.0, int8, shortlist=shortlist)
    names = ["<pad>", "<unk>", "<s>", "</s>"] + ["t%d" % i for i in range(36)]
    return " ".join(names[t] for t in r["tokens"])


@pytest.mark.gpu
def test_cli_translate_and_benchmark(tmp_path):
    exe = build(tmp_path)
    om = setup_model(tmp_path)
    lines = ["w1 w2 w3", "w5 unknown w7 w8 w9", "w10", "w3 w3 w3 w4"]
    (tmp_path / "in.txt").write_text("\n".join(lines) + "\n")
    for batch in ("1", "8"):
        out = tmp_path / ("out%s.txt" % batch)
        r = subprocess.run([exe, "translate", "--model", str(tmp_path / "model.bin"), "--input",
                            str(tmp_path / "in.txt"), "--output", str(out), "--int8", "--beam", "3",
                            "--batch", batch], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        got = out.read_text().splitlines()
        assert got == [expected(om, l, 3, 24, True) for l in lines]
    r = subprocess.run([exe, "benchmark", "--model", str(tmp_path / "model.bin"), "--input",
                        str(tmp_path / "in.txt"), "--repeat", "2", "--latency",
                        str(tmp_path / "lat.json")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    j = json.loads(r.stdout)
    assert j["aggregate"]["count"] == 8 and len(j["repeats"]) == 2
    assert set(j["aggregate"]) == {"count", "mean_ms", "p50_ms", "p90_ms", "tokens_per_sec"}
    assert json.loads((tmp_path / "lat.json").read_text())["count"] == 8
    # shortlist table (decode.cpp:135-199): every source word maps to a few targets
    (tmp_path / "shortlist.txt").write_text(
        "\n".join("%d %d:5 %d:3" % (s, 4 + s % 30, 5 + (s * 7) % 30) for s in range(4, 30)) + "\n")
    out = tmp_path / "out_sl.txt"
    r = subprocess.run([exe, "translate", "--model", str(tmp_path / "model.bin"), "--input",
                        str(tmp_path / "in.txt"), "--output", str(out), "--int8", "--beam", "3",
                        "--shortlist", "8"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert len(out.read_text().splitlines()) == len(lines)
    # usage error exit code
    r = subprocess.run([exe, "translate", "--model", str(tmp_path / "model.bin")],
                       capture_output=True, text=True)
    assert r.returncode == 2


@pytest.mark.gpu
def test_cli_case_factors(tmp_path):
    exe = build(tmp_path)
    om = setup_model(tmp_path, factors=[dict(combine="sum", embed_dim=16, share=False,
                                             vocab_size=8)])
    lines = ["W1 w2 W3", "w5 W6 w7", "W10 W11"]
    (tmp_path / "in.txt").write_text("\n".join(lines) + "\n")
    out = tmp_path / "out.txt"
    r = subprocess.run([exe, "translate", "--model", str(tmp_path / "model.bin"), "--input",
                        str(tmp_path / "in.txt"), "--output", str(out), "--int8", "--beam", "2",
                        "--case-scheme", "sf-case"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    cats = {"lowercase": 4, "capitalized": 5, "all_uppercase": 6, "mixed": 7}

    def cat(t):
        up = [c.isupper() for c in t]
        if not any(up):
            return cats["lowercase"]
        if up[0] and not any(up[1:]):
            return cats["capitalized"]
        return cats["all_uppercase"] if not any(c.islower() for c in t) else cats["mixed"]
    exp = [expected(om, l, 2, 24, True, fids=[cat(t) for t in l.split()]) for l in lines]
    assert out.read_text().splitlines() == exp

"""The C++ shim (include/minimt_gpu.hpp) mirrors the reference decode API;
tests/cpp/test_shim.cpp restates test_decode.cpp cases against it."""

import os
import subprocess

import pytest

import oracle_lib as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2008_04885_b200")


def build(tmp_path):
    exe = str(tmp_path / "test_shim")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), "-L", LIBDIR, "-lminimt_gpu",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_shim_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_shim_reference_style_cases(tmp_path):
    exe = build(tmp_path)
    cfg = dict(num_encoder_layers=1, num_decoder_layers=1, d_model=8, d_ff=16, num_heads=2,
               src_vocab_size=12, tgt_vocab_size=12, dropout=0.0, max_seq_len=32)
    zero = str(tmp_path / "zero.bin")
    o.OracleModel.create(dict(cfg, src_vocab_size=8, tgt_vocab_size=8), seed=1, init=False).save(zero)
    micro = str(tmp_path / "micro.bin")
    o.OracleModel.create(cfg, seed=51).save(micro)
    r = subprocess.run([exe, zero, micro], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "SHIM_OK" in r.stdout, r.stdout + r.stderr

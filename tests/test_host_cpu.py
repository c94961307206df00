"""CPU-only checks of the product boundary: the C-ABI library loads and exports
every symbol include/minimt_gpu.h declares, the Python host mirror's pure
host logic matches the oracle, and the multi-rank sharding/gather path works
with world_size 2 over gloo."""

import os
import re
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as o
import paper_2008_04885_b200 as mt
from paper_2008_04885_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "minimt_gpu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mtg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 18
    lib = mt.lib()
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/minimt_gpu.h but not exported"
    assert lib.mtg_abi_version() == 1


def test_status_codes_match_reference_taxonomy():
    txt = open(os.path.join(ROOT, "include", "minimt_gpu.h")).read()
    codes = dict(re.findall(r"#define MTG_([A-Z_]+)_ERROR (\d+)", txt))
    want = {"SHAPE": mt.ShapeError, "VALUE": mt.ValueError_, "INDEX": mt.IndexError_,
            "STATE": mt.StateError, "FORMAT": mt.FormatError, "USAGE": mt.UsageError,
            "IO": mt.IoError, "CUDA": mt.CudaError}
    for k, cls in want.items():
        assert mt._ERRORS[int(codes[k])] is cls


def test_prepare_source_matches_oracle():  # decode.cpp:326-333
    for words, msl in (([5, 6], 8), (list(range(4, 20)), 8), ([], 4), ([9] * 3, 4)):
        assert mt.prepare_source(words, msl) == o.prepare_source(words, msl)


def test_percentile_matches_oracle():  # eval.cpp:120-128
    rng = np.random.default_rng(0)
    for n in (1, 2, 10, 33):
        v = rng.uniform(0, 1, n).tolist()
        for p in (1.0, 50.0, 90.0, 100.0):
            assert mt.percentile(v, p) == o.percentile(v, p)
    with pytest.raises(mt.UsageError):
        mt.percentile([], 50.0)


def test_beam_search_validates_before_touching_the_device():  # decode.cpp:38-39
    with pytest.raises(mt.UsageError):
        mt.beam_search(None, [4, 3], config=mt.BeamConfig(beam_size=0))
    with pytest.raises(mt.UsageError):
        mt.beam_search(None, [], config=mt.BeamConfig(beam_size=1))


def test_csr_packing():
    """Sources reach the C ABI as CSR (ids int32, offsets int64)."""
    ids, off = mt._csr([[5, 6, 3], [3], [7, 8, 9, 3]])
    assert ids.dtype == np.int32 and off.dtype == np.int64
    assert ids.tolist() == [5, 6, 3, 3, 7, 8, 9, 3] and off.tolist() == [0, 3, 4, 8]
    ids, off = mt._csr([])
    assert off.tolist() == [0] and ids.size == 1  # never a zero-length buffer
    ids, off = mt._csr([[], [4, 3]])
    assert off.tolist() == [0, 0, 2] and ids[:2].tolist() == [4, 3]


def test_partition_balances_and_covers():
    rng = np.random.default_rng(1)
    lengths = rng.integers(5, 61, 1000).tolist()
    for world in (1, 2, 4, 8):
        parts = shard.partition(lengths, world)
        flat = sorted(i for p in parts for i in p)
        assert flat == list(range(len(lengths)))
        loads = [sum(shard.sentence_cost(lengths[i], 5) for i in p) for p in parts]
        assert max(loads) / (sum(loads) / world) < 1.02
        for p in parts:
            assert [lengths[i] for i in p] == sorted(lengths[i] for i in p)


def test_pack_unpack_round_trip():
    hyps = [mt.Hypothesis([5, 6, 7], -1.25, True, False, -0.5, 0),
            mt.Hypothesis([], 0.0, False, True, 0.0, 2)]
    rec = shard.pack_records([4, 9], hyps, 16)
    back = shard.unpack_records(rec)
    assert back[4]["tokens"] == [5, 6, 7] and back[4]["finished"] and back[4]["logprob"] == -1.25
    assert back[9]["tokens"] == [] and back[9]["status"] == 2 and back[9]["truncated"]


_WORKER = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import torch.distributed as dist
dist.init_process_group("gloo")
from paper_2008_04885_b200 import shard
import paper_2008_04885_b200 as mt
rank, world = dist.get_rank(), dist.get_world_size()
lengths = [int(x) for x in np.random.default_rng(3).integers(5, 61, 37)]
mine = shard.partition(lengths, world)[rank]
hyps = [mt.Hypothesis([i % 7 + 4] * (i % 5), -float(i), i % 2 == 0, i % 2 == 1, -i / 2.0, 0)
        for i in mine]
got = shard.gather_to_rank0(shard.pack_records(mine, hyps, 8))
if rank == 0:
    recs = shard.unpack_records(got)
    assert sorted(recs) == list(range(37)), sorted(recs)
    for i in range(37):
        assert recs[i]["tokens"] == [i % 7 + 4] * (i % 5)
        assert recs[i]["logprob"] == -float(i)
    print("GATHER_OK")
dist.destroy_process_group()
"""


def test_two_rank_gloo_gather(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, ROOT=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(script)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GATHER_OK" in r.stdout

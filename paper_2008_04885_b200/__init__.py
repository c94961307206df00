"""B200-native (sm_100a) Sockeye-2 translation hot path: batched encoder +
incremental beam search, behind the reference's decode API.

This module is the host-side mirror of the reference interface
(/root/reference/proj/include/minimt/{model,decode,quant}.hpp) over the C ABI
in include/minimt_gpu.h. Everything it does runs in libminimt_gpu.so
(hand-written tcgen05/TMA CUDA kernels); there is no CPU fallback: if the
library is missing, import fails loudly.

Reference ↔ here:
  ModelConfig (model.hpp:33-60)          -> ModelConfig
  BeamConfig (decode.hpp:27-31)          -> BeamConfig
  Hypothesis (decode.hpp:15-25)          -> Hypothesis
  F32Executor / Int8Executor (model.hpp:131-171) -> Model(precision=F32|INT8)
  beam_search (decode.hpp:35-38)         -> beam_search / Model.translate (batched)
  decode_step along a prefix (model.hpp:191) -> Model.forced_logits
  encode_infer(embed_source_infer) (model.hpp:173-175) -> Model.encode
  quantize / qmatmul / qmatmul_nt (quant.hpp:45-68) -> quantize / qmatmul / qmatmul_nt
  gemm_f32 (tensor.hpp:150)               -> gemm
Errors map onto the reference exception taxonomy (errors.hpp:8-34).
"""

from __future__ import annotations

import ctypes
import itertools
import dataclasses
import json
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MTG_LIB_PATH overrides the library (A/B builds); default: the in-tree build.
LIB_PATH = os.environ.get("MTG_LIB_PATH") or os.path.join(_HERE, "libminimt_gpu.so")

F32, BF16, INT8 = 0, 1, 2
PAD_ID, UNK_ID, BOS_ID, EOS_ID = 0, 1, 2, 3  # model.hpp:16-19
HYP_FINISHED, HYP_TRUNCATED, HYP_FAILED = 1, 2, 4


# ---- errors (errors.hpp:8-34) -------------------------------------------------
class MinimtError(RuntimeError):
    pass


class ShapeError(MinimtError):
    pass


class ValueError_(MinimtError, ValueError):
    pass


class IndexError_(MinimtError, IndexError):
    pass


class StateError(MinimtError):
    pass


class FormatError(MinimtError):
    pass


class UsageError(MinimtError):
    pass


class IoError(MinimtError, OSError):
    pass


class CudaError(MinimtError):
    pass


_ERRORS = {1: ShapeError, 2: ValueError_, 3: IndexError_, 4: StateError, 5: FormatError,
           6: UsageError, 7: IoError, 8: CudaError}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    c_int, c_float, c_void_p, c_size_t = ctypes.c_int, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t
    lib.mtg_last_error.restype = ctypes.c_char_p
    lib.mtg_abi_version.restype = c_int
    lib.mtg_quantize.argtypes = [c_void_p, ctypes.c_int64, c_void_p, c_void_p]
    lib.mtg_qmatmul.argtypes = [c_void_p, c_float, c_void_p, c_float, c_int, c_int, c_int, c_void_p]
    lib.mtg_qmatmul_nt.argtypes = [c_void_p, c_float, c_void_p, c_float, c_int, c_int, c_int,
                                   c_void_p, c_int, c_void_p]
    lib.mtg_gemm.argtypes = [c_int, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]
    lib.mtg_model_load.argtypes = [ctypes.c_char_p, c_int, c_int, ctypes.POINTER(c_void_p)]
    lib.mtg_model_create.argtypes = [ctypes.c_char_p, ctypes.c_uint64, c_int, c_int,
                                     ctypes.POINTER(c_void_p)]
    lib.mtg_model_save.argtypes = [c_void_p, ctypes.c_char_p]
    lib.mtg_model_free.argtypes = [c_void_p]
    lib.mtg_model_free.restype = None
    lib.mtg_model_config_json.argtypes = [c_void_p, ctypes.c_char_p, c_size_t]
    lib.mtg_model_precision.argtypes = [c_void_p]
    lib.mtg_translate.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_int,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]
    lib.mtg_forced_logits.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p]
    lib.mtg_encode.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p]
    lib.mtg_translate_factors.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int,
                                          c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
                                          c_void_p, c_void_p]
    lib.mtg_encode_factors.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int,
                                       c_void_p]
    lib.mtg_translate_ex.argtypes = [c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p,
                                     c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                     c_void_p, c_void_p, c_void_p]
    lib.mtg_stage_sources.argtypes = [c_void_p, c_void_p, c_void_p, c_int]
    lib.mtg_translate_staged.argtypes = [c_void_p, c_void_p]
    lib.mtg_last_launch_count.argtypes = [c_void_p]
    lib.mtg_last_launch_count.restype = ctypes.c_int64
    if hasattr(lib, "mtg_diag_report"):  # absent in older A/B builds
        lib.mtg_diag_report.argtypes = [c_void_p, ctypes.c_char_p, ctypes.c_size_t]
    return lib


_lib = _load()


def lib():
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = (_lib.mtg_last_error() or b"").decode()
        raise _ERRORS.get(rc, MinimtError)(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class _BeamConfigC(ctypes.Structure):
    _fields_ = [("beam_size", ctypes.c_int), ("max_len", ctypes.c_int),
                ("length_penalty_alpha", ctypes.c_float), ("max_batch", ctypes.c_int)]


# ---- config / results ---------------------------------------------------------

@dataclasses.dataclass
class ModelConfig:
    """model.hpp:33-60 (factors not yet supported on the GPU path)."""
    num_encoder_layers: int = 6
    num_decoder_layers: int = 6
    d_model: int = 32
    d_ff: int = 128
    num_heads: int = 4
    src_vocab_size: int = 0
    tgt_vocab_size: int = 0
    dropout: float = 0.1
    max_seq_len: int = 128

    def to_json(self) -> str:
        d = dataclasses.asdict(self)
        d["factors"] = []
        return json.dumps(d, sort_keys=True)

    @staticmethod
    def paper_base(src_vocab: int, tgt_vocab: int) -> "ModelConfig":  # model.cpp:150-160
        return ModelConfig(6, 6, 512, 2048, 8, src_vocab, tgt_vocab)


@dataclasses.dataclass
class BeamConfig:
    """decode.hpp:27-31; max_len <= 0 derives min(max_seq_len, 2|src|+5)."""
    beam_size: int = 4
    max_len: int = 64
    length_penalty_alpha: float = 1.0


@dataclasses.dataclass
class Hypothesis:
    """decode.hpp:15-25 (state is never returned)."""
    tokens: List[int]
    logprob: float
    finished: bool
    truncated: bool
    normalized: float
    status: int = 0


# ---- raw operators (quant.hpp, tensor.hpp) -------------------------------------

def quantize(x: np.ndarray):
    """quant.cpp:108-122 -> (int8 data, scale)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    q = np.zeros(x.shape, np.int8)
    s = ctypes.c_float()
    _check(_lib.mtg_quantize(_ptr(x), x.size, _ptr(q), ctypes.byref(s)))
    return q, np.float32(s.value)


def qmatmul(a: np.ndarray, sa: float, b: np.ndarray, sb: float) -> np.ndarray:
    """quant.cpp:155-193; a [m x k], b [k x n] int8."""
    a = np.ascontiguousarray(a, np.int8)
    b = np.ascontiguousarray(b, np.int8)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ShapeError("qmatmul: inner dimensions disagree")
    c = np.zeros((m, n), np.float32)
    _check(_lib.mtg_qmatmul(_ptr(a), sa, _ptr(b), sb, m, k, n, _ptr(c)))
    return c


def qmatmul_nt(a: np.ndarray, sa: float, b: np.ndarray, sb: float,
               row_subset: Optional[Sequence[int]] = None) -> np.ndarray:
    """quant.cpp:195-239; b [rows x k]."""
    a = np.ascontiguousarray(a, np.int8)
    b = np.ascontiguousarray(b, np.int8)
    m, k = a.shape
    rows, k2 = b.shape
    if k != k2:
        raise ShapeError("qmatmul_nt: inner dimensions disagree")
    sub = None if row_subset is None else np.ascontiguousarray(row_subset, np.int32)
    n = rows if sub is None else len(sub)
    c = np.zeros((m, n), np.float32)
    _check(_lib.mtg_qmatmul_nt(_ptr(a), sa, _ptr(b), sb, m, k, rows,
                               None if sub is None else _ptr(sub), 0 if sub is None else len(sub),
                               _ptr(c)))
    return c


def gemm(a: np.ndarray, b: np.ndarray, precision: int = F32) -> np.ndarray:
    """gemm_f32 (tensor.cpp:156-161) on tcgen05 (3xTF32 for F32, or BF16)."""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ShapeError("gemm: inner dimensions disagree")
    c = np.zeros((m, n), np.float32)
    _check(_lib.mtg_gemm(precision, _ptr(a), _ptr(b), m, k, n, _ptr(c)))
    return c


def _factor_block(factors, off, n_factors: int):
    """[n_factors][total] ids aligned with the CSR source ids (minimt_gpu.h)."""
    total = int(off[-1])
    out = np.zeros((max(n_factors, 1), max(total, 1)), np.int32)
    for i, streams in enumerate(factors):
        if len(streams) != n_factors:
            raise ShapeError("factor streams: every sentence needs the same stream count")
        for f, stream in enumerate(streams):
            if len(stream) != off[i + 1] - off[i]:
                raise ShapeError("embed_source: factor stream not aligned with words")
            out[f, off[i]:off[i + 1]] = np.asarray(stream, np.int32)
    return out


def _csr(sources: Sequence[Sequence[int]]):
    off = np.zeros(len(sources) + 1, np.int64)
    np.cumsum([len(s) for s in sources], out=off[1:])
    total = int(off[-1])
    ids = np.zeros(max(total, 1), np.int32)
    if total:
        ids[:total] = np.fromiter(itertools.chain.from_iterable(sources), np.int64, total)
    return ids, off


# ---- model handle (the Executor plugin point) --------------------------------------

class Model:
    """A device-resident model = the reference's Executor (model.hpp:113-171)."""

    def __init__(self, handle, precision: int):
        self._h = handle
        self.precision = precision
        buf = ctypes.create_string_buffer(4096)
        _check(_lib.mtg_model_config_json(self._h, buf, 4096))
        self.config_json = buf.value.decode()
        self.config = json.loads(self.config_json)

    @staticmethod
    def create(config, seed: int = 1, precision: int = F32, device: int = 0) -> "Model":
        """init_params(Rng(seed)) weights (model.cpp:229-238)."""
        cfg = config.to_json() if isinstance(config, ModelConfig) else (
            json.dumps(config) if isinstance(config, dict) else config)
        h = ctypes.c_void_p()
        _check(_lib.mtg_model_create(cfg.encode(), seed, precision, device, ctypes.byref(h)))
        return Model(h, _lib.mtg_model_precision(h))

    @staticmethod
    def load(path: str, precision: int = F32, device: int = 0) -> "Model":
        """SQNT file (io.hpp); int8 files always decode INT8."""
        h = ctypes.c_void_p()
        _check(_lib.mtg_model_load(path.encode(), precision, device, ctypes.byref(h)))
        return Model(h, _lib.mtg_model_precision(h))

    def save(self, path: str) -> None:
        _check(_lib.mtg_model_save(self._h, path.encode()))

    def close(self) -> None:
        if self._h:
            _lib.mtg_model_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def max_seq_len(self) -> int:
        return int(self.config["max_seq_len"])

    def translate(self, sources: Sequence[Sequence[int]], cfg: BeamConfig,
                  max_batch: int = 0, factors=None, shortlists=None) -> List[Hypothesis]:
        """Batched beam_search (decode.cpp:34-109) over id sequences that already
        end with EOS. Per-sentence errors come back in Hypothesis.status.
        factors: per sentence, the model's source-factor streams (each aligned
        with its source, EOS position included). shortlists: per sentence a
        strictly increasing target-id list, or an empty one for the full
        vocabulary (decode.cpp:344-349)."""
        ids, off = _csr(sources)
        n = len(sources)
        T = self.max_seq_len
        toks = np.zeros((max(n, 1), T), np.int32)
        ln = np.zeros(max(n, 1), np.int32)
        lp = np.zeros(max(n, 1), np.float32)
        nm = np.zeros(max(n, 1), np.float32)
        fl = np.zeros(max(n, 1), np.uint32)
        st = np.zeros(max(n, 1), np.int32)
        c = _BeamConfigC(cfg.beam_size, cfg.max_len, cfg.length_penalty_alpha, max_batch)
        if shortlists is not None:
            nf = len(factors[0]) if (factors is not None and n) else 0
            fb = _factor_block(factors, off, nf) if factors is not None else None
            sl_ids, sl_off = _csr(shortlists)
            _check(_lib.mtg_translate_ex(self._h, _ptr(ids), _ptr(off), n,
                                         None if fb is None else _ptr(fb), nf, _ptr(sl_ids),
                                         _ptr(sl_off), ctypes.byref(c), _ptr(toks), T, _ptr(ln),
                                         _ptr(lp), _ptr(nm), _ptr(fl), _ptr(st)))
        elif factors is not None:
            nf = len(factors[0]) if n else 0
            fb = _factor_block(factors, off, nf)
            _check(_lib.mtg_translate_factors(self._h, _ptr(ids), _ptr(off), n, _ptr(fb), nf,
                                              ctypes.byref(c), _ptr(toks), T, _ptr(ln), _ptr(lp),
                                              _ptr(nm), _ptr(fl), _ptr(st)))
        else:
            _check(_lib.mtg_translate(self._h, _ptr(ids), _ptr(off), n, ctypes.byref(c), _ptr(toks),
                                      T, _ptr(ln), _ptr(lp), _ptr(nm), _ptr(fl), _ptr(st)))
        return [Hypothesis(toks[i, :ln[i]].tolist(), float(lp[i]), bool(fl[i] & HYP_FINISHED),
                           bool(fl[i] & HYP_TRUNCATED), float(nm[i]), int(st[i])) for i in range(n)]

    def forced_logits(self, sources: Sequence[Sequence[int]], forced: Sequence[int]) -> np.ndarray:
        """decode_step logits (model.cpp:614-672) along BOS + forced[:-1]."""
        ids, off = _csr(sources)
        f = np.ascontiguousarray(forced, np.int32)
        V = int(self.config["tgt_vocab_size"])
        out = np.zeros((len(sources), len(f), V), np.float32)
        _check(_lib.mtg_forced_logits(self._h, _ptr(ids), _ptr(off), len(sources), _ptr(f), len(f),
                                      _ptr(out)))
        return out

    def encode(self, sources: Sequence[Sequence[int]], factors=None) -> np.ndarray:
        """encode_infer(embed_source_infer(.)) rows, concatenated."""
        ids, off = _csr(sources)
        out = np.zeros((int(off[-1]), int(self.config["d_model"])), np.float32)
        if factors is not None:
            nf = len(factors[0]) if len(sources) else 0
            fb = _factor_block(factors, off, nf)
            _check(_lib.mtg_encode_factors(self._h, _ptr(ids), _ptr(off), len(sources), _ptr(fb),
                                           nf, _ptr(out)))
        else:
            _check(_lib.mtg_encode(self._h, _ptr(ids), _ptr(off), len(sources), _ptr(out)))
        return out

    # benchmark helpers: device-resident sources
    def stage(self, sources: Sequence[Sequence[int]]) -> None:
        ids, off = _csr(sources)
        _check(_lib.mtg_stage_sources(self._h, _ptr(ids), _ptr(off), len(sources)))

    def run_staged(self, cfg: BeamConfig) -> None:
        c = _BeamConfigC(cfg.beam_size, cfg.max_len, cfg.length_penalty_alpha, 0)
        _check(_lib.mtg_translate_staged(self._h, ctypes.byref(c)))

    def last_launch_count(self) -> int:
        return int(_lib.mtg_last_launch_count(self._h))

    def diag_report(self) -> str:
        """Per-kernel decode-step times (needs MTG_DIAG_EVENTS=1 at model creation)."""
        buf = ctypes.create_string_buffer(1 << 16)
        _check(_lib.mtg_diag_report(self._h, buf, len(buf)))
        return buf.value.decode()


def beam_search(model: Model, src_ids: Sequence[int], factor_ids=(), config: BeamConfig = None,
                shortlist=None) -> Hypothesis:
    """decode.hpp:35-38 for one sentence."""
    cfg = config or BeamConfig()
    if cfg.beam_size < 1:
        raise UsageError("beam_search: beam size >= 1")
    if len(src_ids) == 0:
        raise UsageError("beam_search: empty source")
    n_f = len(model.config.get("factors", []) or [])
    fac = [[list(f) for f in factor_ids]] if (factor_ids or n_f) else None
    sl = [list(shortlist)] if shortlist is not None else None
    h = model.translate([list(src_ids)], cfg, factors=fac, shortlists=sl)[0]
    if h.status:
        raise _ERRORS.get(h.status, MinimtError)("beam_search failed")
    return h


def prepare_source(word_ids: Sequence[int], max_seq_len: int) -> List[int]:
    """translate_one (decode.cpp:326-333): append EOS, truncate keeping EOS."""
    src = list(word_ids) + [EOS_ID]
    if len(src) > max_seq_len:
        src = src[:max_seq_len - 1] + [EOS_ID]
    return src


def percentile(durations: Sequence[float], p: float) -> float:
    """eval.cpp:120-128 nearest-rank percentile."""
    import math
    if not durations:
        raise UsageError("percentile: empty list")
    if p <= 0.0 or p > 100.0:
        raise UsageError("percentile: need 0 < p <= 100")
    v = sorted(durations)
    rank = max(1, int(math.ceil(p / 100.0 * len(v))))
    return v[rank - 1]

"""ctypes wrapper over oracle/build/liboracle.so -- TEST INFRASTRUCTURE.

The oracle is the CPU restatement of the reference inference path
(oracle/oracle.hpp). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm may use it, and only as the checker.
"""

from __future__ import annotations

import ctypes
import json
import os
from typing import Optional, Sequence

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_PATH = os.path.join(ROOT, "oracle", "build", "liboracle.so")

_c_int, _c_float, _vp = ctypes.c_int, ctypes.c_float, ctypes.c_void_p


def _load():
    if not os.path.exists(ORACLE_PATH):
        raise ImportError(f"{ORACLE_PATH} missing: run `make -C oracle`")
    lib = ctypes.CDLL(ORACLE_PATH)
    lib.orc_last_error.restype = ctypes.c_char_p
    lib.orc_model_create.restype = _vp
    lib.orc_model_create.argtypes = [ctypes.c_char_p, ctypes.c_uint64, _c_int]
    lib.orc_model_load.restype = _vp
    lib.orc_model_load.argtypes = [ctypes.c_char_p]
    lib.orc_model_free.argtypes = [_vp]
    lib.orc_model_free.restype = None
    lib.orc_model_save.argtypes = [_vp, ctypes.c_char_p, _c_int]
    lib.orc_model_config_json.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.orc_param_count.argtypes = [_vp]
    lib.orc_param_count.restype = ctypes.c_longlong
    lib.orc_get_param.argtypes = [_vp, ctypes.c_char_p, _vp, ctypes.c_longlong]
    lib.orc_set_param.argtypes = [_vp, ctypes.c_char_p, _vp, ctypes.c_longlong]
    lib.orc_get_qparam.argtypes = [_vp, ctypes.c_char_p, _vp, ctypes.c_longlong, _vp]
    lib.orc_pos_enc.argtypes = [_vp, _vp]
    lib.orc_encode_factors.argtypes = [_vp, _c_int, _vp, _c_int, _vp, _c_int, _vp]
    lib.orc_beam_search_factors.argtypes = [_vp, _c_int, _vp, _c_int, _vp, _c_int, _c_int, _c_int,
                                            _c_float, _vp, _c_int, _vp, _vp, _vp, _vp]
    lib.orc_beam_search.argtypes = [_vp, _c_int, _vp, _c_int, _c_int, _c_int, _c_float, _vp, _c_int,
                                    _vp, _c_int, _vp, _vp, _vp, _vp]
    lib.orc_translate_batch.argtypes = [_vp, _c_int, _vp, _vp, _c_int, _c_int, _c_int, _c_float,
                                        _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp]
    lib.orc_forced_logits.argtypes = [_vp, _c_int, _vp, _c_int, _vp, _c_int, _vp]
    lib.orc_teacher_forced.argtypes = [_vp, _vp, _c_int, _vp, _c_int, _vp]
    lib.orc_encode.argtypes = [_vp, _c_int, _vp, _c_int, _vp]
    lib.orc_quantize.argtypes = [_vp, ctypes.c_longlong, _vp, _vp]
    lib.orc_qmatmul.argtypes = [_vp, _c_float, _vp, _c_float, _c_int, _c_int, _c_int, _vp]
    lib.orc_layer_norm.argtypes = [_vp, _c_int, _c_int, _vp, _vp, _vp]
    lib.orc_log_softmax.argtypes = [_vp, _c_int, _vp]
    lib.orc_det_expf.argtypes = [_c_float]
    lib.orc_det_expf.restype = _c_float
    lib.orc_det_logf.argtypes = [_c_float]
    lib.orc_det_logf.restype = _c_float
    lib.orc_det_powf.argtypes = [_c_float, _c_float]
    lib.orc_det_powf.restype = _c_float
    lib.orc_normalized_score.argtypes = [_c_int, _c_float, _c_float]
    lib.orc_normalized_score.restype = _c_float
    lib.orc_percentile.argtypes = [_vp, _c_int, ctypes.c_double, _vp]
    lib.orc_prepare_source.argtypes = [_vp, _c_int, _c_int, _vp, _vp]
    return lib


lib = _load()

ERR_NAMES = {1: "ShapeError", 2: "ValueError", 3: "IndexError", 4: "StateError",
             5: "FormatError", 6: "UsageError", 7: "IoError"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERR_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERR_NAMES.get(code)


def check(rc: int) -> None:
    if rc:
        raise OracleError(rc, (lib.orc_last_error() or b"").decode())


def P(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def i32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


class OracleModel:
    def __init__(self, handle):
        if not handle:
            raise OracleError(lib.orc_last_error_code(), (lib.orc_last_error() or b"").decode())
        self.h = ctypes.c_void_p(handle)
        buf = ctypes.create_string_buffer(4096)
        check(lib.orc_model_config_json(self.h, buf, 4096))
        self.config_json = buf.value.decode()
        self.config = json.loads(self.config_json)

    @staticmethod
    def create(config, seed: int = 1, init: bool = True) -> "OracleModel":
        cfg = config if isinstance(config, str) else json.dumps(config)
        return OracleModel(lib.orc_model_create(cfg.encode(), seed, 1 if init else 0))

    @staticmethod
    def load(path: str) -> "OracleModel":
        return OracleModel(lib.orc_model_load(path.encode()))

    def __del__(self):
        try:
            lib.orc_model_free(self.h)
        except Exception:
            pass

    def save(self, path: str, quantized: bool = False) -> None:
        check(lib.orc_model_save(self.h, path.encode(), 1 if quantized else 0))

    @property
    def V(self) -> int:
        return int(self.config["tgt_vocab_size"])

    def param_count(self) -> int:
        return int(lib.orc_param_count(self.h))

    def get(self, name: str, shape) -> np.ndarray:
        out = np.zeros(shape, np.float32)
        check(lib.orc_get_param(self.h, name.encode(), P(out), out.size))
        return out

    def set(self, name: str, value: np.ndarray) -> None:
        v = np.ascontiguousarray(value, np.float32)
        check(lib.orc_set_param(self.h, name.encode(), P(v), v.size))

    def qparam(self, name: str, shape):
        out = np.zeros(shape, np.int8)
        s = ctypes.c_float()
        check(lib.orc_get_qparam(self.h, name.encode(), P(out), out.size, ctypes.byref(s)))
        return out, np.float32(s.value)

    def pos_enc(self) -> np.ndarray:
        out = np.zeros((self.config["max_seq_len"], self.config["d_model"]), np.float32)
        check(lib.orc_pos_enc(self.h, P(out)))
        return out

    def beam_search(self, src: Sequence[int], beam: int, max_len: int, alpha: float = 1.0,
                    int8: bool = False, shortlist: Optional[Sequence[int]] = None) -> dict:
        s = i32(src)
        cap = max(max_len, 1) + 1
        toks = np.zeros(cap, np.int32)
        n = ctypes.c_int()
        lp = ctypes.c_float()
        nm = ctypes.c_float()
        fl = ctypes.c_int()
        sl = None if shortlist is None else i32(shortlist)
        check(lib.orc_beam_search(self.h, int(int8), P(s), len(s), beam, max_len, alpha,
                                  None if sl is None else P(sl), 0 if sl is None else len(sl),
                                  P(toks), cap, ctypes.byref(n), ctypes.byref(lp), ctypes.byref(nm),
                                  ctypes.byref(fl)))
        return dict(tokens=toks[:n.value].tolist(), logprob=lp.value, norm=nm.value,
                    finished=bool(fl.value & 1), truncated=bool(fl.value & 2))

    def translate_batch(self, sources, beam: int, max_len: int = 0, alpha: float = 1.0,
                        int8: bool = False, threads: int = 1):
        n = len(sources)
        off = np.zeros(n + 1, np.int64)
        for i, s in enumerate(sources):
            off[i + 1] = off[i] + len(s)
        ids = np.zeros(max(int(off[-1]), 1), np.int32)
        for i, s in enumerate(sources):
            ids[off[i]:off[i + 1]] = s
        stride = int(self.config["max_seq_len"]) + 1
        toks = np.zeros((max(n, 1), stride), np.int32)
        ln = np.zeros(max(n, 1), np.int32)
        lp = np.zeros(max(n, 1), np.float32)
        nm = np.zeros(max(n, 1), np.float32)
        fl = np.zeros(max(n, 1), np.int32)
        st = np.zeros(max(n, 1), np.int32)
        check(lib.orc_translate_batch(self.h, int(int8), P(ids), P(off), n, beam, max_len, alpha,
                                      threads, P(toks), stride, P(ln), P(lp), P(nm), P(fl), P(st)))
        return [dict(tokens=toks[i, :ln[i]].tolist(), logprob=float(lp[i]), norm=float(nm[i]),
                     finished=bool(fl[i] & 1), truncated=bool(fl[i] & 2), status=int(st[i]))
                for i in range(n)]

    def forced_logits(self, src, forced, int8: bool = False) -> np.ndarray:
        s, f = i32(src), i32(forced)
        out = np.zeros((len(f), self.V), np.float32)
        check(lib.orc_forced_logits(self.h, int(int8), P(s), len(s), P(f), len(f), P(out)))
        return out

    def teacher_forced(self, src, tgt) -> np.ndarray:
        s, t = i32(src), i32(tgt)
        out = np.zeros((len(t), self.V), np.float32)
        check(lib.orc_teacher_forced(self.h, P(s), len(s), P(t), len(t), P(out)))
        return out

    def encode(self, src, int8: bool = False, factors=None) -> np.ndarray:
        s = i32(src)
        out = np.zeros((len(s), self.config["d_model"]), np.float32)
        if factors is not None:
            f = i32(np.asarray(factors, np.int32).reshape(-1))
            check(lib.orc_encode_factors(self.h, int(int8), P(s), len(s), P(f), len(factors), P(out)))
        else:
            check(lib.orc_encode(self.h, int(int8), P(s), len(s), P(out)))
        return out

    def beam_search_factors(self, src, factors, beam: int, max_len: int, alpha: float = 1.0,
                            int8: bool = False) -> dict:
        """decode.hpp:35-38 with source-factor streams (each aligned with src)."""
        s = i32(src)
        f = i32(np.asarray(factors, np.int32).reshape(-1))
        cap = max(max_len, 1) + 1
        toks = np.zeros(cap, np.int32)
        n = ctypes.c_int()
        lp = ctypes.c_float()
        nm = ctypes.c_float()
        fl = ctypes.c_int()
        check(lib.orc_beam_search_factors(self.h, int(int8), P(s), len(s), P(f), len(factors), beam,
                                          max_len, alpha, P(toks), cap, ctypes.byref(n),
                                          ctypes.byref(lp), ctypes.byref(nm), ctypes.byref(fl)))
        return dict(tokens=toks[:n.value].tolist(), logprob=lp.value, norm=nm.value,
                    finished=bool(fl.value & 1), truncated=bool(fl.value & 2))


def quantize(x: np.ndarray):
    x = np.ascontiguousarray(x, np.float32)
    q = np.zeros(x.shape, np.int8)
    s = ctypes.c_float()
    check(lib.orc_quantize(P(x), x.size, P(q), ctypes.byref(s)))
    return q, np.float32(s.value)


def qmatmul(a, sa, b, sb) -> np.ndarray:
    a = np.ascontiguousarray(a, np.int8)
    b = np.ascontiguousarray(b, np.int8)
    c = np.zeros((a.shape[0], b.shape[1]), np.float32)
    check(lib.orc_qmatmul(P(a), sa, P(b), sb, a.shape[0], a.shape[1], b.shape[1], P(c)))
    return c


def layer_norm(x, g, b) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(x)
    check(lib.orc_layer_norm(P(x), x.shape[0], x.shape[1], P(np.ascontiguousarray(g, np.float32)),
                             P(np.ascontiguousarray(b, np.float32)), P(out)))
    return out


def log_softmax(x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    out = np.zeros_like(x)
    check(lib.orc_log_softmax(P(x), x.size, P(out)))
    return out


def percentile(v, p: float) -> float:
    a = np.ascontiguousarray(v, np.float64)
    out = ctypes.c_double()
    check(lib.orc_percentile(P(a), len(a), p, ctypes.byref(out)))
    return out.value


def det_expf(x: float) -> float:
    return lib.orc_det_expf(x)


def det_logf(x: float) -> float:
    return lib.orc_det_logf(x)


def normalized_score(n_tokens: int, logprob: float, alpha: float) -> float:
    return lib.orc_normalized_score(n_tokens, logprob, alpha)


def prepare_source(words, max_seq_len: int):
    w = i32(words)
    out = np.zeros(len(w) + 1, np.int32)
    n = ctypes.c_int()
    check(lib.orc_prepare_source(P(w), len(w), max_seq_len, P(out), ctypes.byref(n)))
    return out[:n.value].tolist()


def synthetic_sources(n: int, length: int, vocab: int, seed: int = 7):
    """SURVEY §8d synthetic inputs: ids uniform over [4, vocab) from
    std::mt19937_64(seed) semantics are not needed bit-for-bit; numpy's PCG64
    stream is used (same distribution), then EOS appended."""
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(4, vocab, length))) + [3] for _ in range(n)]

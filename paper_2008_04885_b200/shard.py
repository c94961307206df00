"""Multi-GPU plumbing for the translation path.

Sentences are independent (the reference runs them as independent calls,
decode.cpp:370-398), so a corpus is sharded across ranks with no data-path
collective: each rank owns a replica of the model and a length-balanced
subset of sentences. The only collective is one gather of fixed-size
hypothesis records to rank 0 at the end (NCCL on B200s; gloo in CPU tests).
"""

from __future__ import annotations

from typing import List, Sequence

import numpy as np


def sentence_cost(src_len: int, beam: int, max_seq_len: int = 128) -> float:
    """Relative work of one sentence: encoder ~ S rows; decoder ~ max_len
    steps x beam rows, max_len = min(max_seq_len, 2S+5) (decode.cpp:352-355).
    The 20:2 per-row FLOP ratio (encoder row : decoder row-step) is ~1 : 0.55."""
    steps = min(max_seq_len, 2 * src_len + 5)
    return src_len * 1.0 + steps * beam * 0.55


def partition(lengths: Sequence[int], world_size: int, beam: int = 5,
              max_seq_len: int = 128) -> List[List[int]]:
    """Greedy longest-processing-time assignment of sentences to ranks on the
    estimated cost; each rank's list is returned sorted by source length so
    its device batches are length-bucketed."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    order = sorted(range(len(lengths)),
                   key=lambda i: (-sentence_cost(lengths[i], beam, max_seq_len), i))
    loads = [0.0] * world_size
    parts: List[List[int]] = [[] for _ in range(world_size)]
    for i in order:
        r = min(range(world_size), key=lambda k: (loads[k], k))
        parts[r].append(i)
        loads[r] += sentence_cost(lengths[i], beam, max_seq_len)
    for p in parts:
        p.sort(key=lambda i: (lengths[i], i))
    return parts


def batches(indices: Sequence[int], max_batch: int) -> List[List[int]]:
    """Consecutive length-sorted chunks of at most max_batch sentences."""
    idx = list(indices)
    return [idx[i:i + max_batch] for i in range(0, len(idx), max(1, max_batch))]


RECORD_HEADER = 6  # sentence id, n_tokens, flags, status, logprob bits, norm bits


def pack_records(ids: Sequence[int], hyps, max_len: int) -> np.ndarray:
    """Fixed-size int32 records {id, n, flags, status, logprob, norm, tokens[max_len]}."""
    rec = np.full((len(ids), RECORD_HEADER + max_len), -1, np.int32)
    for row, (i, h) in enumerate(zip(ids, hyps)):
        rec[row, 0] = i
        rec[row, 1] = len(h.tokens)
        rec[row, 2] = (1 if h.finished else 0) | (2 if h.truncated else 0)
        rec[row, 3] = h.status
        rec[row, 4] = np.float32(h.logprob).view(np.int32)
        rec[row, 5] = np.float32(h.normalized).view(np.int32)
        rec[row, RECORD_HEADER:RECORD_HEADER + len(h.tokens)] = h.tokens
    return rec


def unpack_records(rec: np.ndarray):
    """Inverse of pack_records -> {sentence id: dict}."""
    out = {}
    for r in rec:
        if r[0] < 0:
            continue
        n = int(r[1])
        out[int(r[0])] = dict(tokens=r[RECORD_HEADER:RECORD_HEADER + n].tolist(),
                              finished=bool(r[2] & 1), truncated=bool(r[2] & 2),
                              status=int(r[3]),
                              logprob=float(np.int32(r[4]).view(np.float32)),
                              normalized=float(np.int32(r[5]).view(np.float32)))
    return out


def gather_to_rank0(records: np.ndarray, device=None):
    """One collective: all-gather the (padded) record tables so rank 0 holds
    every hypothesis. Uses torch.distributed's active backend (NCCL over
    NVLink on the GPU box, gloo in CPU tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    n = torch.tensor([records.shape[0]], dtype=torch.int64, device=device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n)
    width = records.shape[1]
    cap = int(max(int(c.item()) for c in counts))
    pad = np.full((cap, width), -1, np.int32)
    pad[:records.shape[0]] = records
    t = torch.from_numpy(pad).to(device) if device is not None else torch.from_numpy(pad)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if dist.get_rank() != 0:
        return None
    return np.concatenate([p.cpu().numpy()[:int(c.item())] for p, c in zip(parts, counts)])

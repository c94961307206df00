# BASELINE configs[2] and [4] on one B200:
#   * 6:6 vs 10:10 vs 20:2 batched decoding sweep (batch 1-256, beam 1/5/10),
#     fp32 and int8, 20-token synthetic sources (PAPER Table 1 protocol), plus
#     p50/p90 batch-1 latency (nearest rank, eval.cpp:120-128) at beam 5;
#   * a length-bucketed corpus (uniform 5-60 tokens, the 1M-sentence sharding
#     workload's length mix) through the public translate call with
#     max_batch-sized device batches (the per-rank loop of shard.py at world 1).
# Device-resident sweep points time mtg_translate_staged (wall clock around a
# synchronized call, median of 3 after a warm-up); the corpus and latency
# rows go through mtg_translate with host buffers.
#
#   python tools/sweep.py [--quick] [--out profiles/r01_sweep.json]
import argparse, json, os, sys, time
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_04885_b200 as mt
from paper_2008_04885_b200 import shard

BASE = dict(d_model=512, d_ff=2048, num_heads=8, src_vocab_size=32000, tgt_vocab_size=32000,
            dropout=0.1, max_seq_len=128)
MODELS = {"6:6": (6, 6), "10:10": (10, 10), "20:2": (20, 2)}


def srcs(n, length, seed):
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(4, 32000, length))) + [3] for _ in range(n)]


def timed(f, reps=3):
    f()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--corpus", type=int, default=20000)
    ap.add_argument("--corpus-only", action="store_true")
    a = ap.parse_args()
    batches = [1, 16, 64] if a.quick else [1, 16, 64, 256]
    beams = [1, 5, 10]
    rows = []
    for mname, (le, ld) in MODELS.items():
        if a.corpus_only and mname != "20:2":
            continue
        cfg = dict(BASE, num_encoder_layers=le, num_decoder_layers=ld)
        for pname, prec in (("f32", mt.F32), ("int8", mt.INT8)):
            m = mt.Model.create(cfg, seed=1, precision=prec)
            for beam in ([] if a.corpus_only else beams):
                for b in batches:
                    s = srcs(b, 20, 7)
                    m.stage(s)
                    bc = mt.BeamConfig(beam, 0, 1.0)
                    t = timed(lambda: m.run_staged(bc))
                    rows.append(dict(kind="throughput", model=mname, precision=pname, beam=beam,
                                     batch=b, sentences_per_s=b / t, ms_per_batch=t * 1e3))
                    print(json.dumps(rows[-1]), flush=True)
            lat = []
            bc = mt.BeamConfig(5, 0, 1.0)
            one = srcs(4 if a.corpus_only else 30, 20, 99)
            for x in one[:3]:
                m.translate([x], bc)
            for x in one:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                m.translate([x], bc)
                lat.append((time.perf_counter() - t0) * 1e3)
            rows.append(dict(kind="latency", model=mname, precision=pname, beam=5, batch=1,
                             p50_ms=mt.percentile(lat, 50.0), p90_ms=mt.percentile(lat, 90.0)))
            print(json.dumps(rows[-1]), flush=True)
            if mname == "20:2":
                rng = np.random.default_rng(11)
                lens = rng.integers(5, 61, a.corpus)
                corpus = [list(map(int, rng.integers(4, 32000, int(n)))) + [3] for n in lens]
                order = shard.partition([len(x) for x in corpus], 1)[0]
                bc = mt.BeamConfig(5, 0, 1.0)
                for mb in (128, 256):
                    chunks = shard.batches(order, mb)
                    m.translate([corpus[i] for i in chunks[0]], bc)  # warm-up
                    # pass 1: every batch shape new (captures, plans); pass 2: steady state
                    for pas in ("first", "second"):
                        torch.cuda.synchronize()
                        t0 = time.perf_counter()
                        n_out = 0
                        for ch in chunks:
                            n_out += len(m.translate([corpus[i] for i in ch], bc))
                        torch.cuda.synchronize()
                        t = time.perf_counter() - t0
                        rows.append(dict(kind="bucketed_corpus", model=mname, precision=pname,
                                         beam=5, max_batch=mb, sentences=n_out, pass_=pas,
                                         src_len="uniform 5-60 (+EOS)",
                                         sentences_per_s=n_out / t, seconds=t))
                        print(json.dumps(rows[-1]), flush=True)
            m.close()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(dict(gpu=torch.cuda.get_device_name(0), rows=rows), f, indent=1)


if __name__ == "__main__":
    main()

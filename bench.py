#!/usr/bin/env python3
"""Benchmark: sentences/s of batched beam search (beam 5) on the 20:2
transformer with synthetic 25-token sources, batch 64 per GPU
(BASELINE.json configs[1]); one JSON line on stdout (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision f32|int8|bf16]
  python bench.py --impl reference ...   # the reference CPU decoder (oracle port)

A "step" = one call of the batched beam search over one batch of 64 sentences
(encoder + every decode step + top-k + beam bookkeeping). `value` times the
device-resident path (sources staged in HBM) with CUDA events on the engine's
stream; `e2e` times the public C-ABI call (mtg_translate) with host buffers,
H2D of the sources and D2H of the hypotheses inside the timed region.
Multi-GPU (torchrun): weak scaling, each rank decodes its own 64-sentence
batch per step; timing is the max over ranks; hypotheses are gathered to
rank 0 with one NCCL all-gather after the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sentences/sec (beam 5, 20:2, synthetic) at 1/2/4/8 B200; p90 batch-1 latency"
UNIT = "sentences/s"
CONFIG_20_2 = dict(num_encoder_layers=20, num_decoder_layers=2, d_model=512, d_ff=2048,
                   num_heads=8, src_vocab_size=32000, tgt_vocab_size=32000, dropout=0.1,
                   max_seq_len=128)
BATCH, SRC_LEN, BEAM = 64, 25, 5


def sources(n: int, seed: int):
    import numpy as np
    rng = np.random.default_rng(seed)
    return [list(map(int, rng.integers(4, 32000, SRC_LEN))) + [3] for _ in range(n)]


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def config_block(args, world):
    return {"workload": "20:2 transformer (d512 ff2048 h8, V=32k) random-init, beam 5, "
                        "batch 64 x 25-token synthetic sources per GPU (BASELINE configs[1])",
            "model": "sockeye2-20:2", "global_batch": BATCH * world, "src_len": SRC_LEN + 1,
            "beam": BEAM, "max_len": "2*|src|+5 = 57", "precision": args.precision,
            "parallelism": f"dp{world} (sentence sharding, replicas)",
            "l2": "flushed between timed steps (256 MiB write)"}


# ---- reference arm ----------------------------------------------------------------

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as orc
    threads = os.cpu_count() or 1
    int8 = args.precision == "int8"
    om = orc.OracleModel.create(CONFIG_20_2, seed=1)
    srcs = sources(BATCH, 7)
    sample = min(BATCH, max(threads, 1))
    for _ in range(args.warmup):
        orc_run = om.translate_batch(srcs[:min(sample, 2)], BEAM, 0, 1.0, int8=int8,
                                     threads=threads)
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        orc_run = om.translate_batch(srcs[:sample], BEAM, 0, 1.0, int8=int8, threads=threads)
        times.append(time.perf_counter() - t0)
    assert all(r["status"] == 0 for r in orc_run)
    total = sum(times)
    value = sample * args.steps / total
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "int8" if int8 else "f32", "data": "synthetic (random-init weights, "
            "uniform token ids)", "config": config_block(args, 1),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} of the 64 sentences per step, "
                                       f"parallel_sentences={threads} (decode.cpp:370-398); "
                                       "reference unbuildable here (Eigen3/vendor absent), "
                                       "oracle/ C++ restatement timed instead"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- GPU arm --------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.proc = None
        self.index = index
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r]
        except OSError:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if len(r) >= 9]
        smax = [float(r[2]) for r in rows if len(r) >= 9]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(sm), "window": "warm-up + timed steps (100 ms period)"}


def run_gpu(args):
    import numpy as np
    import torch
    import paper_2008_04885_b200 as mt

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prec = {"f32": mt.F32, "int8": mt.INT8, "bf16": mt.BF16}[args.precision]
    model = mt.Model.create(CONFIG_20_2, seed=1, precision=prec, device=local)
    stream = torch.cuda.ExternalStream(mt.lib().mtg_model_stream(model._h))
    cfg = mt.BeamConfig(BEAM, 0, 1.0)
    srcs = sources(BATCH, 7 + rank)
    model.stage(srcs)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # nvidia-smi needs ~0.1-0.2 s to start sampling and a 5-step region lasts
    # ~70-110 ms, so the sampler runs from the first warm-up step (same load)
    # through the timed steps.
    with ClockSampler(local) as clocks:
        for _ in range(max(args.warmup, 3)):
            model.run_staged(cfg)
        torch.cuda.synchronize()

        # ---- device-resident timed region ----
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(k))
                starts[k].record(stream)
            model.run_staged(cfg)
            with torch.cuda.stream(stream):
                ends[k].record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(step_ms)
    launches = model.last_launch_count() * args.steps
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * BATCH * args.steps / (total_ms / 1000.0)

    # ---- end-to-end through the public C-ABI (host buffers, H2D + D2H) ----
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        hyps = model.translate(srcs, cfg)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    assert all(h.status == 0 for h in hyps)
    h2d = sum(len(s) for s in srcs) * 4 + (BATCH + 1) * 8
    d2h = BATCH * (4 * CONFIG_20_2["max_seq_len"] + 4 * 5)

    # ---- gather hypotheses to rank 0 (the only collective) ----
    if world > 1:
        from paper_2008_04885_b200 import shard
        rec = shard.pack_records([rank * BATCH + i for i in range(BATCH)], hyps,
                                 CONFIG_20_2["max_seq_len"])
        gathered = shard.gather_to_rank0(rec, device=torch.device("cuda", local))
        if rank == 0:
            assert len(shard.unpack_records(gathered)) == world * BATCH

    extra = {}
    if rank == 0:
        # roofline: dominant kernel timed alone with CUDA events on the engine stream
        import ctypes
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except OSError:
            pass
        hbm_peak = peaks.get("hbm_gbs", 6650.0)
        tc_peak = peaks.get("bf16_tflops", 1590.0)
        ms, by, fl = ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        kern = {}
        for kid, name in ((0, "logits_gemm"), (1, "logsoftmax_topk"), (2, "dec_self_attention"),
                          (3, "enc_ffn_w1_gemm")):
            rc = mt.lib().mtg_time_kernel(model._h, kid, 20, ctypes.byref(ms), ctypes.byref(by),
                                          ctypes.byref(fl))
            if rc == 0:
                kern[name] = dict(ms=ms.value, bytes=by.value, flops=fl.value)
        g = kern["logits_gemm"]
        # ncu summaries: the latest round's capture of the projection kernel
        # (DRAM traffic per launch), the measured tensor peaks from round 1.
        ncu, ncu_r01 = {}, {}
        for path in (os.path.join(ROOT, "profiles", "r02", "r02_ncu.json"),
                     os.path.join(ROOT, "profiles", "r01_ncu.json")):
            try:
                ncu = json.load(open(path))
                break
            except OSError:
                pass
        try:
            ncu_r01 = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu.json")))
        except OSError:
            pass
        measured = ncu.get("peaks_measured", ncu_r01.get("peaks_measured", {}))
        if prec == mt.INT8:
            tc_frac_peak = measured.get("int8_tops", 2.0 * tc_peak)
            src = ("int8 dense s8 TOPS measured by tools/peaks.py (torch._int_mm 8192^3), "
                   "profiles/r01_ncu.json; MEASURED_PEAKS.json has no int8 entry")
        elif prec == mt.F32:
            tc_frac_peak = measured.get("tf32_tflops", tc_peak)
            src = ("tf32 dense TFLOP/s measured by tools/peaks.py (profiles/r01_ncu.json); "
                   "achieved counts the 3 tf32 MMAs of 3xTF32")
        else:
            tc_frac_peak = tc_peak
            src = "MEASURED_PEAKS.json bf16_tflops (burst)"
        nk = ncu.get("kernels", {}).get("logits_gemm_" + args.precision)
        traffic = (nk["dram_read_bytes"] + nk["dram_write_bytes"]) if nk else None
        achieved = g["flops"] / (g["ms"] * 1e-3) / 1e12
        extra["roofline"] = {
            "kernel": "logits_gemm (tcgen05 output projection, R=320 x V=32000 x K=512)",
            "bound": "tensor", "achieved": achieved, "peak": tc_frac_peak,
            "unit": "TFLOP/s",  # int8: tera-ops (2 per multiply-add)
            "frac": achieved / tc_frac_peak, "traffic": traffic,
            "algorithmic_bytes": g["bytes"], "peak_source": src}
        extra["kernels"] = {
            k: dict(ms=v["ms"], gbs=v["bytes"] / (v["ms"] * 1e-3) / 1e9,
                    hbm_frac=v["bytes"] / (v["ms"] * 1e-3) / 1e9 / hbm_peak,
                    tflops=v["flops"] / (v["ms"] * 1e-3) / 1e12) for k, v in kern.items()}
        # p90 batch-1 latency (nearest rank, eval.cpp:120-128) on the same model
        # 50 single-sentence calls after 3 untimed ones (the first call after the
        # batch-64 run re-plans and re-captures for the small workspace).
        lat = []
        one = sources(53, 99)
        for s in one[:3]:
            model.translate([s], cfg)
        one = one[3:]
        for s in one:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            model.translate([s], cfg)
            lat.append((time.perf_counter() - t0) * 1000)
        extra["p90_batch1_ms"] = mt.percentile(lat, 90.0)
        extra["p50_batch1_ms"] = mt.percentile(lat, 50.0)
        # Batch-1 (small-batch GEMV path) kernels, each chained 50x in one CUDA
        # graph with PDL on the last batch-1 workspace: in-graph time per launch
        # and its weight / KV bytes against the HBM roofline.
        b1 = {}
        for kid, name in ((13, "gemv_logits_partials"), (12, "gemv_ln_w1"), (11, "gemv_wo"),
                          (16, "self_attention_t56")):
            rc = mt.lib().mtg_time_kernel(model._h, kid, 50, ctypes.byref(ms), ctypes.byref(by),
                                          ctypes.byref(fl))
            if rc == 0:
                gbs = by.value / (ms.value * 1e-3) / 1e9
                b1[name] = dict(us=ms.value * 1e3, bytes=by.value, gbs=gbs, hbm_frac=gbs / hbm_peak)
        extra["batch1_kernels"] = b1
        # CPU baseline: oracle port, bounded sample, all host threads
        if world == 1 and not args.no_cpu_baseline:
            sys.path.insert(0, os.path.join(ROOT, "tests"))
            import oracle_lib as orc
            threads = os.cpu_count() or 1
            om = orc.OracleModel.create(CONFIG_20_2, seed=1)
            sample = min(BATCH, threads)
            t0 = time.perf_counter()
            om.translate_batch(srcs[:sample], BEAM, 0, 1.0, int8=(prec == mt.INT8), threads=threads)
            cpu_s = time.perf_counter() - t0
            extra["cpu_baseline"] = {
                "value": sample / cpu_s, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"{sample} of the 64 sentences, parallel_sentences={threads}; oracle/ "
                          "C++ restatement (reference unbuildable: Eigen3/vendor absent)"}
        else:
            extra["cpu_baseline"] = None

        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": {"f32": "f32 (3xTF32 tcgen05, fp32 accumulate)", "int8": "int8 (s8xs8->s32)",
                          "bf16": "bf16 (fp32 accumulate)"}[args.precision],
                "data": "synthetic (random-init weights per model.cpp:229-238, uniform ids)",
                "config": config_block(args, world),
                "e2e": {"value": world * BATCH * e2e_steps / e2e_s, "unit": UNIT,
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": launches, "clocks": clocks.summary()}
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="f32", choices=["f32", "int8", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

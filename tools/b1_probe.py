# Batch-1 latency breakdown: whole translate vs encoder alone (wall clock,
# synchronized), per precision.
import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
precs = sys.argv[1:] or ["int8", "f32"]
for name in precs:
    prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[name]
    m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
    one = sources(20, 99)
    cfg = mt.BeamConfig(5, 0, 1.0)
    for s in one[:3]: m.translate([s], cfg); m.encode([s])
    def t(f):
        ts = []
        for s in one:
            torch.cuda.synchronize(); t0 = time.perf_counter(); f(s); ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort(); return ts[len(ts) // 2]
    tr = t(lambda s: m.translate([s], cfg)); en = t(lambda s: m.encode([s]))
    print(f"{name}: translate p50 {tr:.2f} ms, encode p50 {en:.2f} ms, launches {m.last_launch_count()}")

# Encoder-only timing (mtg_encode: stage + encoder + D2H of the states).
import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
for name, prec in (("int8", mt.INT8), ("f32", mt.F32)):
    m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
    srcs = sources(64, 7)
    for _ in range(3): m.encode(srcs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): m.encode(srcs)
    torch.cuda.synchronize()
    print(name, "encode 64 sentences: %.3f ms" % ((time.perf_counter() - t0) * 100), "launches", m.last_launch_count())

# Encoder-only wall time (min over 40 calls of mtg_encode, 64 sentences).
import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
for name in sys.argv[1:] or ["int8", "f32"]:
    prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[name]
    m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
    srcs = sources(64, 7)
    for _ in range(5): m.encode(srcs)
    ts = []
    for _ in range(40):
        torch.cuda.synchronize(); t0 = time.perf_counter(); m.encode(srcs); ts.append(time.perf_counter() - t0)
    ts.sort()
    print(name, "encode 64: min %.3f ms  p25 %.3f ms" % (ts[0] * 1e3, ts[10] * 1e3))

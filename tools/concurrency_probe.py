# Probe: do independent beam searches on separate engines/streams overlap?
import sys, time, threading, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
prec = mt.INT8
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
per = int(sys.argv[2]) if len(sys.argv) > 2 else 64
models = [mt.Model.create(CONFIG_20_2, seed=1, precision=prec) for _ in range(K)]
srcs = [sources(per, 7 + i) for i in range(K)]
cfg = mt.BeamConfig(5, 0, 1.0)
for m, s in zip(models, srcs):
    m.stage(s); m.run_staged(cfg); m.run_staged(cfg)
torch.cuda.synchronize()
def run(i, n):
    for _ in range(n): models[i].run_staged(cfg)
for k in range(1, K + 1):
    ths = [threading.Thread(target=run, args=(i, 5)) for i in range(k)]
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for t in ths: t.start()
    for t in ths: t.join()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"engines={k} sentences/s={k * per * 5 / dt:.1f}")

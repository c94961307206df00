# Per-chunk timing of the length-bucketed corpus path: cold (first call for a
# shape: graph captures), warm host-API call, and device-staged run.
import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from paper_2008_04885_b200 import shard
from tools.sweep import BASE
prec = {'f32': mt.F32, 'int8': mt.INT8}[sys.argv[1] if len(sys.argv) > 1 else 'int8']
m = mt.Model.create(dict(BASE, num_encoder_layers=20, num_decoder_layers=2), seed=1, precision=prec)
rng = np.random.default_rng(11)
lens = rng.integers(5, 61, 4096)
corpus = [list(map(int, rng.integers(4, 32000, int(n)))) + [3] for n in lens]
order = shard.partition([len(x) for x in corpus], 1)[0]
chunks = shard.batches(order, 256)
bc = mt.BeamConfig(5, 0, 1.0)
def t(f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3
for ci in (0, 1, 5, 10, 15):
    ch = [corpus[i] for i in chunks[ci]]
    cold = t(lambda: m.translate(ch, bc)); warm = t(lambda: m.translate(ch, bc))
    m.stage(ch); dev = t(lambda: m.run_staged(bc))
    print(f"chunk {ci}: n {len(ch)} len {len(ch[0])}-{len(ch[-1])} cold {cold:.1f} ms warm {warm:.1f} ms staged {dev:.1f} ms")
